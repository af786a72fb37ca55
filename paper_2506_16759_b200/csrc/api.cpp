// libh2 C ABI + host driver of Algorithm 1: the level loop, the adaptive
// sample controller (§III-B, updateSamples L386) and the marshaling of per-level
// batch descriptors (§IV-A).  Every arithmetic step runs in the sm_100a kernels of
// sketch.cu / gen_bsr.cu / cpqr.cu / matvec.cu; the host only sizes levels (prefix sums of
// ranks read back once per convergence test) and launches.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "alloc.hpp"
#include "comm.hpp"
#include "kernels.hpp"
#include "tree.hpp"

namespace h2 {
thread_local int64_t g_launches = 0;
void count_launch() { ++g_launches; }
}  // namespace h2

namespace {

thread_local std::string g_err;
thread_local double g_alloc_ms = 0;
   // host time inside cudaMallocAsync (H2_TRACE=1 diagnostics)

// Stream-ordered device array on the libh2 block cache (alloc.hpp): the per-level "single
// allocation per operation" of PAPER.md L384 is a cache hit after the first build.
template <class T>
struct DArr {
  T* p = nullptr;
  int64_t n = 0;
  cudaStream_t st = 0;     // stream the array is freed on (stream order)
  DArr() = default;
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
  DArr& operator=(DArr&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      st = o.st;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DArr() { release(); }
  void release() {
    if (p) h2::cache_free(p, st);
    p = nullptr;
    n = 0;
  }
  // arrays that outlive the build (the H^2 matrix) are freed on the legacy default stream
  void detach() { st = 0; }
  void alloc(int64_t cnt, cudaStream_t stream) {
    release();
    n = cnt;
    st = stream;
    auto t0 = std::chrono::steady_clock::now();
    p = static_cast<T*>(h2::cache_alloc(sizeof(T) * std::max<int64_t>(cnt, 1), stream));
    g_alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc((int64_t)v.size(), st);
    if (!v.empty()) H2_CUDA(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  }
  int64_t bytes() const { return p ? (int64_t)sizeof(T) * std::max<int64_t>(n, 1) : 0; }
};

// one processed depth t of the basis tree
struct Level {
  int t = 0;
  int32_t nclus = 0;
  std::vector<int32_t> m, k;
  std::vector<int64_t> poff, roff, xoff;
  int64_t rows = 0, rtot = 0, xtot = 0;
  int32_t max_m = 0, max_k = 0;
  DArr<int32_t> d_m, d_k, d_perm, d_skel;
  DArr<int64_t> d_poff, d_roff, d_xoff;
  DArr<double> X, cert;
  // couplings of this depth (unique far pairs, s < b)
  std::vector<int64_t> B_off;
  DArr<int64_t> d_B_off;
  DArr<double> B;
};

}  // namespace

struct h2_matrix {
  std::shared_ptr<h2_tree> tree;
  int top = 0, Dl = 0;
  int nranks = 1, rank = 0;   // built with a communicator: rank owns a subtree range per depth
  bool partial = false;       // true until h2_matrix_allgather completed every rank's copy
  int64_t n = 0;
  std::vector<Level> lv;   // index t - top
  DArr<double> D;
  h2_build_stats stats{};
  Level& L(int t) { return lv[t - top]; }
  const Level& L(int t) const { return lv[t - top]; }
  // non-symmetric build (h2_build_nonsym): lv holds the row side (ranks, skeletons I~, bases U/E,
  // and the couplings B_{s,b} of every ORDERED far pair in CSR order), lvc the column side
  // (J~, V/F); D holds every ordered near pair in CSR order at offsets D_off
  bool nonsym = false;
  std::vector<Level> lvc;
  std::vector<int64_t> D_off;
  DArr<int64_t> d_D_off;
  Level& C(int t) { return lvc[t - top]; }
  const Level& C(int t) const { return lvc[t - top]; }
  Level& S(int sd, int t) { return sd ? C(t) : L(t); }
  const Level& S(int sd, int t) const { return sd ? C(t) : L(t); }
};

namespace {

using namespace h2;

struct PhaseTimer {
  cudaStream_t st;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
  int cur = -1;
  cudaEvent_t cur_ev{};
  double host_ms[H2_NPHASE] = {};   // host wall time spent issuing each phase (H2_TRACE=1)
  std::chrono::steady_clock::time_point h0;
  explicit PhaseTimer(cudaStream_t s) : st(s) {}
  // NVTX ranges (SURVEY §5 tracing): one per phase ("h2 sketch", "h2 bsr", ...) nested in one
  // per processed depth ("h2 depth t"), for nsys / ncu --nvtx
  bool depth_open = false;
  void begin(int ph) {
    static const char* names[H2_NPHASE] = {"h2 rand", "h2 sketch", "h2 gen", "h2 bsr", "h2 cpqr", "h2 id", "h2 misc"};
    nvtxRangePushA(names[ph]);
    h0 = std::chrono::steady_clock::now();
    cudaEvent_t e;
    H2_CUDA(cudaEventCreate(&e));
    H2_CUDA(cudaEventRecord(e, st));
    cur = ph;
    cur_ev = e;
  }
  void end() {
    cudaEvent_t e;
    H2_CUDA(cudaEventCreate(&e));
    H2_CUDA(cudaEventRecord(e, st));
    ev.push_back({cur, {cur_ev, e}});
    host_ms[cur] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    nvtxRangePop();
  }
  void collect(double* out) {
    for (auto& x : ev) {
      float ms = 0;
      cudaEventElapsedTime(&ms, x.second.first, x.second.second);
      out[x.first] += ms;
    }
  }
  // per-depth device time (h2_build_stats.t_depth_ms): [mark(t), mark(next)) on the build stream
  std::vector<std::pair<int, cudaEvent_t>> marks;
  void mark(int t) {
    if (depth_open) nvtxRangePop();
    depth_open = t >= 0;
    if (depth_open) {
      char nm[32];
      snprintf(nm, sizeof nm, "h2 depth %d", t);
      nvtxRangePushA(nm);
    }
    cudaEvent_t e;
    H2_CUDA(cudaEventCreate(&e));
    H2_CUDA(cudaEventRecord(e, st));
    marks.push_back({t, e});
  }
  void collect_depths(double* out) {
    for (size_t i = 0; i + 1 < marks.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, marks[i].second, marks[i + 1].second);
      if (marks[i].first >= 0 && marks[i].first < 64) out[marks[i].first] += ms;
    }
  }
  ~PhaseTimer() {
    for (auto& x : ev) {
      cudaEventDestroy(x.second.first);
      cudaEventDestroy(x.second.second);
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
  }
};

template <class T>
std::vector<T> download(const DArr<T>& a, int64_t n, cudaStream_t st) {
  std::vector<T> v(n);
  if (n) H2_CUDA(cudaMemcpyAsync(v.data(), a.p, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaStreamSynchronize(st));
  return v;
}

// Sample panel of one depth: Y^l / Omega^l rows x ld, row-major (a point's samples contiguous,
// the CPQR column of A = (Y^loc)^T).  Columns are appended in place; ld grows on demand.
struct Panel {
  DArr<double> Y, O;
  int64_t rows = 0, ld = 0;
  void alloc(int64_t r, int64_t l, cudaStream_t st) {
    rows = r;
    ld = l;
    Y.alloc(std::max<int64_t>(r, 1) * l, st);
    O.alloc(std::max<int64_t>(r, 1) * l, st);
  }
  void release() {
    Y.release();
    O.release();
    rows = ld = 0;
  }
};

void matvec_impl(const h2_matrix& H, const double* x, int64_t ldx, double* y, int64_t ldy, int32_t q, double alpha,
                 double beta, cudaStream_t st, int rank = 0, int nranks = 1);
void ensure_partition_uploaded(const h2_tree* tree);
bool ensure_near_chunks(const h2_tree* tree);
KernelParams tree_kernel(const h2_tree* tree, const h2_kernel& k, cudaStream_t st);
void apply_sketch_op(const h2_tree& T, const h2_sketch& S, const double* Om, int64_t ldo, int nc, double* Y,
                     int64_t ldy, bool quarters, bool exact, cudaStream_t st);

// Cluster ownership under a communicator (S§8(e)): cluster c of depth t (2^t clusters) belongs
// to rank floor(c P / 2^t).  Ranges are contiguous and subtree-aligned (the children of an owned
// cluster are owned), so every per-cluster array in cluster order has one contiguous segment
// per rank and all-gathers are single in-place allgatherv calls.
inline int own_begin(int t, int r, int P) {
  const int64_t n = int64_t(1) << t;
  return (int)((r * n + P - 1) / P);
}

// in-place all-gather of per-rank byte segments through the caller's communicator
void comm_allgather(const h2_comm* comm, void* base, const std::vector<int64_t>& counts,
                    const std::vector<int64_t>& displs, cudaStream_t st) {
  int64_t tot = 0;
  for (int64_t c : counts) tot += c;
  if (tot == 0) return;
  if (!comm->allgatherv) {   // in-library NCCL: stream-ordered, no host synchronisation
    nccl_allgatherv(comm->nccl, comm->nranks, base, counts.data(), displs.data(), st);
    return;
  }
  // the segments are produced by kernels on `st`; a host-staged communicator reads them on the
  // host side, so complete them first (a few times per level)
  H2_CUDA(cudaStreamSynchronize(st));
  const int rc = comm->allgatherv(comm->ctx, base, counts.data(), displs.data(), st);
  if (rc != 0) throw Error(H2_ERR_CALLBACK, "communicator allgatherv returned " + std::to_string(rc));
}

// all-to-all of byte segments (the column-split sketch exchange, S§8(e)): the caller's
// alltoallv (host-staged: the send segments are completed first) or the in-library NCCL group
void comm_alltoall(const h2_comm* comm, const void* send, const std::vector<int64_t>& sc,
                   const std::vector<int64_t>& sd, void* recv, const std::vector<int64_t>& rc,
                   const std::vector<int64_t>& rd, cudaStream_t st) {
  if (comm->alltoallv) {
    H2_CUDA(cudaStreamSynchronize(st));
    const int r = comm->alltoallv(comm->ctx, send, sc.data(), sd.data(), recv, rc.data(), rd.data(), st);
    if (r != 0) throw Error(H2_ERR_CALLBACK, "communicator alltoallv returned " + std::to_string(r));
    return;
  }
  H2_REQUIRE(comm->nccl, "column-split sketch: the communicator has no all-to-all (alltoallv or NCCL)");
  nccl_alltoallv(comm->nccl, comm->rank, comm->nranks, send, sc.data(), sd.data(), recv, rc.data(), rd.data(), st);
}

// all-gather of a per-cluster array of depth t: element offsets off(c), c in [0, 2^t]
template <class F>
void comm_allgather_clusters(const h2_comm* comm, void* base, size_t es, int t, F off, cudaStream_t st) {
  const int P = comm->nranks;
  std::vector<int64_t> cnt(P), dsp(P);
  for (int r = 0; r < P; ++r) {
    const int64_t a = off(own_begin(t, r, P)), b = off(own_begin(t, r + 1, P));
    dsp[r] = a * (int64_t)es;
    cnt[r] = (b - a) * (int64_t)es;
  }
  comm_allgather(comm, base, cnt, dsp, st);
}

// Per-device internal streams (created once, never destroyed): the build runs on a
// greatest-priority stream linked to the caller's stream by events, the speculative next sketch
// pass on a least-priority stream, so the construction kernels take the SMs as the long sketch
// CTAs retire and the sketch fills the rest (overlap of the O(N^2) pass with the O(N) levels).
cudaStream_t prio_stream(bool high) {
  static std::mutex mu;
  static cudaStream_t s[64][2] = {};
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  cudaStream_t& x = s[dev & 63][high ? 1 : 0];
  if (!x) {
    int lo = 0, hi = 0;
    H2_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    H2_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, high ? hi : lo));
  }
  return x;
}

// per-device side stream of the overlapped per-level all-gathers (default priority)
cudaStream_t side_stream() {
  static std::mutex mu;
  static cudaStream_t s[64] = {};
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  cudaStream_t& x = s[dev & 63];
  if (!x) H2_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  return x;
}

void stream_after(cudaStream_t later, cudaStream_t earlier) {
  cudaEvent_t e;
  H2_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  H2_CUDA(cudaEventRecord(e, earlier));
  H2_CUDA(cudaStreamWaitEvent(later, e, 0));
  H2_CUDA(cudaEventDestroy(e));
}

struct Builder {
  const h2_tree& T;
  const h2_sketch& S;
  const h2_entry& E;
  double tol;
  h2_build_opts o;
  cudaStream_t st;
  h2_matrix& H;
  KernelParams ekp{}, skp{};
  int d = 0;
  Panel cur;                    // full-width panel of the depth being processed
  Panel curc;                   // non-symmetric build: the column-side panel (Z, Omega^l)
  DArr<double> Wc;              // its CPQR workspace
  DArr<double> sumsq_acc;
  DArr<int> nonfinite;
  DArr<double> W;               // CPQR workspace
  DArr<int32_t> fail_flag;      // CPQR early exit of a failing convergence test (CpqrArgs)
  PhaseTimer timer;
  int64_t entries_sketch = 0;
  const h2_comm* comm = nullptr;   // NULL: one GPU
  int P = 1, R = 0;
  cudaStream_t user_st = nullptr;  // the caller's stream (st becomes the internal high-priority one)
  DArr<double> leaf_part;          // per-leaf sums of squares of the current draw
  bool ex = false;                 // exact-order mode (opts.exact_order, exact.cu)

  // Omega columns [c0, c0+nc) (all n rows) -> Od: the h2_omega stream, or the caller's array
  void fill_omega(double* Od, int64_t ld, int c0, int nc, cudaStream_t s) {
    if (o.omega_ext) {
      if (nc > 0)
        H2_CUDA(cudaMemcpy2DAsync(Od, ld * 8, o.omega_ext + c0, o.ld_omega_ext * 8, (size_t)nc * 8, T.n,
                                  cudaMemcpyDeviceToDevice, s));
    } else {
      launch_omega(o.seed, o.stream_id, 0, T.n, c0, nc, Od, ld, s);
    }
  }
  // the int8 tensor-core sketch needs the exactly representable stream (quarters)
  bool quarters() const { return o.omega_ext == nullptr; }
  // explicit dense operator (H2_S_DENSE_MATRIX): the int8 tensor-core product of the h2 stream
  // (one HBM read of A per pass of up to 128 columns) or cuBLAS DGEMM
  bool dense_tc = false;
  double dense_amax = -1.0;
  void dense_op_sketch(const double* Od, int64_t ld, int nc, double* Yd, cudaStream_t s) {
    if (dense_tc) {
      if (dense_amax < 0) dense_amax = dense_absmax(S.A, S.ld_A, T.n, s);
      launch_dense_op_tc(S.A, S.ld_A, T.n, row_b(), row_e(), dense_amax, Od, ld, nc, Yd + row_b() * ld, ld, s);
    } else {
      dense_matrix_sketch(S.A, S.ld_A, T.n, row_b(), row_e(), Od, ld, nc, Yd + row_b() * ld, ld, s);
    }
  }
  void sketch_rows(const double* Od, int64_t ld, int nc, double* Yd, cudaStream_t s) {
    if (ex) launch_exact_sketch(skp, T.d_x, T.d_y, T.d_z, T.n, row_b(), row_e(), Od, ld, nc, Yd + row_b() * ld, ld, s);
    else launch_dense_sketch(skp, T.d_x, T.d_y, T.d_z, T.n, row_b(), row_e(), Od, ld, nc, Yd + row_b() * ld, ld,
                             quarters(), s);
  }

  Builder(const h2_tree& t, const h2_sketch& s, const h2_entry& e, double tl, const h2_build_opts& op,
          cudaStream_t stream, h2_matrix& h, const h2_comm* cm)
      : T(t), S(s), E(e), tol(tl), o(op), st(stream), H(h), timer(stream), comm(cm) {
    if (comm && comm->nranks > 1) {
      P = comm->nranks;
      R = comm->rank;
    } else {
      comm = nullptr;
    }
  }
  // owned clusters [cb(t), ce(t)) of depth t; owned leaf rows [row_b, row_e)
  int cb(int t) const { return own_begin(t, R, P); }
  int ce(int t) const { return own_begin(t, R + 1, P); }
  int64_t leaf_row(int c) const { return c < (1 << T.Dl) ? T.begin[T.Dl][c] : T.n; }
  int64_t row_b() const { return leaf_row(cb(T.Dl)); }
  int64_t row_e() const { return leaf_row(ce(T.Dl)); }

  // unique pairs (us[u], ub[u]) with an owned endpoint (both orientations of every block a
  // BSR row of this rank reads); NULL list = all pairs (one GPU)
  std::vector<int32_t> owned_pairs(const PairCSR& F, int t) const {
    std::vector<int32_t> l;
    for (int64_t u = 0; u < F.nuniq(); ++u) {
      const int a = F.us[u], b = F.ub[u];
      if ((a >= cb(t) && a < ce(t)) || (b >= cb(t) && b < ce(t))) l.push_back((int32_t)u);
    }
    return l;
  }

  // ordered pairs e (row os[e], column F.idx[e]) with an owned endpoint: the blocks a rank's row
  // and column BSRs read in the non-symmetric construction
  std::vector<int32_t> owned_ordered(const PairCSR& F, const std::vector<int32_t>& os, int t) const {
    std::vector<int32_t> l;
    for (int64_t e = 0; e < F.nnz(); ++e) {
      const int a = os[e], b = F.idx[e];
      if ((a >= cb(t) && a < ce(t)) || (b >= cb(t) && b < ce(t))) l.push_back((int32_t)e);
    }
    return l;
  }

  // all-gather rows [roff_r, roff_{r+1}) (per rank) of a row-major panel, columns [0, ncols)
  void allgather_rows(double* p, int64_t ld, int ncols, const std::vector<int64_t>& rowb, int64_t nrows,
                      cudaStream_t s = nullptr) {
    if (!comm || ncols <= 0) return;
    if (!s) s = st;
    std::vector<int64_t> cnt(P), dsp(P);
    if (ld == ncols) {
      for (int r = 0; r < P; ++r) {
        dsp[r] = rowb[r] * ld * 8;
        cnt[r] = (rowb[r + 1] - rowb[r]) * ld * 8;
      }
      comm_allgather(comm, p, cnt, dsp, s);
      return;
    }
    DArr<double> pk;   // packed rows x ncols
    pk.alloc(std::max<int64_t>(nrows, 1) * ncols, s);
    const int64_t r0 = rowb[R], r1 = rowb[R + 1];
    if (r1 > r0)
      H2_CUDA(cudaMemcpy2DAsync(pk.p + r0 * ncols, ncols * 8, p + r0 * ld, ld * 8, (size_t)ncols * 8, r1 - r0,
                                cudaMemcpyDeviceToDevice, s));
    for (int r = 0; r < P; ++r) {
      dsp[r] = rowb[r] * ncols * 8;
      cnt[r] = (rowb[r + 1] - rowb[r]) * ncols * 8;
    }
    comm_allgather(comm, pk.p, cnt, dsp, s);
    if (nrows > 0)
      H2_CUDA(cudaMemcpy2DAsync(p, ld * 8, pk.p, ncols * 8, (size_t)ncols * 8, nrows, cudaMemcpyDeviceToDevice, s));
  }
  // rows of the panel built by shrink(u): skeleton rows of depth u in roff order.  Their only
  // remote reader is the BSR of depth u - 1 (far pairs of depth u, Algorithm 1), so by
  // default (H2_HALO=1, a communicator with an all-to-all) only the HALO moves: rank R sends the
  // rows of its cluster b to rank q iff b has a far partner owned by q (S§8(e): ~0.4x the
  // all-gather bytes at P = 8).  H2_HALO=0: every rank's rows to every rank (all-gather).
  int64_t halo_rows_sent = 0;
  void allgather_skel_rows(int u, double* p, int64_t ld, int ncols, cudaStream_t s = nullptr, int sd = 0) {
    if (!comm) return;
    if (ncols > 0 && (comm->alltoallv || comm->nccl) && env_int("H2_HALO", 1) != 0) {
      halo_skel_rows(u, p, ld, ncols, s ? s : st, sd);
      return;
    }
    const Level& L = H.S(sd, u);
    std::vector<int64_t> rowb(P + 1);
    for (int r = 0; r <= P; ++r) {
      const int c = own_begin(u, r, P);
      rowb[r] = c < L.nclus ? L.roff[c] : L.rtot;
    }
    allgather_rows(p, ld, ncols, rowb, L.rtot, s);
  }
  void halo_skel_rows(int u, double* p, int64_t ld, int ncols, cudaStream_t s, int side = 0) {
    const Level& L = H.S(side, u);
    const PairCSR& F = T.far[u];
    const int n = L.nclus;
    auto owner = [&](int c) { return (int)((int64_t)c * P / n); };
    std::vector<std::vector<int32_t>> sendb(P), recvb(P);
    std::vector<char> mark(P);
    for (int b = cb(u); b < ce(u); ++b) {   // own clusters with a partner owned by q (ascending b)
      std::fill(mark.begin(), mark.end(), 0);
      for (int32_t e = F.ptr[b]; e < F.ptr[b + 1]; ++e) mark[owner(F.idx[e])] = 1;
      for (int q = 0; q < P; ++q)
        if (q != R && mark[q]) sendb[q].push_back(b);
    }
    for (int s0 = cb(u); s0 < ce(u); ++s0)   // remote partners of own clusters, per owner
      for (int32_t e = F.ptr[s0]; e < F.ptr[s0 + 1]; ++e) {
        const int b = F.idx[e], q = owner(b);
        if (q != R) recvb[q].push_back(b);
      }
    std::vector<int32_t> srows, rrows;
    std::vector<int64_t> sc(P, 0), sd(P, 0), rc(P, 0), rd(P, 0);
    for (int q = 0; q < P; ++q) {
      std::sort(recvb[q].begin(), recvb[q].end());
      recvb[q].erase(std::unique(recvb[q].begin(), recvb[q].end()), recvb[q].end());
      sd[q] = (int64_t)srows.size() * ncols * 8;
      for (int b : sendb[q])
        for (int i = 0; i < L.k[b]; ++i) srows.push_back((int32_t)(L.roff[b] + i));
      sc[q] = (int64_t)srows.size() * ncols * 8 - sd[q];
      rd[q] = (int64_t)rrows.size() * ncols * 8;
      for (int b : recvb[q])
        for (int i = 0; i < L.k[b]; ++i) rrows.push_back((int32_t)(L.roff[b] + i));
      rc[q] = (int64_t)rrows.size() * ncols * 8 - rd[q];
    }
    halo_rows_sent += (int64_t)srows.size();
    DArr<int32_t> sr, rr;
    DArr<double> sbuf, rbuf;
    sr.upload(srows, s);
    rr.upload(rrows, s);
    sbuf.alloc(std::max<int64_t>((int64_t)srows.size() * ncols, 1), s);
    rbuf.alloc(std::max<int64_t>((int64_t)rrows.size() * ncols, 1), s);
    launch_rows_move(p, ld, sr.p, (int64_t)srows.size(), ncols, sbuf.p, 0, s);
    comm_alltoall(comm, sbuf.p, sc, sd, rbuf.p, rc, rd, s);
    launch_rows_move(p, ld, rr.p, (int64_t)rrows.size(), ncols, rbuf.p, 1, s);
  }

  // Algorithm 1 line 258 (gen_B) with the all-gather of the parent panel's Omega^{l+1} rows
  // (S§8(e); the BSR partners' samples of the next depth) overlapped: the gather runs on a side
  // stream once the shrink is done while B is generated on the build stream (B needs only the
  // skeletons, gathered in commit); the build stream waits for the gather before the next depth
  // reads the panel.  gen_B is enqueued first, so a host-staged communicator (which blocks the
  // host inside the gather) also overlaps with the device generating B.  H2_AG_OVERLAP=0: serial.
  void gen_B_with_gather(int t, Panel* next, int ncols) {
    if (!comm || !next) {
      gen_B(t);
      return;
    }
    if (env_int("H2_AG_OVERLAP", 1) == 0) {
      allgather_skel_rows(t, next->O.p, next->ld, ncols);
      gen_B(t);
      return;
    }
    cudaStream_t cs = side_stream();
    stream_after(cs, st);
    gen_B(t);
    allgather_skel_rows(t, next->O.p, next->ld, ncols, cs);
    stream_after(st, cs);
  }

  // panel leading dimension: d_max when the panel is small, else the needed width + 2 blocks
  int64_t ld_for(int64_t rows, int dneed) const {
    const int64_t full = o.d_max;
    if (rows * full * 16 <= (int64_t(1) << 30)) return full;
    int64_t l = ((dneed + 2 * (int64_t)o.d_blk + 31) / 32) * 32;
    return std::min<int64_t>(std::max<int64_t>(l, dneed), full);
  }

  // widen panel P to >= dneed columns, keeping its first `keep` columns (default: d)
  void grow(Panel& P, int dneed, int keep = -1) {
    if (dneed <= P.ld) return;
    if (keep < 0) keep = d;
    Panel Q;
    Q.alloc(P.rows, ld_for(P.rows, dneed), st);
    if (P.rows > 0 && keep > 0) {
      H2_CUDA(cudaMemcpy2DAsync(Q.Y.p, Q.ld * 8, P.Y.p, P.ld * 8, (size_t)keep * 8, P.rows, cudaMemcpyDeviceToDevice, st));
      H2_CUDA(cudaMemcpy2DAsync(Q.O.p, Q.ld * 8, P.O.p, P.ld * 8, (size_t)keep * 8, P.rows, cudaMemcpyDeviceToDevice, st));
    }
    P = std::move(Q);
  }

  // ---------------------------------------------------------------- sketch of stream columns
  // Omega(:, c0:c0+nc) -> Od, Y = K_blk(Omega) -> Yd (pointers at the first destination column)
  // Speculative sketch columns: the int8 tensor-core
  // sketch is bound by the FP64 evaluation of K, and one pass contracts each K tile with up to
  // W = sketch_tc_pass_cols() (128) Omega columns at the same evaluation cost as 32.  A draw of
  // nc < W columns therefore computes the whole pass and keeps the extra columns c0+nc.. for the
  // next updateSamples draws.  Omega columns are counter-based and every sketch column is computed
  // independently (exact integer accumulation), so the samples consumed are bit-identical to
  // unspeculated draws.
  bool spec_on = false;
  int spec_w = 64;              // pass width W
  Panel spec;                   // n x W: columns [spec_c0, spec_c0 + spec_n) at offset spec_off
  int spec_c0 = -1, spec_n = 0, spec_off = 0;
  int64_t sketch_columns = 0;
  // Optional (H2_PREFETCH=1): the pass after the first one is computed ahead, on the low-priority
  // stream, while the leaf and lower levels are constructed (large problems need > W samples); a
  // draw that reaches its columns waits for it; unused, it is waited for at the end of the build.
  // Measured at N=2^18: 519 vs 526 ms (the construction slows down under the shared SMs), so it
  // is off by default.
  Panel pre;
  int pre_c0 = -1;
  bool pre_live = false, pre_started = false;
  cudaEvent_t pre_done = nullptr;

  void launch_prefetch(int c0) {
    cudaStream_t ss = prio_stream(false);
    stream_after(ss, st);
    pre.alloc(T.n, spec_w, ss);
    cudaEvent_t t0, t1;
    H2_CUDA(cudaEventCreate(&t0));
    H2_CUDA(cudaEventCreate(&t1));
    H2_CUDA(cudaEventRecord(t0, ss));
    fill_omega(pre.O.p, pre.ld, c0, spec_w, ss);
    launch_dense_sketch(skp, T.d_x, T.d_y, T.d_z, T.n, row_b(), row_e(), pre.O.p, pre.ld, spec_w,
                        pre.Y.p + row_b() * pre.ld, pre.ld, true, ss);
    H2_CUDA(cudaEventRecord(t1, ss));
    timer.ev.push_back({H2_PH_SKETCH, {t0, t1}});
    H2_CUDA(cudaEventCreateWithFlags(&pre_done, cudaEventDisableTiming));
    H2_CUDA(cudaEventRecord(pre_done, ss));
    entries_sketch += T.n * T.n;
    sketch_columns += spec_w;
    pre_c0 = c0;
    pre_live = pre_started = true;
  }
  void join_prefetch() {
    if (!pre_live) return;
    H2_CUDA(cudaStreamWaitEvent(st, pre_done, 0));
    H2_CUDA(cudaEventDestroy(pre_done));
    pre_live = false;
  }

  void sketch_cols(double* Yd, double* Od, int64_t ld, int c0, int nc) {
    fill_omega(Od, ld, c0, nc, st);
    timer.end();
    timer.begin(H2_PH_SKETCH);
    // this rank's leaf rows only (Omega is regenerated for all rows on every rank)
    sketch_rows(Od, ld, nc, Yd, st);
    entries_sketch += T.n * T.n * (int64_t)div_up(nc, spec_on ? spec_w : 64);
    sketch_columns += nc;
  }

  // H2_S_CALLBACK sketch of stream columns [c0, c0+nc) (Od/Yd at the draw's first column):
  // this rank's leaf rows of Y.  Row split (default): one call for the rank's rows.  Column split
  // (opts.sketch_split = H2_SPLIT_COLS under a communicator, S§8(e)): the callback produces ALL n
  // rows of this rank's column slice [c_R, c_{R+1}), c_r = floor(r nc / P), into a packed n x w
  // panel whose rows of rank h are one contiguous segment; one all-to-all moves segment h to rank
  // h, which receives its rows of every slice (packed per source rank) and scatters them into Yd.
  int64_t a2a_bytes = 0;
  void callback_sketch(const double* Od, int64_t ld, int c0, int nc, double* Yd) {
    h2_sketch_req rq{};
    rq.n = T.n;
    rq.omega = Od;
    rq.ld_omega = ld;
    rq.stream = st;
    if (!comm || o.sketch_split != H2_SPLIT_COLS) {
      rq.row_begin = row_b();
      rq.row_end = row_e();
      rq.col0 = c0;
      rq.ncols = nc;
      rq.y = Yd + row_b() * ld;
      rq.ld_y = ld;
      const int rc = S.fn(S.ctx, &rq);
      if (rc != 0) throw Error(H2_ERR_CALLBACK, "sketch callback returned " + std::to_string(rc));
      return;
    }
    std::vector<int> cs(P + 1);
    std::vector<int64_t> rb(P + 1);
    for (int r = 0; r <= P; ++r) {
      cs[r] = (int)((int64_t)r * nc / P);
      rb[r] = leaf_row(own_begin(T.Dl, r, P));
    }
    const int w = cs[R + 1] - cs[R];
    const int64_t mine = rb[R + 1] - rb[R];
    DArr<double> sb, rbuf;
    sb.alloc(std::max<int64_t>(T.n * w, 1), st);
    rbuf.alloc(std::max<int64_t>(mine * nc, 1), st);
    if (w > 0) {
      rq.row_begin = 0;
      rq.row_end = T.n;
      rq.col0 = c0 + cs[R];
      rq.ncols = w;
      rq.omega = Od + cs[R];
      rq.y = sb.p;
      rq.ld_y = w;
      const int rc = S.fn(S.ctx, &rq);
      if (rc != 0) throw Error(H2_ERR_CALLBACK, "sketch callback returned " + std::to_string(rc));
    }
    std::vector<int64_t> sc(P), sd(P), rc(P), rd(P);
    for (int h = 0; h < P; ++h) {
      sd[h] = rb[h] * w * 8;
      sc[h] = (rb[h + 1] - rb[h]) * w * 8;
      rd[h] = mine * cs[h] * 8;
      rc[h] = mine * (cs[h + 1] - cs[h]) * 8;
      if (h != R) a2a_bytes += sc[h];
    }
    comm_alltoall(comm, sb.p, sc, sd, rbuf.p, rc, rd, st);
    for (int h = 0; h < P; ++h) {
      const int wh = cs[h + 1] - cs[h];
      if (wh > 0 && mine > 0)
        H2_CUDA(cudaMemcpy2DAsync(Yd + rb[R] * ld + cs[h], ld * 8, rbuf.p + mine * cs[h], (size_t)wh * 8,
                                  (size_t)wh * 8, mine, cudaMemcpyDeviceToDevice, st));
    }
  }

  // ---------------------------------------------------------------- sketch of stream columns
  // Omega(:, c0:c0+nc) -> Od, Y = K_blk(Omega) -> Yd (pointers at the first destination column)
  void draw(double* Yd, double* Od, int64_t ld, int c0, int nc) {
    timer.begin(H2_PH_RAND);
    if (pre_live && spec_n == 0 && c0 == pre_c0) {   // the prefetched pass becomes the bank
      join_prefetch();
      std::swap(spec, pre);
      spec_c0 = pre_c0;
      spec_n = spec_w;
      spec_off = 0;
    }
    if (S.kind == H2_S_DENSE_KERNEL && spec_on && nc < spec_w && c0 == spec_c0 && nc <= spec_n) {
      H2_CUDA(cudaMemcpy2DAsync(Yd, ld * 8, spec.Y.p + spec_off, spec.ld * 8, (size_t)nc * 8, T.n,
                                cudaMemcpyDeviceToDevice, st));
      H2_CUDA(cudaMemcpy2DAsync(Od, ld * 8, spec.O.p + spec_off, spec.ld * 8, (size_t)nc * 8, T.n,
                                cudaMemcpyDeviceToDevice, st));
      spec_c0 += nc;
      spec_n -= nc;
      spec_off += nc;
      timer.end();
      timer.begin(H2_PH_SKETCH);
    } else if (S.kind == H2_S_DENSE_KERNEL && spec_on && nc < spec_w && c0 + spec_w <= o.d_max) {
      if (spec.rows == 0) spec.alloc(T.n, spec_w, st);
      sketch_cols(spec.Y.p, spec.O.p, spec.ld, c0, spec_w);
      H2_CUDA(cudaMemcpy2DAsync(Yd, ld * 8, spec.Y.p, spec.ld * 8, (size_t)nc * 8, T.n, cudaMemcpyDeviceToDevice, st));
      H2_CUDA(cudaMemcpy2DAsync(Od, ld * 8, spec.O.p, spec.ld * 8, (size_t)nc * 8, T.n, cudaMemcpyDeviceToDevice, st));
      spec_c0 = c0 + nc;
      spec_n = spec_w - nc;
      spec_off = nc;
      if (!pre_started && skp.kind == H2_K_EXP && c0 + 2 * spec_w <= o.d_max && env_int("H2_PREFETCH", 0) != 0)
        launch_prefetch(c0 + spec_w);
    } else if (S.kind == H2_S_DENSE_KERNEL) {
      sketch_cols(Yd, Od, ld, c0, nc);
    } else {
      fill_omega(Od, ld, c0, nc, st);
      timer.end();
      timer.begin(H2_PH_SKETCH);
      sketch_columns += nc;
      if (S.kind == H2_S_DENSE_MATRIX) {
        dense_op_sketch(Od, ld, nc, Yd, st);
      } else if (S.kind == H2_S_H2_LOWRANK) {
        // K_blk = A_H Omega + U (U^T Omega); under a communicator the rank's
        // own leaf rows only (row-sharded matvec of the complete, replicated base)
        matvec_impl(*S.base, Od, ld, Yd, ld, nc, 1.0, 0.0, st, R, P);
        DArr<double> scr;
        scr.alloc((int64_t)(div_up(T.n, 1024) + 1) * S.rank * nc, st);
        launch_lowrank_sketch(S.U, S.ld_U, S.rank, Od, ld, nc, T.n, Yd, ld, scr.p, st);
      } else {
        callback_sketch(Od, ld, c0, nc, Yd);
      }
    }
    timer.end();
    timer.begin(H2_PH_MISC);
    // R10: ||Y||_F^2 accumulated over the draws; per-leaf partials (owned leaves), all-gathered,
    // summed in leaf order: bitwise the same for any number of GPUs
    const int nleaf = 1 << T.Dl;
    if (leaf_part.n < nleaf) leaf_part.alloc(nleaf, st);
    if (ex) launch_exact_sumsq_leaf(Yd, T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ld, 0, nc, leaf_part.p, st);
    else launch_sumsq_leaf(Yd, T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ld, 0, nc, leaf_part.p, st);
    if (comm) comm_allgather_clusters(comm, leaf_part.p, 8, T.Dl, [](int c) { return (int64_t)c; }, st);
    if (ex) launch_exact_sumsq_total(leaf_part.p, nleaf, sumsq_acc.p, nonfinite.p, st);
    else launch_sumsq_total(leaf_part.p, nleaf, sumsq_acc.p, nonfinite.p, st);
    timer.end();
  }

  // nu ~ ||K||_2 by power iteration through the sketch operator ("an approximate
  // norm ... provided via sketching"; literal rule with opts.norm <= 0): x = e/|e| with e column 0
  // of the h2_omega stream (seed, stream_id + 3); y = K_blk x; nu = |y|; x = y (norm_iters times).
  // Replicated on every rank (all rows), so every rank holds the same nu.
  double estimate_norm() {
    timer.begin(H2_PH_SKETCH);
    const int nleaf = 1 << T.Dl;
    DArr<double> x, y, part, acc;
    DArr<int> nf;
    x.alloc(T.n, st);
    y.alloc(T.n, st);
    part.alloc(nleaf, st);
    acc.alloc(1, st);
    nf.alloc(1, st);
    launch_omega(o.seed, o.stream_id + 3, 0, T.n, 0, 1, x.p, 1, st);
    auto norm2 = [&](const double* v) {
      H2_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double), st));
      H2_CUDA(cudaMemsetAsync(nf.p, 0, sizeof(int), st));
      launch_sumsq_leaf(v, T.d_leaf_begin, 0, nleaf, 1, 0, 1, part.p, st);
      launch_sumsq_total(part.p, nleaf, acc.p, nf.p, st);
      double a = 0;
      int bad = 0;
      H2_CUDA(cudaMemcpyAsync(&a, acc.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      H2_CUDA(cudaMemcpyAsync(&bad, nf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      H2_CUDA(cudaStreamSynchronize(st));
      if (bad) throw Error(H2_ERR_NONFINITE, "norm estimate: non-finite sketch sample");
      return std::sqrt(a);
    };
    double nu = 0;
    const int iters = std::max(1, o.norm_iters);
    for (int it = 0; it < iters; ++it) {
      const double nx = norm2(x.p);
      if (!(nx > 0)) break;
      launch_scale(x.p, T.n, 1, 1, 1.0 / nx, st);
      apply_sketch_op(T, S, x.p, 1, 1, y.p, 1, false, ex, st);
      nu = norm2(y.p);
      std::swap(x, y);
    }
    timer.end();
    return nu;
  }

  double eps_now(int t) {
    // level schedule (R31, S§8(f) NEXT #2 study): eps_t = eps * eps_decay^(Dl - t)
    const double lvl = o.eps_decay == 1.0 ? 1.0 : std::pow(o.eps_decay, (double)(T.Dl - t));
    double acc = 0;
    int nf = 0;
    H2_CUDA(cudaMemcpyAsync(&acc, sumsq_acc.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaMemcpyAsync(&nf, nonfinite.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaStreamSynchronize(st));
    if (nf) throw Error(H2_ERR_NONFINITE, "the sketch produced a non-finite sample");
    // non-symmetric: acc holds ||Y||^2 + ||Z||^2 (R29: RMS over both sketches)
    if (o.tol_rule == H2_TOL_RMS) return lvl * (o.tol_safety * tol * std::sqrt(acc / (double)(ns ? 2 * T.n : T.n)));
    return lvl * (tol * o.norm);
  }

  // ---------------------------------------------------------------- batched entry generation
  void gen(const GenArgs& g) {
    if (g.nblocks == 0) return;
    timer.begin(H2_PH_GEN);
    if (E.kind == H2_E_BUILTIN) {
      launch_gen(ekp, T.d_x, T.d_y, T.d_z, g, st);
    } else if (E.kind == H2_E_DENSE_MATRIX) {
      launch_gen_dense(E.A, E.ld_A, g, st);
    } else {
      DArr<int32_t> m, nc, ld;
      DArr<int64_t> ro, co;
      DArr<double*> outp;
      m.alloc(g.nblocks, st);
      nc.alloc(g.nblocks, st);
      ld.alloc(g.nblocks, st);
      ro.alloc(g.nblocks, st);
      co.alloc(g.nblocks, st);
      outp.alloc(g.nblocks, st);
      launch_gen_batch_desc(g, m.p, nc.p, ro.p, co.p, outp.p, ld.p, st);
      h2_block_batch bb{g.nblocks, m.p, nc.p, ro.p, co.p, g.idx, g.idx2 ? g.idx2 : g.idx, outp.p, ld.p, st};
      int rc = E.fn(E.ctx, &bb);
      if (rc != 0) throw Error(H2_ERR_CALLBACK, "entry callback returned " + std::to_string(rc));
      H2_CUDA(cudaStreamSynchronize(st));
    }
    timer.end();
  }

  // ---------------------------------------------------------------- algorithmic work (stats)
  // h2_build_stats.work_flops / work_bytes (DESIGN.md §6 "whole-build roofline"): what the
  // method computes and moves per phase, counted on the host from the partition and the ranks
  double wf[H2_NPHASE] = {}, wb[H2_NPHASE] = {};
  std::map<int, std::pair<double, double>> bsr_work;   // depth t -> (sum rows_s cols_b, rows)
  std::pair<double, double> bsr_entries(int t) {
    auto it = bsr_work.find(t);
    if (it != bsr_work.end()) return it->second;
    const bool leaf = t == T.Dl;
    const PairCSR& P = leaf ? T.near : T.far[t + 1];
    const int tc = leaf ? T.Dl : t + 1;
    auto rows = [&](int c) -> double {
      return leaf ? (double)(T.end[T.Dl][c] - T.begin[T.Dl][c]) : (double)H.L(t + 1).k[c];
    };
    double e = 0, r = 0;
    for (int c = cb(tc); c < ce(tc); ++c) {
      const double rc = rows(c);
      r += rc;
      for (int q = P.ptr[c]; q < P.ptr[c + 1]; ++q) e += rc * rows(P.idx[q]);
    }
    return bsr_work[t] = {e, r};
  }

  // ---------------------------------------------------------------- leaf subtraction (L213)
  // With the built-in exp dense-kernel sketch on the tensor cores and the same kernel as the entry
  // evaluator, Y^loc = Y - sum_{b in N} D_{tau,b} Omega_b is computed from the kernel itself on the
  // int8 tensor cores (launch_near_sketch_tc: near leaves only, the sketch's fixed-point K) instead
  // of the BSR product over the stored D blocks: no D read from HBM (the D blocks are still
  // generated for the H^2).  H2_NEAR_TC=0 keeps the BSR path.
  bool near_tc_ok(int nc) {
    static const bool on = env_int("H2_NEAR_TC", 1) != 0;
    if (!on || ex || !spec_on || S.kind != H2_S_DENSE_KERNEL || S.kern.kind != H2_K_EXP) return false;
    if (E.kind != H2_E_BUILTIN || E.kern.kind != S.kern.kind || E.kern.param != S.kern.param) return false;
    if (nc > sketch_tc_pass_cols(skp.kind)) return false;
    return ensure_near_chunks(&T);
  }
  void leaf_subtract(double* Yp, const double* Op, int64_t ld, int nc) {
    if (!near_tc_ok(nc)) {
      bsr(T.Dl, Yp, Op, ld, nc);
      return;
    }
    timer.begin(H2_PH_BSR);
    const auto er = bsr_entries(T.Dl);   // the same algorithmic work as the BSR form
    wf[H2_PH_BSR] += 2.0 * nc * er.first;
    wb[H2_PH_BSR] += 8.0 * nc * 3.0 * er.second;
    // Omega: every row (the near leaves' j), Y: this rank's leaf rows
    launch_near_sketch_tc(skp, T.d_x, T.d_y, T.d_z, T.n, row_b(), row_e(), Op, ld, nc, Yp + row_b() * ld, ld,
                          T.d_nl_ptr, T.d_nl_chunk, T.d_nl_mask, st);
    timer.end();
  }

  // ---------------------------------------------------------------- BSR subtraction on a panel of depth t
  // leaf (t == Dl): Y(I_tau) -= sum_{b in N_tau} D Om(I_b)   (L213)
  // inner: Y^l_t(rows of child nu) -= sum_{b in F_nu} B_{nu,b} Om^l_t(rows of b)   (L240-243)
  // Y, O point at the first column to update; nc columns.
  void bsr(int t, double* Yp, const double* Op, int64_t ld, int nc) {
    timer.begin(H2_PH_BSR);
    BsrArgs a{};
    a.c0 = 0;
    a.ncols = nc;
    if (t == T.Dl) {
      a.c_begin = cb(T.Dl);
      a.nclusters = ce(T.Dl) - cb(T.Dl);
      a.max_rows = H.L(T.Dl).max_m;
      a.yoff = a.ooff = T.d_leaf_begin;
      a.cnt = T.d_leaf_size;
      a.ptr = T.d_near.ptr;
      a.idx = T.d_near.idx;
      a.uidx = T.d_near.uidx;
      a.us = T.d_near.us;
      a.blk_off = T.d_D_off;
      a.blk = H.D.p;
    } else {
      Level& C = H.L(t + 1);
      a.c_begin = cb(t + 1);
      a.nclusters = ce(t + 1) - cb(t + 1);
      a.max_rows = C.max_k;
      a.yoff = a.ooff = C.d_roff.p;
      a.cnt = C.d_k.p;
      a.ptr = T.d_far[t + 1].ptr;
      a.idx = T.d_far[t + 1].idx;
      a.uidx = T.d_far[t + 1].uidx;
      a.us = T.d_far[t + 1].us;
      a.blk_off = C.d_B_off.p;
      a.blk = C.B.p;
    }
    a.Y = Yp;
    a.Om = Op;
    a.ldy = a.ldo = ld;
    {
      const auto er = bsr_entries(t);   // block entries (each orientation) read once, Y in/out, Omega once
      wf[H2_PH_BSR] += 2.0 * nc * er.first;
      wb[H2_PH_BSR] += 8.0 * er.first + 8.0 * nc * 3.0 * er.second;
    }
    if (ex) launch_exact_bsr(a, st);
    else launch_bsr(a, st);
    timer.end();
  }

  // ---------------------------------------------------------------- level set-up
  void setup_level(int t, int sd = 0) {
    Level& L = H.S(sd, t);
    L.t = t;
    L.nclus = 1 << t;
    L.m.resize(L.nclus);
    L.poff.resize(L.nclus);
    if (t == T.Dl) {
      for (int c = 0; c < L.nclus; ++c) {
        L.m[c] = (int32_t)(T.end[t][c] - T.begin[t][c]);
        L.poff[c] = T.begin[t][c];
      }
    } else {
      const Level& C = H.S(sd, t + 1);
      for (int c = 0; c < L.nclus; ++c) {
        L.m[c] = C.k[2 * c] + C.k[2 * c + 1];
        L.poff[c] = C.roff[2 * c];
      }
    }
    L.rows = 0;
    L.max_m = 0;
    for (int c = 0; c < L.nclus; ++c) {
      L.rows += L.m[c];
      L.max_m = std::max(L.max_m, L.m[c]);
    }
    L.d_m.upload(L.m, st);
    L.d_poff.upload(L.poff, st);
    L.d_k.alloc(L.nclus, st);
    L.d_perm.alloc(std::max<int64_t>(L.rows, 1), st);
    L.cert.alloc(2 * L.nclus, st);
  }

  // CPQR of every panel of depth t (current panel, d columns); returns host ranks
  void cpqr(int t, double eps, int sd = 0) {
    Level& L = H.S(sd, t);
    DArr<double>& W = sd ? Wc : this->W;
    const Panel& cur = sd ? curc : this->cur;
    int64_t need = std::max<int64_t>(L.rows * d, 1);
    if (W.n < need) W.alloc(need, st);
    timer.begin(H2_PH_CPQR);
    CpqrArgs a{};
    a.c_begin = cb(t);
    a.nclusters = ce(t) - cb(t);
    a.max_m = std::max(L.max_m, 1);
    a.Y = cur.Y.p;
    a.ldy = cur.ld;
    a.poff = L.d_poff.p;
    a.m = L.d_m.p;
    a.d = d;
    a.eps = eps;
    a.kmax = o.max_rank;
    a.W = W.p;
    a.k = L.d_k.p;
    a.perm = L.d_perm.p;
    a.cert = L.cert.p;
    a.rows = L.rows;
    // adaptive early exit of a failing convergence test (CpqrArgs::fail_cap; H2_CQ_EARLY=0: off):
    // the level decision is unchanged, the discarded round stops at the first definitive failure
    const int pos = (o.tol_rule == H2_TOL_RMS) ? o.p_os : 0;
    if (o.adaptive && !ex && d - pos - 1 >= 0 && env_int("H2_CQ_EARLY", 1) != 0) {
      if (fail_flag.n == 0) fail_flag.alloc(1, st);
      H2_CUDA(cudaMemsetAsync(fail_flag.p, 0, sizeof(int32_t), st));
      a.fail_cap = d - pos - 1;
      a.fail_k = d - pos;
      a.fail_flag = fail_flag.p;
    }
    if (ex) {
      launch_exact_cpqr(a, st);
      H.stats.cpqr_variants |= H2_CQ_V_EXACT;
    } else {
      H.stats.cpqr_variants |= launch_cpqr(a, st);
    }
    timer.end();
    if (comm) comm_allgather_clusters(comm, L.d_k.p, 4, t, [](int c) { return (int64_t)c; }, st);
    L.k = download(L.d_k, L.nclus, st);
    for (int c = cb(t); c < ce(t); ++c) {   // sum_{i<k} 4 (d-i)(m-i); panel read + written
      const double kk = L.k[c], mm = L.m[c], dd = d;
      wf[H2_PH_CPQR] += 4.0 * (kk * dd * mm - (dd + mm) * kk * (kk - 1) / 2 + (kk - 1) * kk * (2 * kk - 1) / 6);
      wb[H2_PH_CPQR] += 16.0 * dd * mm;
    }
  }

  void commit(int t, int sd = 0) {
    Level& L = H.S(sd, t);
    DArr<double>& W = sd ? Wc : this->W;
    L.roff.assign(L.nclus, 0);
    L.xoff.assign(L.nclus, 0);
    L.rtot = L.xtot = 0;
    L.max_k = 0;
    for (int c = 0; c < L.nclus; ++c) {
      L.roff[c] = L.rtot;
      L.xoff[c] = L.xtot;
      L.rtot += L.k[c];
      L.xtot += (int64_t)L.m[c] * L.k[c];
      L.max_k = std::max(L.max_k, L.k[c]);
    }
    L.d_roff.upload(L.roff, st);
    L.d_xoff.upload(L.xoff, st);
    L.X.alloc(L.xtot, st);
    L.d_skel.alloc(L.rtot, st);
    timer.begin(H2_PH_ID);
    IdArgs a{};
    a.c_begin = cb(t);
    a.nclusters = ce(t) - cb(t);
    a.W = W.p;
    a.d = d;
    a.poff = L.d_poff.p;
    a.m = L.d_m.p;
    a.k = L.d_k.p;
    a.perm = L.d_perm.p;
    a.xoff = L.d_xoff.p;
    a.X = L.X.p;
    a.ibar = (t == T.Dl) ? T.d_iota : H.S(sd, t + 1).d_skel.p;
    a.roff = L.d_roff.p;
    a.skel = L.d_skel.p;
    a.max_k = L.max_k;
    a.max_red = 0;
    for (int c = 0; c < L.nclus; ++c) a.max_red = std::max(a.max_red, L.m[c] - L.k[c]);
    if (ex) launch_exact_id(a, st);
    else launch_id(a, st);
    for (int c = cb(t); c < ce(t); ++c) {   // T = R11^-1 R12: k^2 (m-k); R read, X written
      const double kk = L.k[c], mm = L.m[c];
      wf[H2_PH_ID] += kk * kk * (mm - kk);
      wb[H2_PH_ID] += 8.0 * (mm * kk + kk * mm);
    }
    if (comm)   // skeletons I~ of every cluster (B generation of cross-rank pairs, parent Ibar)
      comm_allgather_clusters(comm, L.d_skel.p, 4, t,
                              [&](int c) { return c < L.nclus ? L.roff[c] : L.rtot; }, st);
    timer.end();
  }

  // batchedShrink + Omega upsweep of committed depth u, nc columns: source panel (depth u)
  // -> destination panel (depth u-1); pointers at the first column of each.
  void shrink(int u, const double* Ys, const double* Os, int64_t lds, double* Yd, double* Od, int64_t ldd, int nc,
              int sd = 0) {
    Level& L = H.S(sd, u);
    timer.begin(H2_PH_ID);
    ShrinkArgs a{};
    a.c_begin = cb(u);
    a.nclusters = ce(u) - cb(u);
    a.poff = L.d_poff.p;
    a.m = L.d_m.p;
    a.k = L.d_k.p;
    a.perm = L.d_perm.p;
    a.xoff = L.d_xoff.p;
    a.X = L.X.p;
    a.roff = L.d_roff.p;
    a.Yl = Ys;
    a.Ol = Os;
    a.ld = lds;
    a.Yp = Yd;
    a.Op = Od;
    a.ldp = ldd;
    a.c0 = 0;
    a.c1 = nc;
    a.max_k = L.max_k;
    launch_shrink_project(a, st);
    for (int c = cb(u); c < ce(u); ++c) {   // 2 k (m-k) nc; Y^l, Omega^l rows in, skeleton rows out
      const double kk = L.k[c], mm = L.m[c];
      wf[H2_PH_ID] += 2.0 * kk * (mm - kk) * nc;
      wb[H2_PH_ID] += 8.0 * nc * (2.0 * mm + 2.0 * kk);
    }
    timer.end();
  }

  void gen_B(int t) {
    Level& L = H.L(t);
    const PairCSR& F = T.far[t];
    L.B_off.assign(F.nuniq() + 1, 0);
    for (int64_t u = 0; u < F.nuniq(); ++u)
      L.B_off[u + 1] = L.B_off[u] + (int64_t)L.k[F.us[u]] * L.k[F.ub[u]];
    L.d_B_off.upload(L.B_off, st);
    L.B.alloc(L.B_off.back(), st);
    GenArgs g{};
    g.nblocks = F.nuniq();
    DArr<int32_t> ul;
    if (comm) {
      const std::vector<int32_t> l = owned_pairs(F, t);
      ul.upload(l, st);
      g.ulist = ul.p;
      g.nblocks = (int64_t)l.size();
    }
    g.us = T.d_far[t].us;
    g.ub = T.d_far[t].ub;
    g.cnt = L.d_k.p;
    g.off = L.d_roff.p;
    g.idx = L.d_skel.p;
    g.out_off = L.d_B_off.p;
    g.out = L.B.p;
    if (E.kind == H2_E_H2_LOWRANK) update_B(t);
    else gen(g);
  }

  // B blocks of M = A_H + U U^T at depth t (PAPER.md L445 entry extraction; h2update.cu)
  DArr<const int32_t*> base_k;
  DArr<const int64_t*> base_xoff;
  DArr<const double*> base_X;
  // R_s = A's expanded basis rows at the skeletons of level Ln (depth t), kn_s x kb_s per cluster
  void expand_base_rows(int t, const Level& Ln, DArr<double>& R, std::vector<int64_t>& rowoff,
                        DArr<int64_t>& d_rowoff) {
    const h2_matrix& A = *E.base;
    const Level& La = A.L(t);
    if (!base_k.p) {   // per-depth device pointers of A's levels
      std::vector<const int32_t*> kk(T.Dl + 1, nullptr);
      std::vector<const int64_t*> xo(T.Dl + 1, nullptr);
      std::vector<const double*> xx(T.Dl + 1, nullptr);
      for (int u = A.top; u <= A.Dl; ++u) {
        kk[u] = A.L(u).d_k.p;
        xo[u] = A.L(u).d_xoff.p;
        xx[u] = A.L(u).X.p;
      }
      base_k.upload(kk, st);
      base_xoff.upload(xo, st);
      base_X.upload(xx, st);
    }
    rowoff.assign(Ln.nclus + 1, 0);
    std::vector<int32_t> ptc(std::max<int64_t>(Ln.rtot, 1), 0);
    int kmax = 1;
    for (int c = 0; c < Ln.nclus; ++c) {
      rowoff[c + 1] = rowoff[c] + (int64_t)Ln.k[c] * La.k[c];
      for (int i = 0; i < Ln.k[c]; ++i) ptc[Ln.roff[c] + i] = c;
    }
    for (int u = t; u <= T.Dl; ++u)
      for (int32_t kv : A.L(u).k) kmax = std::max(kmax, kv);
    DArr<int32_t> d_ptc;
    d_rowoff.upload(rowoff, st);
    d_ptc.upload(ptc, st);
    R.alloc(std::max<int64_t>(rowoff.back(), 1), st);
    ExpandArgs ea{};
    ea.npoints = Ln.rtot;
    ea.pt_cluster = d_ptc.p;
    ea.roff_new = Ln.d_roff.p;
    ea.skel_new = Ln.d_skel.p;
    ea.nleaf = 1 << T.Dl;
    ea.leaf_begin = T.d_leaf_begin;
    ea.Dl = T.Dl;
    ea.t = t;
    ea.kb = base_k.p;
    ea.xoff = base_xoff.p;
    ea.X = base_X.p;
    ea.kmax = kmax;
    ea.R = R.p;
    ea.rowoff = d_rowoff.p;
    launch_expand_rows(ea, st);
  }

  void update_B(int t) {
    Level& L = H.L(t);
    const h2_matrix& A = *E.base;
    const Level& La = A.L(t);
    const PairCSR& F = T.far[t];
    if (F.nuniq() == 0) return;
    timer.begin(H2_PH_GEN);
    std::vector<int64_t> rowoff;
    DArr<int64_t> d_rowoff;
    DArr<double> R;
    expand_base_rows(t, L, R, rowoff, d_rowoff);
    int64_t gmax = 1;
    for (int64_t u = 0; u < F.nuniq(); ++u)
      gmax = std::max<int64_t>(gmax, (int64_t)La.k[F.us[u]] * L.k[F.ub[u]]);
    DArr<int32_t> ul;
    int64_t nb = F.nuniq();
    if (comm) {   // the rank's owned pairs (as gen_B)
      const std::vector<int32_t> l = owned_pairs(F, t);
      ul.upload(l, st);
      nb = (int64_t)l.size();
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nb, 148 * 4));
    DArr<double> scratch;
    scratch.alloc(gmax * grid, st);
    UpdateBArgs ba{};
    ba.nblocks = nb;
    ba.ulist = ul.p;
    ba.us = T.d_far[t].us;
    ba.ub = T.d_far[t].ub;
    ba.kn = L.d_k.p;
    ba.kb = La.d_k.p;
    ba.out = L.B.p;
    ba.out_off = L.d_B_off.p;
    ba.R = R.p;
    ba.rowoff = d_rowoff.p;
    ba.Bbase = La.B.p;
    ba.Boff = La.d_B_off.p;
    ba.U = E.U;
    ba.ldu = E.ld_U;
    ba.r = E.rank;
    ba.skel = L.d_skel.p;
    ba.roff_new = L.d_roff.p;
    ba.scratch = scratch.p;
    ba.gmax = gmax;
    launch_update_B(ba, grid, st);
    timer.end();
  }

  // updateSamples (L216-217, L246-247, L386): one new block of b stream columns, swept up through
  // the committed depths Dl..t+1 with the stored D/B/J/U/E, appended to the panel of depth t.
  // Intermediate depths use b-wide scratch panels; only depth t holds all d columns.
  void update_samples(int t, int b) {
    const int c0 = d;
    grow(cur, d + b);
    if (t == T.Dl) {
      draw(cur.Y.p + c0, cur.O.p + c0, cur.ld, c0, b);
      leaf_subtract(cur.Y.p + c0, cur.O.p + c0, cur.ld, b);
      return;
    }
    Panel src;
    src.alloc(T.n, b, st);
    draw(src.Y.p, src.O.p, b, c0, b);
    leaf_subtract(src.Y.p, src.O.p, b, b);
    for (int u = T.Dl; u > t; --u) {
      if (u - 1 == t) {
        shrink(u, src.Y.p, src.O.p, src.ld, cur.Y.p + c0, cur.O.p + c0, cur.ld, b);
        allgather_skel_rows(u, cur.O.p + c0, cur.ld, b);   // partners' Omega^t rows (BSR)
        bsr(t, cur.Y.p + c0, cur.O.p + c0, cur.ld, b);
      } else {
        Panel dst;
        dst.alloc(H.L(u).rtot, b, st);
        shrink(u, src.Y.p, src.O.p, src.ld, dst.Y.p, dst.O.p, dst.ld, b);
        allgather_skel_rows(u, dst.O.p, dst.ld, b);
        bsr(u - 1, dst.Y.p, dst.O.p, dst.ld, b);
        src = std::move(dst);
      }
    }
  }

  // ================================================================ eager sweep of sketch passes
  //   One tensor-core sketch pass computes up to spec_w stream columns at the cost
  // of one evaluation of K (R27).  Instead of banking the extra columns and replaying every d_blk
  // block later through all committed depths (leaf BSR, shrink + projection and inner BSR, once
  // per block and depth: updateSamples L216-217/L246-247), every column of a pass is swept up
  // with the panel: each BSR / shrink launch of a depth covers the panel's full width dw, and a
  // convergence round that needs the next d_blk samples finds them already in its panel.  The
  // samples CONSUMED are unchanged (the first d columns; the tolerance scale adds each d_blk
  // block's sum of squares when the block is consumed, from per-leaf partials taken right after
  // the sketch), and the arithmetic is column-separable, so the H^2 is bitwise the block-by-block
  // (lazy) result -- H2_EAGER=0 selects the lazy driver (tests compare the two).
  int dw = 0;                                           // columns present in the current panel
  std::vector<std::pair<int, DArr<double>>> blk_part;   // consumption block start -> per-leaf partials

  // consumption blocks: [0, d_init), then d_blk columns each
  int block_end(int b0) const { return b0 == 0 ? std::min(o.d_init, o.d_max) : std::min(b0 + o.d_blk, o.d_max); }
  // width of the pass starting at stream column c0 (a block boundary): whole blocks, as many as
  // one tensor-core pass evaluates K for (spec_w), at least one block
  int pass_width(int c0) const {
    int e = block_end(c0);
    if ((S.kind == H2_S_DENSE_KERNEL || S.kind == H2_S_DENSE_MATRIX) && spec_on)
      while (e < o.d_max && block_end(e) - c0 <= spec_w) e = block_end(e);
    return e - c0;
  }
  // Omega + K_blk(Omega) for stream columns [c0, c0+nc) into (Yd, Od) (pointers at column c0) and
  // the per-leaf sums of squares of every consumption block of the pass (R10)
  void draw_pass(double* Yd, double* Od, int64_t ld, int c0, int nc) {
    timer.begin(H2_PH_RAND);
    if (S.kind == H2_S_DENSE_KERNEL) {
      sketch_cols(Yd, Od, ld, c0, nc);
    } else {
      fill_omega(Od, ld, c0, nc, st);
      timer.end();
      timer.begin(H2_PH_SKETCH);
      sketch_columns += nc;
      if (S.kind == H2_S_DENSE_MATRIX) {
        dense_op_sketch(Od, ld, nc, Yd, st);
      } else if (S.kind == H2_S_H2_LOWRANK) {
        matvec_impl(*S.base, Od, ld, Yd, ld, nc, 1.0, 0.0, st, R, P);
        DArr<double> scr;
        scr.alloc((int64_t)(div_up(T.n, 1024) + 1) * S.rank * nc, st);
        launch_lowrank_sketch(S.U, S.ld_U, S.rank, Od, ld, nc, T.n, Yd, ld, scr.p, st);
      } else {
        callback_sketch(Od, ld, c0, nc, Yd);
      }
    }
    timer.end();
    timer.begin(H2_PH_MISC);
    const int nleaf = 1 << T.Dl;
    for (int b0 = c0; b0 < c0 + nc; b0 = block_end(b0)) {
      const int b1 = block_end(b0);
      DArr<double> part;
      part.alloc(nleaf, st);
      if (ex) launch_exact_sumsq_leaf(Yd + (b0 - c0), T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ld, 0, b1 - b0, part.p, st);
      else launch_sumsq_leaf(Yd + (b0 - c0), T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ld, 0, b1 - b0, part.p, st);
      if (comm) comm_allgather_clusters(comm, part.p, 8, T.Dl, [](int c) { return (int64_t)c; }, st);
      blk_part.emplace_back(b0, std::move(part));
    }
    timer.end();
  }
  // the block starting at column b0 is consumed: ||Y||_F^2 += its sum of squares
  void consume(int b0) {
    for (auto it = blk_part.begin(); it != blk_part.end(); ++it)
      if (it->first == b0) {
        timer.begin(H2_PH_MISC);
        if (ex) launch_exact_sumsq_total(it->second.p, 1 << T.Dl, sumsq_acc.p, nonfinite.p, st);
        else launch_sumsq_total(it->second.p, 1 << T.Dl, sumsq_acc.p, nonfinite.p, st);
        timer.end();
        blk_part.erase(it);
        return;
      }
    throw Error(H2_ERR_INVALID_ARG, "internal: sample block " + std::to_string(b0) + " was never drawn");
  }
  // the next pass (columns [dw, dw + W)) swept up through the committed depths Dl..t+1 and
  // appended to the panel of depth t
  void extend(int t) {
    const int c0 = dw, W = pass_width(dw);
    grow(cur, dw + W, dw);
    if (t == T.Dl) {
      draw_pass(cur.Y.p + c0, cur.O.p + c0, cur.ld, c0, W);
      leaf_subtract(cur.Y.p + c0, cur.O.p + c0, cur.ld, W);
    } else {
      Panel src;
      src.alloc(T.n, W, st);
      draw_pass(src.Y.p, src.O.p, W, c0, W);
      leaf_subtract(src.Y.p, src.O.p, W, W);
      for (int u = T.Dl; u > t; --u) {
        if (u - 1 == t) {
          shrink(u, src.Y.p, src.O.p, src.ld, cur.Y.p + c0, cur.O.p + c0, cur.ld, W);
          allgather_skel_rows(u, cur.O.p + c0, cur.ld, W);
          bsr(t, cur.Y.p + c0, cur.O.p + c0, cur.ld, W);
        } else {
          Panel dst;
          dst.alloc(H.L(u).rtot, W, st);
          shrink(u, src.Y.p, src.O.p, src.ld, dst.Y.p, dst.O.p, dst.ld, W);
          allgather_skel_rows(u, dst.O.p, dst.ld, W);
          bsr(u - 1, dst.Y.p, dst.O.p, dst.ld, W);
          src = std::move(dst);
        }
      }
    }
    dw += W;
  }

  void run_eager() {
    const int Dl = T.Dl;
    d = std::min(o.d_init, o.d_max);
    dw = pass_width(0);
    // line 1: Y = K_blk(Omega) for the first pass into the leaf panel (Y^loc in place)
    cur.alloc(T.n, ld_for(T.n, dw), st);
    draw_pass(cur.Y.p, cur.O.p, cur.ld, 0, dw);
    consume(0);
    tree_ready();                                   // the partition (overlapped with the pass)
    const int top = H.top;
    timer.mark(Dl);
    gen_D();                                        // line 212
    setup_level(Dl);
    leaf_subtract(cur.Y.p, cur.O.p, cur.ld, dw);    // line 213, every column of the pass
    for (int t = Dl; t >= top; --t) {
      if (t < Dl) {
        timer.mark(t);
        setup_level(t);
        bsr(t, cur.Y.p, cur.O.p, cur.ld, dw);       // lines 240-243
      }
      Level& L = H.L(t);
      int rounds = 0;
      double eps = 0;
      while (true) {
        eps = eps_now(t);
        cpqr(t, eps);                               // first d columns
        ++rounds;
        if (!o.adaptive) break;
        bool conv = true;
        const int pos = (o.tol_rule == H2_TOL_RMS) ? o.p_os : 0;
        for (int c = 0; c < L.nclus && conv; ++c) conv = (L.m[c] <= d) || (L.k[c] <= d - 1 - pos);
        if (conv) break;
        if (d + o.d_blk > o.d_max) {
          H.stats.failed_depth = t;
          throw Error(H2_ERR_NOT_CONVERGED, "adaptive sampling reached d_max=" + std::to_string(o.d_max) +
                                                " at depth " + std::to_string(t));
        }
        if (d + o.d_blk > dw) extend(t);            // updateSamples: a new pass, swept up to depth t
        consume(d);
        d += o.d_blk;
      }
      H.stats.rounds[t] = rounds;
      H.stats.eps = eps;
      commit(t);                                    // lines 221-224 / 250-253
      Panel next;
      if (t > top) {                                // lines 222-223 / 251-252, every column
        next.alloc(L.rtot, ld_for(L.rtot, dw), st);
        shrink(t, cur.Y.p, cur.O.p, cur.ld, next.Y.p, next.O.p, next.ld, dw);
      }
      gen_B_with_gather(t, t > top ? &next : nullptr, dw);   // line 258 || Omega^{l+1} all-gather
      cur = std::move(next);
    }
    timer.mark(-1);
    finish(top, Dl);
  }

  // ================================================================ non-symmetric construction
  // h2_build_nonsym ("the extension to the non-symmetric case is straightforward";
  // DESIGN.md R29; oracle/h2_nonsym.py).  Two panels per depth: cur = (Y^l: samples of K Omega,
  // Psi^l: the column stream projected with the ROW bases) in the row layout, curc = (Z^l: samples
  // of K^T Psi, Omega^l projected with the COLUMN bases) in the column layout.  Each side runs the
  // per-level steps of the symmetric build on its own panel (CPQR/ID, shrink + projection); they
  // meet in the BSR subtraction: Y -= B Omega^l (blocks B_{s,b} read directly) and
  // Z -= B^T Psi^l (B_{b,s} read transposed).  D and B are stored for every ORDERED pair in CSR
  // order (D_{s,b} = K(I_s, I_b), B_{s,b} = K(I~_s, J~_b)).
  bool ns = false;
  struct Ordered {
    std::vector<int32_t> os;   // row cluster of CSR entry e
    DArr<int32_t> d_os, d_tpos;   // d_tpos[e]: CSR position of the transposed pair
  };
  Ordered near_o;
  std::vector<Ordered> far_o;
  void ordered_of(const PairCSR& F, int nclus, Ordered& O) {
    const int64_t nnz = F.nnz();
    O.os.assign(nnz, 0);
    std::vector<int32_t> tpos(nnz, 0);
    for (int c = 0; c < nclus; ++c)
      for (int e = F.ptr[c]; e < F.ptr[c + 1]; ++e) O.os[e] = c;
    for (int64_t e = 0; e < nnz; ++e) {
      const int b = F.idx[e], c = O.os[e];
      auto it = std::lower_bound(F.idx.begin() + F.ptr[b], F.idx.begin() + F.ptr[b + 1], c);
      if (it == F.idx.begin() + F.ptr[b + 1] || *it != c) throw Error(H2_ERR_INVALID_ARG, "pair set is not symmetric");
      tpos[e] = (int32_t)(it - F.idx.begin());
    }
    O.d_os.upload(O.os, st);
    O.d_tpos.upload(tpos, st);
  }

  // Omega -> Om (column panel), Psi -> Ps (row panel), Y = K Omega, Z = K^T Psi; ||Y||^2 + ||Z||^2
  void ns_draw(double* Y, double* Ps, int64_t ldr, double* Z, double* Om, int64_t ldc, int c0, int nc) {
    timer.begin(H2_PH_RAND);
    launch_omega(o.seed, o.stream_id, 0, T.n, c0, nc, Om, ldc, st);
    launch_omega(o.seed, o.stream_id + 1, 0, T.n, c0, nc, Ps, ldr, st);
    timer.end();
    timer.begin(H2_PH_SKETCH);
    sketch_columns += nc;
    // under a communicator: this rank's leaf rows of Y and Z (Omega / Psi regenerated for all rows)
    const int64_t r0 = row_b(), r1 = row_e();
    for (int tr = 0; tr < 2; ++tr) {
      const double* in = tr ? Ps : Om;
      const int64_t ldi = tr ? ldr : ldc;
      double* out = tr ? Z : Y;
      const int64_t ldo = tr ? ldc : ldr;
      if (S.kind == H2_S_DENSE_KERNEL) {   // the built-in kernels are symmetric: K^T Psi = K Psi
        launch_dense_sketch(skp, T.d_x, T.d_y, T.d_z, T.n, r0, r1, in, ldi, nc, out + r0 * ldo, ldo, true, st);
        entries_sketch += (r1 - r0) * T.n * (int64_t)div_up(nc, 64);
      } else if (S.kind == H2_S_DENSE_MATRIX) {
        dense_matrix_sketch(S.A, S.ld_A, T.n, r0, r1, in, ldi, nc, out + r0 * ldo, ldo, st, tr == 1);
      } else if (S.kind == H2_S_H2_LOWRANK) {
        // M = A_H + U V^T (A_H symmetric): Y = A_H Omega + U (V^T Omega), Z = A_H Psi + V (U^T Psi);
        // row-sharded matvec of the complete base under a communicator
        matvec_impl(*S.base, in, ldi, out, ldo, nc, 1.0, 0.0, st, R, P);
        if (S.rank > 0) {
          const double* V = S.V ? S.V : S.U;
          const int64_t ldv = S.V ? S.ld_V : S.ld_U;
          DArr<double> scr;
          scr.alloc((int64_t)(div_up(T.n, 1024) + 1) * S.rank * nc, st);
          if (tr == 0) launch_lowrank_sketch(S.U, S.ld_U, S.rank, in, ldi, nc, T.n, out, ldo, scr.p, st, V, ldv);
          else launch_lowrank_sketch(V, ldv, S.rank, in, ldi, nc, T.n, out, ldo, scr.p, st, S.U, S.ld_U);
        }
      } else {
        h2_sketch_req rq{};
        rq.n = T.n;
        rq.row_begin = r0;
        rq.row_end = r1;
        rq.col0 = c0;
        rq.ncols = nc;
        rq.omega = in;
        rq.ld_omega = ldi;
        rq.y = out + r0 * ldo;
        rq.ld_y = ldo;
        rq.stream = st;
        rq.transpose = tr;
        int rc = S.fn(S.ctx, &rq);
        if (rc != 0) throw Error(H2_ERR_CALLBACK, "sketch callback returned " + std::to_string(rc));
      }
    }
    timer.end();
    timer.begin(H2_PH_MISC);
    const int nleaf = 1 << T.Dl;
    if (leaf_part.n < nleaf) leaf_part.alloc(nleaf, st);
    // per-leaf partials of the owned leaves, all-gathered, summed in leaf order (R10)
    launch_sumsq_leaf(Y, T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ldr, 0, nc, leaf_part.p, st);
    if (comm) comm_allgather_clusters(comm, leaf_part.p, 8, T.Dl, [](int c) { return (int64_t)c; }, st);
    launch_sumsq_total(leaf_part.p, nleaf, sumsq_acc.p, nonfinite.p, st);
    launch_sumsq_leaf(Z, T.d_leaf_begin, cb(T.Dl), ce(T.Dl), ldc, 0, nc, leaf_part.p, st);
    if (comm) comm_allgather_clusters(comm, leaf_part.p, 8, T.Dl, [](int c) { return (int64_t)c; }, st);
    launch_sumsq_total(leaf_part.p, nleaf, sumsq_acc.p, nonfinite.p, st);
    timer.end();
  }

  // side sd (0: rows, 1: columns) of the BSR subtraction on a panel of depth t
  void ns_bsr(int t, int sd, double* Yp, int64_t ldy, const double* Op, int64_t ldo, int nc) {
    timer.begin(H2_PH_BSR);
    BsrArgs a{};
    a.c0 = 0;
    a.ncols = nc;
    a.tmode = sd ? 2 : 1;
    a.c_begin = cb(t == T.Dl ? T.Dl : t + 1);   // owned row clusters (all on one GPU)
    a.nclusters = ce(t == T.Dl ? T.Dl : t + 1) - a.c_begin;
    if (t == T.Dl) {
      a.max_rows = H.L(T.Dl).max_m;
      a.yoff = a.ooff = T.d_leaf_begin;
      a.cnt = T.d_leaf_size;
      a.ptr = T.d_near.ptr;
      a.idx = T.d_near.idx;
      a.uidx = sd ? near_o.d_tpos.p : nullptr;
      a.blk_off = H.d_D_off.p;
      a.blk = H.D.p;
    } else {
      const Level& Ls = H.S(sd, t + 1);
      const Level& Lo = H.S(1 - sd, t + 1);
      a.max_rows = Ls.max_k;
      a.yoff = Ls.d_roff.p;
      a.ooff = Lo.d_roff.p;
      a.cnt = Ls.d_k.p;
      a.kcnt = Lo.d_k.p;
      a.ptr = T.d_far[t + 1].ptr;
      a.idx = T.d_far[t + 1].idx;
      a.uidx = sd ? far_o[t + 1].d_tpos.p : nullptr;
      a.blk_off = H.L(t + 1).d_B_off.p;
      a.blk = H.L(t + 1).B.p;
    }
    a.Y = Yp;
    a.ldy = ldy;
    a.Om = Op;
    a.ldo = ldo;
    launch_bsr(a, st);
    timer.end();
  }

  void ns_gen_D() {
    const PairCSR& F = T.near;
    H.D_off.assign(F.nnz() + 1, 0);
    for (int64_t e = 0; e < F.nnz(); ++e)
      H.D_off[e + 1] = H.D_off[e] + (T.end[T.Dl][near_o.os[e]] - T.begin[T.Dl][near_o.os[e]]) *
                                        (T.end[T.Dl][F.idx[e]] - T.begin[T.Dl][F.idx[e]]);
    H.d_D_off.upload(H.D_off, st);
    H.D.alloc(H.D_off.back(), st);
    GenArgs g{};
    g.nblocks = F.nnz();
    DArr<int32_t> ul;
    if (comm) {
      ul.upload(owned_ordered(F, near_o.os, T.Dl), st);
      g.ulist = ul.p;
      g.nblocks = ul.n;
    }
    g.us = near_o.d_os.p;
    g.ub = T.d_near.idx;
    g.cnt = T.d_leaf_size;
    g.off = T.d_leaf_begin;
    g.idx = T.d_iota;
    g.out_off = H.d_D_off.p;
    g.out = H.D.p;
    if (E.kind == H2_E_H2_LOWRANK) {   // D_A (unique, transposed for s > b) + U(I_s) V(I_b)^T
      timer.begin(H2_PH_GEN);
      UpdateNsArgs a{};
      a.nblocks = g.nblocks;
      a.ulist = g.ulist;
      a.os = near_o.d_os.p;
      a.ob = T.d_near.idx;
      a.uidx = T.d_near.uidx;
      a.us = T.d_near.us;
      a.Bbase = E.base->D.p;
      a.Boff = T.d_D_off;
      a.out = H.D.p;
      a.out_off = H.d_D_off.p;
      a.cnt = T.d_leaf_size;
      a.begin = T.d_leaf_begin;
      a.U = E.U;
      a.ldu = E.ld_U;
      a.V = E.V ? E.V : E.U;
      a.ldv = E.V ? E.ld_V : E.ld_U;
      a.r = E.rank;
      launch_update_ns(a, false, (int)std::min<int64_t>(std::max<int64_t>(a.nblocks, 1), 148 * 8), st);
      timer.end();
      return;
    }
    gen(g);
  }

  void ns_gen_B(int t) {
    Level& L = H.L(t);
    const Level& C = H.C(t);
    const PairCSR& F = T.far[t];
    L.B_off.assign(F.nnz() + 1, 0);
    for (int64_t e = 0; e < F.nnz(); ++e)
      L.B_off[e + 1] = L.B_off[e] + (int64_t)L.k[far_o[t].os[e]] * C.k[F.idx[e]];
    L.d_B_off.upload(L.B_off, st);
    L.B.alloc(L.B_off.back(), st);
    GenArgs g{};
    g.nblocks = F.nnz();
    DArr<int32_t> ul;
    if (comm) {
      ul.upload(owned_ordered(F, far_o[t].os, t), st);
      g.ulist = ul.p;
      g.nblocks = ul.n;
    }
    g.us = far_o[t].d_os.p;
    g.ub = T.d_far[t].idx;
    g.cnt = L.d_k.p;
    g.off = L.d_roff.p;
    g.idx = L.d_skel.p;
    g.cnt2 = C.d_k.p;
    g.off2 = C.d_roff.p;
    g.idx2 = C.d_skel.p;
    g.out_off = L.d_B_off.p;
    g.out = L.B.p;
    if (E.kind == H2_E_H2_LOWRANK) {
      if (F.nnz() == 0) return;
      timer.begin(H2_PH_GEN);
      const Level& La = E.base->L(t);
      std::vector<int64_t> ro_r, ro_c;
      DArr<int64_t> d_ro_r, d_ro_c;
      DArr<double> Rr, Rc;
      expand_base_rows(t, L, Rr, ro_r, d_ro_r);   // base rows at the row skeletons I~
      expand_base_rows(t, C, Rc, ro_c, d_ro_c);   // and at the column skeletons J~
      int64_t gmax = 1;
      for (int64_t e = 0; e < F.nnz(); ++e)
        gmax = std::max<int64_t>(gmax, (int64_t)La.k[far_o[t].os[e]] * C.k[F.idx[e]]);
      const int grid = (int)std::min<int64_t>(std::max<int64_t>(g.nblocks, 1), 148 * 4);
      DArr<double> scratch;
      scratch.alloc(gmax * grid, st);
      UpdateNsArgs a{};
      a.nblocks = g.nblocks;
      a.ulist = g.ulist;
      a.os = far_o[t].d_os.p;
      a.ob = T.d_far[t].idx;
      a.uidx = T.d_far[t].uidx;
      a.us = T.d_far[t].us;
      a.Bbase = La.B.p;
      a.Boff = La.d_B_off.p;
      a.out = L.B.p;
      a.out_off = L.d_B_off.p;
      a.cnt = L.d_k.p;
      a.cnt2 = C.d_k.p;
      a.kb = La.d_k.p;
      a.U = E.U;
      a.ldu = E.ld_U;
      a.V = E.V ? E.V : E.U;
      a.ldv = E.V ? E.ld_V : E.ld_U;
      a.r = E.rank;
      a.R = Rr.p;
      a.R2 = Rc.p;
      a.rowoff = d_ro_r.p;
      a.rowoff2 = d_ro_c.p;
      a.skel = L.d_skel.p;
      a.skel2 = C.d_skel.p;
      a.roff = L.d_roff.p;
      a.roff2 = C.d_roff.p;
      a.scratch = scratch.p;
      a.gmax = gmax;
      launch_update_ns(a, true, grid, st);
      timer.end();
      return;
    }
    gen(g);
  }

  void ns_bsr_both(int t, Panel& R, Panel& Cp, int c0, int nc) {
    ns_bsr(t, 0, R.Y.p + c0, R.ld, Cp.O.p + c0, Cp.ld, nc);
    ns_bsr(t, 1, Cp.Y.p + c0, Cp.ld, R.O.p + c0, R.ld, nc);
  }

  // updateSamples for both sides: b new columns of Omega and Psi swept up to depth t
  void ns_update_samples(int t, int b) {
    const int c0 = d;
    grow(cur, d + b);
    grow(curc, d + b);
    if (t == T.Dl) {
      ns_draw(cur.Y.p + c0, cur.O.p + c0, cur.ld, curc.Y.p + c0, curc.O.p + c0, curc.ld, c0, b);
      ns_bsr_both(T.Dl, cur, curc, c0, b);
      return;
    }
    Panel sr, sc;
    sr.alloc(T.n, b, st);
    sc.alloc(T.n, b, st);
    ns_draw(sr.Y.p, sr.O.p, sr.ld, sc.Y.p, sc.O.p, sc.ld, c0, b);
    ns_bsr_both(T.Dl, sr, sc, 0, b);
    for (int u = T.Dl; u > t; --u) {
      if (u - 1 == t) {
        shrink(u, sr.Y.p, sr.O.p, sr.ld, cur.Y.p + c0, cur.O.p + c0, cur.ld, b, 0);
        shrink(u, sc.Y.p, sc.O.p, sc.ld, curc.Y.p + c0, curc.O.p + c0, curc.ld, b, 1);
        allgather_skel_rows(u, cur.O.p + c0, cur.ld, b, nullptr, 0);
        allgather_skel_rows(u, curc.O.p + c0, curc.ld, b, nullptr, 1);
        ns_bsr_both(t, cur, curc, c0, b);
      } else {
        Panel dr, dc;
        dr.alloc(H.L(u).rtot, b, st);
        dc.alloc(H.C(u).rtot, b, st);
        shrink(u, sr.Y.p, sr.O.p, sr.ld, dr.Y.p, dr.O.p, dr.ld, b, 0);
        shrink(u, sc.Y.p, sc.O.p, sc.ld, dc.Y.p, dc.O.p, dc.ld, b, 1);
        allgather_skel_rows(u, dr.O.p, dr.ld, b, nullptr, 0);
        allgather_skel_rows(u, dc.O.p, dc.ld, b, nullptr, 1);
        ns_bsr_both(u - 1, dr, dc, 0, b);
        sr = std::move(dr);
        sc = std::move(dc);
      }
    }
  }

  void run_nonsym() {
    ns = true;
    user_st = st;
    st = prio_stream(true);
    timer.st = st;
    stream_after(st, user_st);
    const int Dl = T.Dl;
    const int top = T.top < 0 ? Dl : T.top;
    H.nonsym = true;
    H.top = top;
    H.Dl = Dl;
    H.n = T.n;
    H.lv.resize(Dl - top + 1);
    H.lvc.resize(Dl - top + 1);
    if (S.kind == H2_S_DENSE_KERNEL) skp = tree_kernel(&T, S.kern, st);
    if (E.kind == H2_E_BUILTIN) ekp = make_kernel(E.kern);
    d = std::min(o.d_init, o.d_max);
    sumsq_acc.alloc(1, st);
    nonfinite.alloc(1, st);
    H2_CUDA(cudaMemsetAsync(sumsq_acc.p, 0, sizeof(double), st));
    H2_CUDA(cudaMemsetAsync(nonfinite.p, 0, sizeof(int), st));
    ordered_of(T.near, 1 << Dl, near_o);
    far_o.resize(Dl + 1);
    for (int t = top; t <= Dl; ++t) ordered_of(T.far[t], 1 << t, far_o[t]);

    cur.alloc(T.n, ld_for(T.n, d), st);
    curc.alloc(T.n, ld_for(T.n, d), st);
    ns_draw(cur.Y.p, cur.O.p, cur.ld, curc.Y.p, curc.O.p, curc.ld, 0, d);   // line 1, both sketches
    timer.mark(Dl);
    ns_gen_D();                                                            // line 212, ordered pairs
    setup_level(Dl, 0);
    setup_level(Dl, 1);
    ns_bsr_both(Dl, cur, curc, 0, d);                                      // line 213
    for (int t = Dl; t >= top; --t) {
      if (t < Dl) {
        timer.mark(t);
        setup_level(t, 0);
        setup_level(t, 1);
        ns_bsr_both(t, cur, curc, 0, d);                                   // lines 240-243
      }
      Level& L = H.L(t);
      Level& C = H.C(t);
      int rounds = 0;
      double eps = 0;
      while (true) {
        eps = eps_now(t);
        cpqr(t, eps, 0);
        cpqr(t, eps, 1);
        ++rounds;
        if (!o.adaptive) break;
        bool conv = true;
        const int pos = (o.tol_rule == H2_TOL_RMS) ? o.p_os : 0;
        for (int c = 0; c < L.nclus && conv; ++c)
          conv = (L.m[c] <= d || L.k[c] <= d - 1 - pos) && (C.m[c] <= d || C.k[c] <= d - 1 - pos);
        if (conv) break;
        if (d + o.d_blk > o.d_max) {
          H.stats.failed_depth = t;
          throw Error(H2_ERR_NOT_CONVERGED, "adaptive sampling reached d_max=" + std::to_string(o.d_max) +
                                                " at depth " + std::to_string(t));
        }
        ns_update_samples(t, o.d_blk);
        d += o.d_blk;
      }
      H.stats.rounds[t] = rounds;
      H.stats.eps = eps;
      commit(t, 0);
      commit(t, 1);
      Panel nr, nc;
      if (t > top) {
        nr.alloc(L.rtot, ld_for(L.rtot, d), st);
        nc.alloc(C.rtot, ld_for(C.rtot, d), st);
        shrink(t, cur.Y.p, cur.O.p, cur.ld, nr.Y.p, nr.O.p, nr.ld, d, 0);
        shrink(t, curc.Y.p, curc.O.p, curc.ld, nc.Y.p, nc.O.p, nc.ld, d, 1);
        // the other side's BSR partners' projected samples (S§8(e); halo or all-gather)
        allgather_skel_rows(t, nr.O.p, nr.ld, d, nullptr, 0);
        allgather_skel_rows(t, nc.O.p, nc.ld, d, nullptr, 1);
      }
      ns_gen_B(t);                                                         // line 258, ordered pairs
      cur = std::move(nr);
      curc = std::move(nc);
    }
    timer.mark(-1);
    finish(top, Dl);
  }

  ~Builder() {
    // an exception may leave work queued on the internal streams: drain them before the
    // members (allocated on them) are released
    if (user_st) {
      cudaStreamSynchronize(prio_stream(false));
      cudaStreamSynchronize(st);
      if (pre_live) cudaEventDestroy(pre_done);
    }
  }

  // the block partition is needed from here on (an asynchronous tree: wait for its host thread
  // and upload the CSR descriptors), and the level structure of H follows from its top depth
  bool tree_ready_done = false;
  void tree_ready() {
    if (tree_ready_done) return;
    tree_ready_done = true;
    ensure_partition_uploaded(&T);
    const int Dl = T.Dl;
    const int top = T.top < 0 ? Dl : T.top;
    H.top = top;
    H.Dl = Dl;
    H.n = T.n;
    H.lv.resize(Dl - top + 1);
  }

  void run() {
    // internal high-priority stream, ordered after the caller's stream
    user_st = st;
    st = prio_stream(true);
    timer.st = st;
    stream_after(st, user_st);
    const int Dl = T.Dl;
    ex = o.exact_order != 0;
    // the first tensor-core sketch pass needs only the ordering: with an asynchronous tree it is
    // launched before the partition is waited for (run_eager), so the host's dual traversal and
    // CSR construction overlap the O(N^2) pass on the GPU
    const bool lazy = env_int("H2_EAGER", 1) != 0 && S.kind == H2_S_DENSE_KERNEL && S.kern.kind == H2_K_EXP &&
                      !comm && o.tol_rule == H2_TOL_RMS && !o.exact_order;
    if (!lazy) tree_ready();
    if (S.kind == H2_S_DENSE_KERNEL) {
      skp = tree_kernel(&T, S.kern, st);
      spec_on = !ex && quarters() && sketch_tc_supported(skp) && env_int("H2_SK_TC", 1) != 0 &&
                env_int("H2_SPEC", 1) != 0;
      spec_w = sketch_tc_pass_cols(skp.kind);
    }
    if (S.kind == H2_S_DENSE_MATRIX) {   // tensor-core operator product: passes of 128 columns
      dense_tc = !ex && quarters() && env_int("H2_DENSE_TC", 1) != 0;
      spec_on = dense_tc && env_int("H2_SPEC", 1) != 0;
      spec_w = 128;
    }
    if (o.tol_rule == H2_TOL_LITERAL && !(o.norm > 0)) o.norm = estimate_norm();
    if (o.tol_rule == H2_TOL_LITERAL) H.stats.norm_est = o.norm;
    if (E.kind == H2_E_BUILTIN) ekp = make_kernel(E.kern);
    sumsq_acc.alloc(1, st);
    nonfinite.alloc(1, st);
    H2_CUDA(cudaMemsetAsync(sumsq_acc.p, 0, sizeof(double), st));
    H2_CUDA(cudaMemsetAsync(nonfinite.p, 0, sizeof(int), st));
    if (env_int("H2_EAGER", 1) != 0) {   // DESIGN.md §5b; H2_EAGER=0: block-by-block replays
      run_eager();
      return;
    }
    d = std::min(o.d_init, o.d_max);

    // line 1: Y = K_blk(Omega) into the leaf panel (leaf Y^loc is computed in place)
    cur.alloc(T.n, ld_for(T.n, d), st);
    draw(cur.Y.p, cur.O.p, cur.ld, 0, d);
    // line 212: D_{tau,b} = K(I_tau, I_b), one unique block per unordered pair
    timer.mark(Dl);
    gen_D();
    setup_level(Dl);
    leaf_subtract(cur.Y.p, cur.O.p, cur.ld, d);   // line 213
    run_levels(H.top, Dl);
  }

  void gen_D() {
    H.D.alloc(T.D_off.back(), st);
    {
      GenArgs g{};
      g.nblocks = T.near.nuniq();
      DArr<int32_t> ul;
      if (comm) {
        const std::vector<int32_t> l = owned_pairs(T.near, T.Dl);
        ul.upload(l, st);
        g.ulist = ul.p;
        g.nblocks = (int64_t)l.size();
      }
      g.us = T.d_near.us;
      g.ub = T.d_near.ub;
      g.cnt = T.d_leaf_size;
      g.off = T.d_leaf_begin;
      g.idx = T.d_iota;
      g.out_off = T.d_D_off;
      g.out = H.D.p;
      if (E.kind == H2_E_H2_LOWRANK) {
        timer.begin(H2_PH_GEN);
        UpdateDArgs a{};
        a.nblocks = g.nblocks;
        a.ulist = g.ulist;
        a.us = g.us;
        a.ub = g.ub;
        a.cnt = T.d_leaf_size;
        a.begin = T.d_leaf_begin;
        a.off = T.d_D_off;
        a.Dbase = E.base->D.p;
        a.out = H.D.p;
        a.U = E.U;
        a.ldu = E.ld_U;
        a.r = E.rank;
        launch_update_D(a, st);
        timer.end();
      } else {
        gen(g);
      }
    }
  }

  void run_levels(int top, int Dl) {
    for (int t = Dl; t >= top; --t) {
      if (t < Dl) {
        timer.mark(t);
        setup_level(t);
        bsr(t, cur.Y.p, cur.O.p, cur.ld, d);   // lines 240-243
      }
      Level& L = H.L(t);
      int rounds = 0;
      double eps = 0;
      while (true) {
        eps = eps_now(t);
        cpqr(t, eps);
        ++rounds;
        if (!o.adaptive) break;
        bool conv = true;
        const int pos = (o.tol_rule == H2_TOL_RMS) ? o.p_os : 0;
        for (int c = 0; c < L.nclus && conv; ++c) conv = (L.m[c] <= d) || (L.k[c] <= d - 1 - pos);
        if (conv) break;
        if (d + o.d_blk > o.d_max) {
          H.stats.failed_depth = t;
          throw Error(H2_ERR_NOT_CONVERGED, "adaptive sampling reached d_max=" + std::to_string(o.d_max) +
                                                " at depth " + std::to_string(t));
        }
        update_samples(t, o.d_blk);
        d += o.d_blk;
      }
      H.stats.rounds[t] = rounds;
      H.stats.eps = eps;
      commit(t);                                    // lines 221-224 / 250-253
      Panel next;
      if (t > top) {                                // lines 222-223 / 251-252 into the parent panel
        next.alloc(L.rtot, ld_for(L.rtot, d), st);
        shrink(t, cur.Y.p, cur.O.p, cur.ld, next.Y.p, next.O.p, next.ld, d);
      }
      gen_B_with_gather(t, t > top ? &next : nullptr, d);    // line 258 || Omega^{l+1} all-gather
      cur = std::move(next);
    }
    timer.mark(-1);
    finish(top, Dl);
  }

  // wait for the build, hand the level arrays to the matrix, fill the statistics
  void finish(int top, int Dl) {
    join_prefetch();   // an unused speculative pass is waited for (at most one pass)
    H2_CUDA(cudaStreamSynchronize(st));
    stream_after(user_st, st);
    cur.release();
    curc.release();
    W.release();
    Wc.release();
    for (auto* lvs : {&H.lv, &H.lvc})
      for (auto& L : *lvs) {
        for (auto* a : {&L.d_m, &L.d_k, &L.d_perm, &L.d_skel}) a->detach();
        for (auto* a : {&L.d_poff, &L.d_roff, &L.d_xoff, &L.d_B_off}) a->detach();
        for (auto* a : {&L.X, &L.cert, &L.B}) a->detach();
      }
    H.D.detach();
    H.d_D_off.detach();
    // stats
    h2_build_stats& s = H.stats;
    s.samples = d;
    s.top_depth = top;
    s.leaf_depth = Dl;
    s.entries_D = ns ? H.D_off.back() : T.D_off.back();
    s.entries_sketch = entries_sketch;
    s.sketch_columns = sketch_columns;
    s.bytes_D = H.D.bytes();
    for (int t = top; t <= Dl; ++t) {
      const Level& L = H.L(t);
      int mn = INT32_MAX, mx = 0;
      double sum = 0;
      for (int c = 0; c < L.nclus; ++c) {
        mn = std::min(mn, L.k[c]);
        mx = std::max(mx, L.k[c]);
        sum += L.k[c];
      }
      s.rank_min[t] = mn;
      s.rank_max[t] = mx;
      s.rank_mean[t] = sum / L.nclus;
      s.entries_B += L.B_off.back();
      s.bytes_B += L.B.bytes();
      if (t == Dl) s.bytes_U += L.X.bytes();
      else s.bytes_E += L.X.bytes();
      if (ns) {
        if (t == Dl) s.bytes_U += H.C(t).X.bytes();
        else s.bytes_E += H.C(t).X.bytes();
      }
    }
    timer.collect(s.t_phase_ms);
    timer.collect_depths(s.t_depth_ms);
    wb[H2_PH_GEN] = 8.0 * (double)(s.entries_D + s.entries_B);
    wb[H2_PH_RAND] = 8.0 * (double)sketch_columns * (double)(row_e() - row_b());
    for (int p = 0; p < H2_NPHASE; ++p) {
      s.work_flops[p] = wf[p];
      s.work_bytes[p] = wb[p];
    }
    if (getenv("H2_TRACE")) {
      fprintf(stderr, "[h2 trace] host ms per phase:");
      for (int p = 0; p < H2_NPHASE; ++p) fprintf(stderr, " %.1f", timer.host_ms[p]);
      fprintf(stderr, " | alloc %.1f ms, cudaMalloc %lld (%.2f GB), cudaFree %lld\n", g_alloc_ms,
              (long long)h2::g_cache_mallocs.exchange(0), h2::g_cache_malloc_bytes.exchange(0) / 1e9,
              (long long)h2::g_cache_frees.exchange(0));
    }
  }
};

// y = alpha K_H x + beta y (CS4: upward pass, couplings, downward pass, dense leaves); stream-ordered,
// workspaces released stream-ordered on return
// Row-sharded form (rank, nranks > 1; S§8(e) "Config 5's H^2 sketch is a distributed h2_matvec"):
// the matrix is complete on every rank and x is replicated (the Omega stream is regenerated on
// every rank); the upward pass runs over all clusters (O(N q), the cheap part), the couplings,
// the downward pass and the dense leaves only over the rank's owned clusters (subtree-aligned
// ranges own_begin), so y is computed for the rank's leaf rows only -- no communication, and
// each owned row's arithmetic is the one-GPU arithmetic (bitwise).
void matvec_impl(const h2_matrix& Hm, const double* x, int64_t ldx, double* y, int64_t ldy, int32_t q, double alpha,
                 double beta, cudaStream_t st, int rank, int nranks) {
  const h2_matrix* H = &Hm;
    const h2_tree& T = *H->tree;
  const int Dl = H->Dl, top = H->top;
  auto ob = [&](int t) { return nranks > 1 ? own_begin(t, rank, nranks) : 0; };
  auto oe = [&](int t) { return nranks > 1 ? own_begin(t, rank + 1, nranks) : (1 << t); };
  // non-symmetric: the upward pass uses the column side (V, F), the downward pass the row side
  const int up = H->nonsym ? 1 : 0;
  std::vector<DArr<double>> xh(Dl + 1), yh(Dl + 1);
  for (int t = top; t <= Dl; ++t) {
    const Level& L = H->L(t);
    xh[t].alloc(std::max<int64_t>(H->S(up, t).rtot, 1) * q, st);
    yh[t].alloc(std::max<int64_t>(L.rtot, 1) * q, st);
    H2_CUDA(cudaMemsetAsync(yh[t].p, 0, sizeof(double) * std::max<int64_t>(L.rtot, 1) * q, st));
  }
  if (beta != 1.0) launch_scale(y, T.n, ldy, q, beta, st);
  // upward pass
  for (int t = Dl; t >= top; --t) {
    const Level& L = H->S(up, t);
    UpArgs a{};
    a.nclusters = L.nclus;
    a.ioff = (t == Dl) ? T.d_leaf_begin : L.d_poff.p;
    a.m = L.d_m.p;
    a.k = L.d_k.p;
    a.xoff = L.d_xoff.p;
    a.X = L.X.p;
    a.roff = L.d_roff.p;
    a.xin = (t == Dl) ? x : xh[t + 1].p;
    a.ldi = (t == Dl) ? ldx : q;
    a.xh = xh[t].p;
    a.ldh = q;
    a.q = q;
    a.max_out = L.max_k;
    launch_upward(a, st);
  }
  // couplings  y^_s += sum_{b in F_s} B_{s,b} x^_b
  for (int t = top; t <= Dl; ++t) {
    const Level& L = H->L(t);
    if (T.far[t].nnz() == 0) continue;
    SpmmArgs s{};
    s.c_begin = ob(t);
    s.nclusters = oe(t) - ob(t);
    s.max_rows = L.max_k;
    s.yoff = s.xoff = L.d_roff.p;
    s.cnt = L.d_k.p;
    s.ptr = T.d_far[t].ptr;
    s.idx = T.d_far[t].idx;
    s.uidx = T.d_far[t].uidx;
    s.us = T.d_far[t].us;
    s.blk_off = L.d_B_off.p;
    s.blk = L.B.p;
    if (H->nonsym) {   // ordered B_{s,b} (k_s x kc_b), read directly
      s.xoff = H->C(t).d_roff.p;
      s.kcnt = H->C(t).d_k.p;
      s.uidx = nullptr;
      s.tmode = 1;
    }
    s.x = xh[t].p;
    s.ldx = q;
    s.y = yh[t].p;
    s.ldy = q;
    s.q = q;
    s.alpha = 1.0;
    launch_spmm(s, st);
  }
  // downward pass
  for (int t = top; t <= Dl; ++t) {
    const Level& L = H->L(t);
    DownArgs a{};
    a.c_begin = ob(t);
    a.nclusters = oe(t) - ob(t);
    a.ioff = (t == Dl) ? T.d_leaf_begin : L.d_poff.p;
    a.m = L.d_m.p;
    a.k = L.d_k.p;
    a.xoff = L.d_xoff.p;
    a.X = L.X.p;
    a.roff = L.d_roff.p;
    a.yh = yh[t].p;
    a.ldh = q;
    a.yout = (t == Dl) ? y : yh[t + 1].p;
    a.ldo = (t == Dl) ? ldy : q;
    a.q = q;
    a.alpha = (t == Dl) ? alpha : 1.0;
    a.accumulate = 1;
    a.max_out = L.max_m;
    launch_downward(a, st);
  }
  // dense leaves  y += alpha sum_{b in N} D x
  {
    SpmmArgs s{};
    s.c_begin = ob(Dl);
    s.nclusters = oe(Dl) - ob(Dl);
    s.max_rows = H->L(Dl).max_m;
    s.yoff = s.xoff = T.d_leaf_begin;
    s.cnt = T.d_leaf_size;
    s.ptr = T.d_near.ptr;
    s.idx = T.d_near.idx;
    s.uidx = T.d_near.uidx;
    s.us = T.d_near.us;
    s.blk_off = T.d_D_off;
    s.blk = H->D.p;
    if (H->nonsym) {
      s.blk_off = H->d_D_off.p;
      s.uidx = nullptr;
      s.tmode = 1;
    }
    s.x = x;
    s.ldx = ldx;
    s.y = y;
    s.ldy = ldy;
    s.q = q;
    s.alpha = alpha;
    launch_spmm(s, st);
  }
}

// the tree is built on the host; its device mirror is created on first use (current device)
// device mirrors of the tree: the ordering part (coordinates, leaf ranges) and, after waiting
// for an asynchronous partition (h2_tree_build_async), the CSR batch descriptors
void ensure_order_uploaded(const h2_tree* tree) {
  h2_tree* T = const_cast<h2_tree*>(tree);
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  if (T->device < 0) tree_upload_order(*T);
  H2_REQUIRE(dev == T->device, "libh2: the tree was uploaded to another device");
}
void ensure_partition_uploaded(const h2_tree* tree) {
  h2_tree* T = const_cast<h2_tree*>(tree);
  T->wait_partition();
  if (!T->part_uploaded) tree_upload_partition(*T);
}
void ensure_uploaded(const h2_tree* tree) {
  ensure_order_uploaded(tree);
  ensure_partition_uploaded(tree);
}

// per-leaf near-field chunk lists for launch_near_sketch_tc (built once per tree, on the tree's
// device): eligible when every leaf holds exactly 64 points at a multiple of 64 (row tiles =
// leaves); leaf s lists the 128-j chunks b / 2 of its near leaves b (ascending) with the mask of
// the 64-j halves (bit b & 1) that are near leaves
bool ensure_near_chunks(const h2_tree* tree) {
  h2_tree& T = *const_cast<h2_tree*>(tree);
  if (T.nl_state != 0) return T.nl_state > 0;
  const int Dl = T.Dl;
  const int nleaf = 1 << Dl;
  bool ok = T.n == ((int64_t)64 << Dl);
  for (int c = 0; c < nleaf && ok; ++c) ok = T.begin[Dl][c] == 64 * (int64_t)c && T.end[Dl][c] == 64 * (int64_t)c + 64;
  if (!ok) {
    T.nl_state = -1;
    return false;
  }
  std::vector<int32_t> ptr(nleaf + 1, 0), chunk;
  std::vector<uint8_t> mask;
  for (int c = 0; c < nleaf; ++c) {
    ptr[c] = (int32_t)chunk.size();
    for (int e = T.near.ptr[c]; e < T.near.ptr[c + 1]; ++e) {   // partners ascending
      const int b = T.near.idx[e];
      if (chunk.size() > (size_t)ptr[c] && chunk.back() == b / 2) mask.back() |= (uint8_t)(1u << (b & 1));
      else {
        chunk.push_back(b / 2);
        mask.push_back((uint8_t)(1u << (b & 1)));
      }
    }
  }
  ptr[nleaf] = (int32_t)chunk.size();
  auto up = [](const void* src, size_t bytes) {   // block cache, as every tree array (tree.cpp)
    void* p = h2::cache_alloc(std::max<size_t>(bytes, 4), nullptr);
    if (bytes) H2_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
    return p;
  };
  T.d_nl_ptr = static_cast<int32_t*>(up(ptr.data(), ptr.size() * 4));
  T.d_nl_chunk = static_cast<int32_t*>(up(chunk.data(), chunk.size() * 4));
  T.d_nl_mask = static_cast<uint8_t*>(up(mask.data(), mask.size()));
  T.nl_state = 1;
  return true;
}

// built-in kernel parameters on a tree: diameter (exp / Helmholtz range guards) and, for the
// Helmholtz tensor-core sketch, the minimum point distance (computed once per tree)
KernelParams tree_kernel(const h2_tree* tree, const h2_kernel& k, cudaStream_t st) {
  h2_tree* T = const_cast<h2_tree*>(tree);
  if (k.kind == H2_K_HELMHOLTZ && T->rmin < 0) {
    const double d2 = min_near_dist2(T->d_x, T->d_y, T->d_z, T->d_leaf_begin, 1 << T->Dl, T->d_near.ptr,
                                     T->d_near.idx, st);
    T->rmin = (d2 > 0 && d2 < 1e300) ? std::sqrt(d2) : 0.0;
  }
  return make_kernel(k, T->diam, k.kind == H2_K_HELMHOLTZ ? T->rmin : 0.0);
}

h2_status fail(const Error& e) {
  g_err = e.what();
  return e.status;
}

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

const char* h2_last_error(void) { return g_err.c_str(); }
const char* h2_version(void) { return "libh2 0.1 (sm_100a)"; }

h2_status h2_tree_build(const double* coords_host, int64_t n, int32_t dim, int32_t leaf_size, double eta,
                        int32_t dist_rule, h2_tree** out) {
  if (!out) return (g_err = "h2_tree_build: out is NULL", H2_ERR_INVALID_ARG);
  *out = nullptr;
  try {
    H2_REQUIRE(coords_host != nullptr, "h2_tree_build: coords is NULL");
    auto* T = new h2_tree();
    std::unique_ptr<h2_tree> guard(T);
    tree_build_host(*T, coords_host, n, dim, leaf_size, eta, dist_rule);   // device upload is lazy
    *out = guard.release();
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    g_err = "h2_tree_build: host out of memory";
    return H2_ERR_OOM;
  }
}

h2_status h2_tree_build_async(const double* coords_host, int64_t n, int32_t dim, int32_t leaf_size, double eta,
                              int32_t dist_rule, h2_tree** out) {
  if (!out) return (g_err = "h2_tree_build_async: out is NULL", H2_ERR_INVALID_ARG);
  *out = nullptr;
  try {
    H2_REQUIRE(coords_host != nullptr, "h2_tree_build_async: coords is NULL");
    auto* T = new h2_tree();
    std::unique_ptr<h2_tree> guard(T);
    // the KD ordering on the GPU when one is present (kd_gpu.cu: the same tree, ~17 -> ~3 ms of
    // host prefix at N = 2^18; H2_KD_GPU=0: the host ordering)
    int ndev = 0;
    const bool gpu = n >= 4096 && env_int("H2_KD_GPU", 1) != 0 && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
    cudaGetLastError();
    if (gpu) tree_build_order_gpu(*T, coords_host, n, dim, leaf_size, eta, dist_rule);
    else tree_build_order(*T, coords_host, n, dim, leaf_size, eta, dist_rule);
    T->part_thread = std::thread([T] {
      try {
        tree_download_order(*T);
        tree_build_partition(*T);
      } catch (const Error& e) {
        T->part_error = e.what();
      } catch (const std::exception& e) {
        T->part_error = std::string("h2_tree_build_async: ") + e.what();
      }
    });
    *out = guard.release();
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    g_err = "h2_tree_build_async: host out of memory";
    return H2_ERR_OOM;
  }
}

h2_status h2_tree_import(const h2_tree_desc* desc, h2_tree** out) {
  if (!out) return (g_err = "h2_tree_import: out is NULL", H2_ERR_INVALID_ARG);
  *out = nullptr;
  try {
    H2_REQUIRE(desc != nullptr, "h2_tree_import: desc is NULL");
    auto* T = new h2_tree();
    std::unique_ptr<h2_tree> guard(T);
    tree_import_host(*T, *desc);
    *out = guard.release();
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    g_err = "h2_tree_import: host out of memory";
    return H2_ERR_OOM;
  }
}

h2_status h2_tree_get_info(const h2_tree* T, h2_tree_info* info) {
  if (!T || !info) return (g_err = "h2_tree_get_info: NULL argument", H2_ERR_INVALID_ARG);
  try {
    const_cast<h2_tree*>(T)->wait_partition();
  } catch (const Error& e) {
    return fail(e);
  }
  info->n = T->n;
  info->dim = T->dim;
  info->leaf_size = T->leaf_size;
  info->leaf_depth = T->Dl;
  info->top_depth = T->top;
  info->near_nnz = T->near.nnz();
  info->far_nnz_total = 0;
  for (auto& f : T->far) info->far_nnz_total += f.nnz();
  info->csp = T->csp;
  return H2_OK;
}

h2_status h2_tree_export(const h2_tree* T, int64_t* perm, int64_t* begin, int64_t* end, int32_t* near_pairs) {
  if (!T) return (g_err = "h2_tree_export: NULL tree", H2_ERR_INVALID_ARG);
  if (perm) std::memcpy(perm, T->perm.data(), sizeof(int64_t) * T->n);
  int64_t pos = 0;
  for (int t = 0; t <= T->Dl; ++t)
    for (size_t c = 0; c < T->begin[t].size(); ++c, ++pos) {
      if (begin) begin[pos] = T->begin[t][c];
      if (end) end[pos] = T->end[t][c];
    }
  if (near_pairs) {
    try {
      const_cast<h2_tree*>(T)->wait_partition();
    } catch (const Error& e) {
      return fail(e);
    }
    for (int64_t s = 0; s < (int64_t)T->near.ptr.size() - 1; ++s)
      for (int e = T->near.ptr[s]; e < T->near.ptr[s + 1]; ++e) {
        near_pairs[2 * e] = (int32_t)s;
        near_pairs[2 * e + 1] = T->near.idx[e];
      }
  }
  return H2_OK;
}

h2_status h2_tree_far_count(const h2_tree* T, int32_t depth, int64_t* nnz) {
  if (!T || !nnz || depth < 0 || depth > T->Dl) return (g_err = "h2_tree_far_count: bad argument", H2_ERR_INVALID_ARG);
  try {
    const_cast<h2_tree*>(T)->wait_partition();
  } catch (const Error& e) {
    return fail(e);
  }
  *nnz = T->far[depth].nnz();
  return H2_OK;
}

h2_status h2_tree_export_far(const h2_tree* T, int32_t depth, int32_t* far_pairs) {
  if (!T || !far_pairs || depth < 0 || depth > T->Dl)
    return (g_err = "h2_tree_export_far: bad argument", H2_ERR_INVALID_ARG);
  try {
    const_cast<h2_tree*>(T)->wait_partition();
  } catch (const Error& e) {
    return fail(e);
  }
  const PairCSR& F = T->far[depth];
  for (int64_t s = 0; s < (int64_t)F.ptr.size() - 1; ++s)
    for (int e = F.ptr[s]; e < F.ptr[s + 1]; ++e) {
      far_pairs[2 * e] = (int32_t)s;
      far_pairs[2 * e + 1] = F.idx[e];
    }
  return H2_OK;
}

void h2_tree_free(h2_tree* T) { delete T; }

void h2_build_opts_default(h2_build_opts* o) {
  if (!o) return;
  o->d_init = 32;
  o->d_blk = 32;
  o->d_max = 512;
  o->adaptive = 1;
  o->tol_rule = H2_TOL_RMS;
  o->tol_safety = 0.04;
  o->p_os = 10;
  o->norm = 0.0;
  o->max_rank = 0;
  o->seed = 1;
  o->stream_id = 0;
  o->verify_probes = 0;
  o->verify_retries = 2;
  o->eps_decay = 1.25;
  o->exact_order = 0;
  o->omega_ext = nullptr;
  o->ld_omega_ext = 0;
  o->norm_iters = 10;
  o->sketch_split = H2_SPLIT_ROWS;
}

h2_status h2_dist_range(int64_t n_clusters, int32_t rank, int32_t nranks, int64_t* begin, int64_t* end) {
  if (!begin || !end || nranks < 1 || rank < 0 || rank >= nranks || n_clusters < 0)
    return (g_err = "h2_dist_range: bad argument", H2_ERR_INVALID_ARG);
  *begin = (rank * n_clusters + nranks - 1) / nranks;
  *end = ((rank + 1) * n_clusters + nranks - 1) / nranks;
  return H2_OK;
}

h2_status h2_build(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                   const h2_build_opts* opts, void* stream, h2_matrix** out, h2_build_stats* stats) {
  return h2_build_dist(tree, sketch, entry, tol, opts, nullptr, stream, out, stats);
}

}  // extern "C"

namespace {
// O10 a-posteriori check: ||H Om_h - K_blk(Om_h)||_F / ||K_blk(Om_h)||_F (h2_verify)
double verify_impl(const h2_matrix& H, const h2_sketch& S, int q, uint64_t seed, uint32_t sid, cudaStream_t st) {
  const h2_tree& T = *H.tree;
  const int nleaf = 1 << T.Dl;
  DArr<double> Om, Yh, part, acc;
  DArr<int> nf;
  Om.alloc(T.n * q, st);
  Yh.alloc(T.n * q, st);
  part.alloc(nleaf, st);
  acc.alloc(2, st);
  nf.alloc(1, st);
  H2_CUDA(cudaMemsetAsync(acc.p, 0, 2 * sizeof(double), st));
  H2_CUDA(cudaMemsetAsync(nf.p, 0, sizeof(int), st));
  launch_omega(seed, sid, 0, T.n, 0, q, Om.p, q, st);
  apply_sketch_op(T, S, Om.p, q, q, Yh.p, q, true, false, st);
  launch_sumsq_leaf(Yh.p, T.d_leaf_begin, 0, nleaf, q, 0, q, part.p, st);
  launch_sumsq_total(part.p, nleaf, acc.p, nf.p, st);
  matvec_impl(H, Om.p, q, Yh.p, q, q, 1.0, -1.0, st);   // Yh = H Om_h - Y_h
  launch_sumsq_leaf(Yh.p, T.d_leaf_begin, 0, nleaf, q, 0, q, part.p, st);
  launch_sumsq_total(part.p, nleaf, acc.p + 1, nf.p, st);
  double a[2];
  int bad = 0;
  H2_CUDA(cudaMemcpyAsync(a, acc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaMemcpyAsync(&bad, nf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Error(H2_ERR_NONFINITE, "h2_verify: non-finite sample");
  return a[0] > 0 ? std::sqrt(a[1] / a[0]) : std::sqrt(a[1]);
}

// The paper's error measure: ||H - K_blk||_2 and ||K_blk||_2 by `iters` power
// iterations each, run independently from nvec unit start vectors (columns 0..nvec-1 of the h2_omega
// stream (seed, sid)) side by side -- one sketch call per iteration for all of them, the dense
// sketch's cost being its kernel evaluations -- x <- A x / ||A x||; the estimate is the largest
// ||A x|| of the last iteration.  Symmetric H and K_blk (A = H - K_blk symmetric: ||A x|| for unit x
// converges to ||A||_2 from below).  Returns (error estimate, norm estimate).
std::pair<double, double> power2_impl(const h2_matrix& H, const h2_sketch& S, int iters, int nvec, uint64_t seed,
                                      uint32_t sid, cudaStream_t st) {
  const h2_tree& T = *H.tree;
  const int nleaf = 1 << T.Dl;
  const int q = nvec;
  DArr<double> x, y, part, acc;
  DArr<int> nf;
  x.alloc(T.n * q, st);
  y.alloc(T.n * q, st);
  part.alloc(nleaf, st);
  acc.alloc(q, st);
  nf.alloc(1, st);
  std::vector<double> nrm(q);
  auto norms = [&](const double* v) {   // per-column 2-norms of an n x q row-major block
    H2_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(double) * q, st));
    H2_CUDA(cudaMemsetAsync(nf.p, 0, sizeof(int), st));
    for (int c = 0; c < q; ++c) {
      launch_sumsq_leaf(v, T.d_leaf_begin, 0, nleaf, q, c, c + 1, part.p, st);
      launch_sumsq_total(part.p, nleaf, acc.p + c, nf.p, st);
    }
    int bad = 0;
    H2_CUDA(cudaMemcpyAsync(nrm.data(), acc.p, sizeof(double) * q, cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaMemcpyAsync(&bad, nf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    H2_CUDA(cudaStreamSynchronize(st));
    if (bad) throw Error(H2_ERR_NONFINITE, "h2_verify_2norm: non-finite vector");
    for (double& v : nrm) v = std::sqrt(v);
  };
  auto power = [&](bool diff) {
    launch_omega(seed, sid, 0, T.n, 0, q, x.p, q, st);
    norms(x.p);
    for (int c = 0; c < q; ++c) launch_scale(x.p + c, T.n, q, 1, 1.0 / nrm[c], st);
    double best = 0;
    for (int it = 0; it < iters; ++it) {
      apply_sketch_op(T, S, x.p, q, q, y.p, q, false, false, st);              // y = K_blk x
      if (diff) matvec_impl(H, x.p, q, y.p, q, q, 1.0, -1.0, st);              // y = H x - K_blk x
      norms(y.p);
      best = 0;
      for (int c = 0; c < q; ++c) best = std::max(best, nrm[c]);
      if (!(best > 0)) return 0.0;
      H2_CUDA(cudaMemcpyAsync(x.p, y.p, sizeof(double) * T.n * q, cudaMemcpyDeviceToDevice, st));
      for (int c = 0; c < q; ++c) launch_scale(x.p + c, T.n, q, 1, nrm[c] > 0 ? 1.0 / nrm[c] : 0.0, st);
    }
    return best;
  };
  const double e = power(true);
  const double k = power(false);
  return {e, k};
}

}  // namespace

namespace {
// Y = K_blk(Om) for all n rows with any sketch operator (a-posteriori check, norm estimate);
// quarters: Om is the h2_omega stream (tensor-core sketch allowed); exact: exact-order sketch
void apply_sketch_op(const h2_tree& T, const h2_sketch& S, const double* Om, int64_t ldo, int q, double* Y,
                     int64_t ldy, bool quarters, bool exact, cudaStream_t st) {
  if (S.kind == H2_S_DENSE_KERNEL) {
    const KernelParams kp = tree_kernel(&T, S.kern, st);
    if (exact) launch_exact_sketch(kp, T.d_x, T.d_y, T.d_z, T.n, 0, T.n, Om, ldo, q, Y, ldy, st);
    else launch_dense_sketch(kp, T.d_x, T.d_y, T.d_z, T.n, 0, T.n, Om, ldo, q, Y, ldy, quarters, st);
  } else if (S.kind == H2_S_DENSE_MATRIX) {
    dense_matrix_sketch(S.A, S.ld_A, T.n, 0, T.n, Om, ldo, q, Y, ldy, st);
  } else if (S.kind == H2_S_H2_LOWRANK) {
    matvec_impl(*S.base, Om, ldo, Y, ldy, q, 1.0, 0.0, st);
    if (S.rank > 0) {
      DArr<double> scr;
      scr.alloc((int64_t)(div_up(T.n, 1024) + 1) * S.rank * q, st);
      launch_lowrank_sketch(S.U, S.ld_U, S.rank, Om, ldo, q, T.n, Y, ldy, scr.p, st);
    }
  } else {
    h2_sketch_req rq{};
    rq.n = T.n;
    rq.row_begin = 0;
    rq.row_end = T.n;
    rq.col0 = 0;
    rq.ncols = q;
    rq.omega = Om;
    rq.ld_omega = ldo;
    rq.y = Y;
    rq.ld_y = ldy;
    rq.stream = st;
    int rc = S.fn(S.ctx, &rq);
    if (rc != 0) throw Error(H2_ERR_CALLBACK, "sketch callback returned " + std::to_string(rc));
  }
}

void reset_matrix(h2_matrix& H) {
  H.lv.clear();
  H.lvc.clear();
  H.D = DArr<double>();
  H.d_D_off = DArr<int64_t>();
  H.D_off.clear();
  H.nonsym = false;
  std::memset(&H.stats, 0, sizeof(H.stats));
  H.stats.failed_depth = -1;
}
}  // namespace

extern "C" {

h2_status h2_verify(const h2_matrix* H, const h2_sketch* sketch, int32_t ncols, uint64_t seed, uint32_t stream_id,
                    void* stream, double* err) {
  try {
    H2_REQUIRE(H && sketch && err, "h2_verify: NULL argument");
    H2_REQUIRE(!H->partial, "h2_verify: distributed matrix: call h2_matrix_allgather first");
    H2_REQUIRE(ncols >= 1 && ncols <= 64, "h2_verify: need 1 <= ncols <= 64");
    H2_REQUIRE(sketch->kind == H2_S_DENSE_KERNEL || (sketch->kind == H2_S_CALLBACK && sketch->fn) ||
                   (sketch->kind == H2_S_H2_LOWRANK && sketch->base && !sketch->base->partial) ||
                   (sketch->kind == H2_S_DENSE_MATRIX && sketch->A && sketch->ld_A >= H->n),
               "h2_verify: bad sketch");
    *err = verify_impl(*H, *sketch, ncols, seed, stream_id, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_verify_2norm(const h2_matrix* H, const h2_sketch* sketch, int32_t iters, int32_t nvec, uint64_t seed,
                          uint32_t stream_id, void* stream, double* err, double* abs_err, double* knorm) {
  try {
    H2_REQUIRE(H && sketch && err, "h2_verify_2norm: NULL argument");
    H2_REQUIRE(!H->partial, "h2_verify_2norm: distributed matrix: call h2_matrix_allgather first");
    H2_REQUIRE(!H->nonsym, "h2_verify_2norm: symmetric matrices only");
    H2_REQUIRE(iters >= 1 && iters <= 1000 && nvec >= 1 && nvec <= 64,
               "h2_verify_2norm: need 1 <= iters <= 1000, 1 <= nvec <= 64");
    H2_REQUIRE(sketch->kind == H2_S_DENSE_KERNEL || (sketch->kind == H2_S_CALLBACK && sketch->fn) ||
                   (sketch->kind == H2_S_H2_LOWRANK && sketch->base && !sketch->base->partial) ||
                   (sketch->kind == H2_S_DENSE_MATRIX && sketch->A && sketch->ld_A >= H->n),
               "h2_verify_2norm: bad sketch");
    const auto ek = power2_impl(*H, *sketch, iters, nvec, seed, stream_id, (cudaStream_t)stream);
    *err = ek.second > 0 ? ek.first / ek.second : ek.first;
    if (abs_err) *abs_err = ek.first;
    if (knorm) *knorm = ek.second;
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

static h2_status build_impl(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                            const h2_build_opts* opts, const h2_comm* comm, void* stream, h2_matrix** out,
                            h2_build_stats* stats, bool nonsym) {
  if (!out) return (g_err = "h2_build: out is NULL", H2_ERR_INVALID_ARG);
  *out = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  h2_build_opts o;
  h2_build_opts_default(&o);
  if (opts) o = *opts;
  auto* H = new h2_matrix();
  std::memset(&H->stats, 0, sizeof(H->stats));
  H->stats.failed_depth = -1;
  int64_t launches0 = h2::g_launches;
  auto t0 = std::chrono::steady_clock::now();
  g_alloc_ms = 0;
  try {
    H2_REQUIRE(tree && sketch && entry, "h2_build: NULL tree/sketch/entry");
    H2_REQUIRE(tol >= 0 && std::isfinite(tol), "h2_build: tol must be finite and >= 0");
    H2_REQUIRE(o.d_init >= 1 && o.d_blk >= 1 && o.d_max >= o.d_init, "h2_build: need 1 <= d_init <= d_max, d_blk >= 1");
    H2_REQUIRE(o.tol_rule == H2_TOL_RMS || o.tol_rule == H2_TOL_LITERAL, "h2_build: bad tol_rule");
    H2_REQUIRE(o.tol_rule != H2_TOL_LITERAL || o.norm > 0 || (!nonsym && o.norm_iters >= 0),
               "h2_build: literal tolerance needs opts.norm > 0 (or the power-iteration estimate, symmetric builds)");
    H2_REQUIRE(!o.exact_order || (!nonsym && sketch->kind == H2_S_DENSE_KERNEL && entry->kind == H2_E_BUILTIN),
               "h2_build: exact_order needs a symmetric build with the built-in dense-kernel sketch and entries");
    H2_REQUIRE(!o.omega_ext || (!nonsym && o.ld_omega_ext >= o.d_max),
               "h2_build: omega_ext needs ld_omega_ext >= d_max (symmetric builds)");
    H2_REQUIRE(sketch->kind == H2_S_DENSE_KERNEL || (sketch->kind == H2_S_CALLBACK && sketch->fn) ||
                   sketch->kind == H2_S_H2_LOWRANK ||
                   (sketch->kind == H2_S_DENSE_MATRIX && sketch->A && sketch->ld_A >= tree->n),
               "h2_build: bad sketch");
    H2_REQUIRE(entry->kind == H2_E_BUILTIN || (entry->kind == H2_E_CALLBACK && entry->fn) ||
                   entry->kind == H2_E_H2_LOWRANK ||
                   (entry->kind == H2_E_DENSE_MATRIX && entry->A && entry->ld_A >= tree->n),
               "h2_build: bad entry");
    for (int which = 0; which < 2; ++which) {
      const bool upd = which == 0 ? sketch->kind == H2_S_H2_LOWRANK : entry->kind == H2_E_H2_LOWRANK;
      if (!upd) continue;
      const h2_matrix* base = which == 0 ? sketch->base : entry->base;
      const double* U = which == 0 ? sketch->U : entry->U;
      const int32_t r = which == 0 ? sketch->rank : entry->rank;
      const int64_t ldu = which == 0 ? sketch->ld_U : entry->ld_U;
      H2_REQUIRE(base && base->tree.get() == tree, "h2_build: the H2+low-rank operator needs a base built on this tree");
      // rank 0 (sketch only): Y = A_H Omega, the O(N) H^2-matvec sketch of an existing H^2 (S§8(f) NEXT #1)
      const bool pure = which == 0 && r == 0;
      H2_REQUIRE(pure || (U && r >= 1 && r <= 1024 && ldu >= r),
                 "h2_build: H2+low-rank operator needs U (n x rank, ld >= rank)");
    }
    for (const h2_kernel* k : {sketch->kind == H2_S_DENSE_KERNEL ? &sketch->kern : nullptr,
                               entry->kind == H2_E_BUILTIN ? &entry->kern : nullptr})
      if (k)
        H2_REQUIRE((k->kind == H2_K_EXP || k->kind == H2_K_HELMHOLTZ || k->kind == H2_K_RATIONAL) && k->param > 0,
                   "h2_build: bad kernel");
    // U V^T (V != U) is a non-symmetric operator
    H2_REQUIRE(nonsym || ((sketch->kind != H2_S_H2_LOWRANK || !sketch->V || sketch->V == sketch->U) &&
                          (entry->kind != H2_E_H2_LOWRANK || !entry->V || entry->V == entry->U)),
               "h2_build: an H2 + U V^T operator with V != U needs h2_build_nonsym");
    for (const h2_matrix* b : {sketch->kind == H2_S_H2_LOWRANK ? sketch->base : nullptr,
                               entry->kind == H2_E_H2_LOWRANK ? entry->base : nullptr})
      H2_REQUIRE(!b || (!b->nonsym && !b->partial), "h2_build: the H2+low-rank base must be a complete symmetric H2");
    const bool dist = comm && comm->nranks > 1;
    if (comm)
      H2_REQUIRE(comm->nranks >= 1 && comm->rank >= 0 && comm->rank < comm->nranks &&
                     (!dist || comm->allgatherv || comm->nccl),
                 "h2_build_dist: bad communicator");
    H2_REQUIRE(o.sketch_split == H2_SPLIT_ROWS || o.sketch_split == H2_SPLIT_COLS, "h2_build: bad sketch_split");
    H2_REQUIRE(!dist || o.sketch_split != H2_SPLIT_COLS || sketch->kind != H2_S_CALLBACK || comm->alltoallv ||
                   comm->nccl,
               "h2_build_dist: sketch_split = H2_SPLIT_COLS needs an all-to-all (comm->alltoallv or NCCL)");
    // H2 + low-rank operators under a communicator: the base must be complete on every rank
    // (checked above: not partial); its matvec is row-sharded, its entries extracted per owned pair
    // subtree-aligned ownership at every processed depth: a power-of-two rank count with at
    // least one cluster per rank at the coarsest processed depth
    if (dist || nonsym) ensure_uploaded(tree);   // the partition up front
    else ensure_order_uploaded(tree);            // Builder::run waits for it (tree_ready)
    H2_REQUIRE(!dist || ((comm->nranks & (comm->nranks - 1)) == 0 && tree->top >= 0 &&
                         (int64_t(1) << tree->top) >= comm->nranks),
               "h2_build_dist: nranks must be a power of two <= 2^top_depth");
    // the tree is owned by the caller; share it without taking ownership
    H->tree = std::shared_ptr<h2_tree>(const_cast<h2_tree*>(tree), [](h2_tree*) {});
    H2_REQUIRE(o.eps_decay > 0 && std::isfinite(o.eps_decay), "h2_build: eps_decay must be > 0");
    H2_REQUIRE(o.verify_probes >= 0 && o.verify_probes <= 64 && o.verify_retries >= 0,
               "h2_build: need 0 <= verify_probes <= 64, verify_retries >= 0");
    for (int rebuilds = 0;; ++rebuilds) {
      {
        Builder B(*tree, *sketch, *entry, tol, o, st, *H, comm);
        if (nonsym) B.run_nonsym();
        else B.run();
      }
      H->stats.tol_safety_used = o.tol_safety;
      H->stats.verify_rebuilds = rebuilds;
      if (dist || o.verify_probes <= 0) break;
      // O10 (R30): held-out columns of stream stream_id + 2; rebuild with s / 3 while e > tol
      const double e = verify_impl(*H, *sketch, o.verify_probes, o.seed, o.stream_id + 2, st);
      H->stats.verify_error = e;
      if (!(e > tol) || rebuilds >= o.verify_retries) break;
      reset_matrix(*H);
      o.tol_safety /= 3;
    }
    if (dist) {
      H->nranks = comm->nranks;
      H->rank = comm->rank;
      H->partial = true;
    }
    H->stats.launches = h2::g_launches - launches0;
    H->stats.t_total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = H->stats;
    *out = H;
    return H2_OK;
  } catch (const Error& e) {
    if (stats) {
      *stats = H->stats;
    }
    cudaStreamSynchronize(st);
    delete H;
    return fail(e);
  } catch (const std::bad_alloc&) {
    delete H;
    g_err = "h2_build: host out of memory";
    return H2_ERR_OOM;
  }
}

h2_status h2_build_dist(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                        const h2_build_opts* opts, const h2_comm* comm, void* stream, h2_matrix** out,
                        h2_build_stats* stats) {
  return build_impl(tree, sketch, entry, tol, opts, comm, stream, out, stats, false);
}

h2_status h2_build_nonsym(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                          const h2_build_opts* opts, void* stream, h2_matrix** out, h2_build_stats* stats) {
  return build_impl(tree, sketch, entry, tol, opts, nullptr, stream, out, stats, true);
}

h2_status h2_build_nonsym_dist(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                               const h2_build_opts* opts, const h2_comm* comm, void* stream, h2_matrix** out,
                               h2_build_stats* stats) {
  return build_impl(tree, sketch, entry, tol, opts, comm, stream, out, stats, true);
}

h2_status h2_matrix_allgather(h2_matrix* H, const h2_comm* comm, void* stream) {
  try {
    H2_REQUIRE(H, "h2_matrix_allgather: NULL matrix");
    if (!H->partial) return H2_OK;
    H2_REQUIRE(comm && comm->nranks == H->nranks && comm->rank == H->rank && (comm->allgatherv || comm->nccl),
               "h2_matrix_allgather: communicator does not match the build");
    cudaStream_t st = (cudaStream_t)stream;
    const h2_tree& T = *H->tree;
    const int P = comm->nranks;
    // blocks stored once per unique pair (s, b), sorted by s: the pairs whose row cluster s is
    // owned by rank r form one contiguous range of unique indices
    auto block_ranges = [&](const PairCSR& F, int t, const std::vector<int64_t>& off, double* base) {
      std::vector<int64_t> cnt(P), dsp(P);
      for (int r = 0; r < P; ++r) {
        const int a = own_begin(t, r, P), b = own_begin(t, r + 1, P);
        const int64_t u0 = std::lower_bound(F.us.begin(), F.us.end(), a) - F.us.begin();
        const int64_t u1 = std::lower_bound(F.us.begin(), F.us.end(), b) - F.us.begin();
        dsp[r] = off[u0] * 8;
        cnt[r] = (off[u1] - off[u0]) * 8;
      }
      comm_allgather(comm, base, cnt, dsp, st);
    };
    if (H->nonsym) {
      // ordered pairs e in CSR order (sorted by the row cluster s): rank r's rows are the entries
      // [ptr[own_begin(r)], ptr[own_begin(r+1)])
      auto ordered_ranges = [&](const PairCSR& F, int t, const std::vector<int64_t>& off, double* base) {
        std::vector<int64_t> cnt(P), dsp(P);
        for (int r = 0; r < P; ++r) {
          const int64_t e0 = F.ptr[own_begin(t, r, P)], e1 = F.ptr[own_begin(t, r + 1, P)];
          dsp[r] = off[e0] * 8;
          cnt[r] = (off[e1] - off[e0]) * 8;
        }
        comm_allgather(comm, base, cnt, dsp, st);
      };
      for (int t = H->top; t <= H->Dl; ++t) {
        for (int sd = 0; sd < 2; ++sd) {
          Level& L = H->S(sd, t);
          comm_allgather_clusters(comm, L.X.p, 8, t, [&](int c) { return c < L.nclus ? L.xoff[c] : L.xtot; }, st);
          comm_allgather_clusters(comm, L.cert.p, 16, t, [](int c) { return (int64_t)c; }, st);
        }
        if (T.far[t].nnz() > 0) ordered_ranges(T.far[t], t, H->L(t).B_off, H->L(t).B.p);
      }
      ordered_ranges(T.near, T.Dl, H->D_off, H->D.p);
      H2_CUDA(cudaStreamSynchronize(st));
      H->partial = false;
      return H2_OK;
    }
    for (int t = H->top; t <= H->Dl; ++t) {
      Level& L = H->L(t);
      comm_allgather_clusters(comm, L.X.p, 8, t, [&](int c) { return c < L.nclus ? L.xoff[c] : L.xtot; }, st);
      comm_allgather_clusters(comm, L.cert.p, 16, t, [](int c) { return (int64_t)c; }, st);
      if (T.far[t].nuniq() > 0) block_ranges(T.far[t], t, L.B_off, L.B.p);
    }
    block_ranges(T.near, T.Dl, T.D_off, H->D.p);
    H2_CUDA(cudaStreamSynchronize(st));
    H->partial = false;
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_matvec(const h2_matrix* H, const double* x, int64_t ldx, double* y, int64_t ldy, int32_t q, double alpha,
                    double beta, void* stream) {
  try {
    H2_REQUIRE(H && x && y, "h2_matvec: NULL argument");
    H2_REQUIRE(!H->partial, "h2_matvec: distributed matrix: call h2_matrix_allgather first");
    H2_REQUIRE(q >= 1 && q <= 64 && ldx >= q && ldy >= q, "h2_matvec: need 1 <= ncols <= 64, ld >= ncols");
    matvec_impl(*H, x, ldx, y, ldy, q, alpha, beta, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_dense_sketch(const h2_tree* T, h2_kernel kern, int64_t row_begin, int64_t row_end, const double* omega,
                          int64_t ld_omega, int32_t ncols, double* y, int64_t ld_y, int32_t flags, void* stream) {
  try {
    H2_REQUIRE(T && omega && y, "h2_dense_sketch: NULL argument");
    H2_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= T->n, "h2_dense_sketch: bad row range");
    H2_REQUIRE(ncols >= 0 && ld_omega >= ncols && ld_y >= ncols, "h2_dense_sketch: bad ncols / leading dims");
    H2_REQUIRE((kern.kind == H2_K_EXP || kern.kind == H2_K_HELMHOLTZ || kern.kind == H2_K_RATIONAL) && kern.param > 0,
               "h2_dense_sketch: bad kernel");
    ensure_uploaded(T);
    launch_dense_sketch(tree_kernel(T, kern, (cudaStream_t)stream), T->d_x, T->d_y, T->d_z, T->n, row_begin, row_end, omega, ld_omega, ncols, y,
                        ld_y, (flags & H2_SKETCH_OMEGA_QUARTERS) != 0, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_dense_op_sketch(const double* A, int64_t lda, int64_t n, int64_t row_begin, int64_t row_end,
                             const double* omega, int64_t ld_omega, int32_t ncols, double* y, int64_t ld_y, int32_t flags,
                             void* stream) {
  try {
    H2_REQUIRE(A && omega && y && n >= 1 && lda >= n, "h2_dense_op_sketch: bad argument");
    H2_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= n, "h2_dense_op_sketch: bad row range");
    H2_REQUIRE(ncols >= 0 && ld_omega >= ncols && ld_y >= ncols, "h2_dense_op_sketch: bad ncols / leading dims");
    cudaStream_t st = (cudaStream_t)stream;
    if (flags & H2_SKETCH_OMEGA_QUARTERS)
      launch_dense_op_tc(A, lda, n, row_begin, row_end, dense_absmax(A, lda, n, st), omega, ld_omega, ncols, y, ld_y, st);
    else
      dense_matrix_sketch(A, lda, n, row_begin, row_end, omega, ld_omega, ncols, y, ld_y, st);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_omega(uint64_t seed, uint32_t stream_id, int64_t row0, int64_t nrows, int32_t col0, int32_t ncols,
                   double* out, int64_t ld, void* stream) {
  try {
    H2_REQUIRE(out && row0 >= 0 && nrows >= 0 && col0 >= 0 && ncols >= 0 && ld >= ncols, "h2_omega: bad argument");
    launch_omega(seed, stream_id, row0, nrows, col0, ncols, out, ld, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_export_size(const h2_matrix* H, int32_t what, int32_t depth, int64_t* count) {
  if (!H || !count) return (g_err = "h2_export_size: NULL argument", H2_ERR_INVALID_ARG);
  if (what == H2_X_D) {
    *count = H->D.n;
    return H2_OK;
  }
  if (depth == H2_ALL_DEPTHS) {
    if (!(what == H2_X_RANK || what == H2_X_SKEL || ((what == H2_X_RANK_C || what == H2_X_SKEL_C) && H->nonsym)))
      return (g_err = "h2_export_size: all depths for ranks / skeletons only", H2_ERR_INVALID_ARG);
    int64_t c = 0;
    for (int t = H->top; t <= H->Dl; ++t) {
      int64_t ct = 0;
      h2_status s = h2_export_size(H, what, t, &ct);
      if (s != H2_OK) return s;
      c += ct;
    }
    *count = c;
    return H2_OK;
  }
  if (depth < H->top || depth > H->Dl) return (g_err = "h2_export_size: depth outside [top, leaf]", H2_ERR_INVALID_ARG);
  if (what >= H2_X_RANK_C && what <= H2_X_CERT_C) {
    if (!H->nonsym) return (g_err = "h2_export_size: column side exists for h2_build_nonsym matrices only", H2_ERR_INVALID_ARG);
    const Level& C = H->C(depth);
    switch (what) {
      case H2_X_RANK_C: *count = C.nclus; break;
      case H2_X_SKEL_C: *count = C.rtot; break;
      case H2_X_BASIS_C: *count = C.xtot; break;
      default: *count = 2 * (int64_t)C.nclus; break;
    }
    return H2_OK;
  }
  const Level& L = H->L(depth);
  switch (what) {
    case H2_X_RANK: *count = L.nclus; break;
    case H2_X_SKEL: *count = L.rtot; break;
    case H2_X_BASIS: *count = L.xtot; break;
    case H2_X_B: *count = L.B_off.empty() ? 0 : L.B_off.back(); break;
    case H2_X_CERT: *count = 2 * (int64_t)L.nclus; break;
    default: return (g_err = "h2_export_size: bad `what`", H2_ERR_INVALID_ARG);
  }
  return H2_OK;
}

h2_status h2_export(const h2_matrix* H, int32_t what, int32_t depth, void* dst) {
  if (H && H->partial && (what == H2_X_BASIS || what == H2_X_D || what == H2_X_B || what == H2_X_CERT || what >= H2_X_RANK_C))
    return (g_err = "h2_export: distributed matrix: call h2_matrix_allgather first", H2_ERR_INVALID_ARG);
  int64_t cnt = 0;
  h2_status s = h2_export_size(H, what, depth, &cnt);
  if (s != H2_OK) return s;
  if (!dst) return (g_err = "h2_export: NULL dst", H2_ERR_INVALID_ARG);
  if (cnt == 0) return H2_OK;
  if (depth == H2_ALL_DEPTHS) {   // ranks / skeletons of every depth: async copies, one sync
    char* out = static_cast<char*>(dst);
    for (int t = H->top; t <= H->Dl; ++t) {
      const Level& L = (what >= H2_X_RANK_C) ? H->C(t) : H->L(t);
      const bool rk = what == H2_X_RANK || what == H2_X_RANK_C;
      const int64_t n = rk ? L.nclus : L.rtot;
      if (n > 0) {
        cudaError_t e = cudaMemcpyAsync(out, rk ? (const void*)L.d_k.p : (const void*)L.d_skel.p, 4 * n,
                                        cudaMemcpyDefault, 0);
        if (e != cudaSuccess) return (g_err = std::string("h2_export: ") + cudaGetErrorString(e), H2_ERR_CUDA);
      }
      out += 4 * n;
    }
    cudaError_t e = cudaStreamSynchronize(0);
    if (e != cudaSuccess) return (g_err = std::string("h2_export: ") + cudaGetErrorString(e), H2_ERR_CUDA);
    return H2_OK;
  }
  const void* src = nullptr;
  size_t el = 8;
  if (what == H2_X_D) src = H->D.p;
  else if (what >= H2_X_RANK_C) {
    const Level& C = H->C(depth);
    switch (what) {
      case H2_X_RANK_C: src = C.d_k.p; el = 4; break;
      case H2_X_SKEL_C: src = C.d_skel.p; el = 4; break;
      case H2_X_BASIS_C: src = C.X.p; break;
      default: src = C.cert.p; break;
    }
  } else {
    const Level& L = H->L(depth);
    switch (what) {
      case H2_X_RANK: src = L.d_k.p; el = 4; break;
      case H2_X_SKEL: src = L.d_skel.p; el = 4; break;
      case H2_X_BASIS: src = L.X.p; break;
      case H2_X_B: src = L.B.p; break;
      case H2_X_CERT: src = L.cert.p; break;
    }
  }
  cudaError_t e = cudaMemcpy(dst, src, el * cnt, cudaMemcpyDefault);
  if (e != cudaSuccess) return (g_err = std::string("h2_export: ") + cudaGetErrorString(e), H2_ERR_CUDA);
  return H2_OK;
}

h2_status h2_matrix_get_stats(const h2_matrix* H, h2_build_stats* stats) {
  if (!H || !stats) return (g_err = "h2_matrix_get_stats: NULL argument", H2_ERR_INVALID_ARG);
  *stats = H->stats;
  return H2_OK;
}

int64_t h2_matrix_device_bytes(const h2_matrix* H) {
  if (!H) return 0;
  int64_t b = H->D.bytes();
  for (auto* lvs : {&H->lv, &H->lvc})
    for (auto& L : *lvs) b += L.X.bytes() + L.B.bytes() + L.d_skel.bytes() + L.d_perm.bytes();
  b += H->d_D_off.bytes();
  return b;
}

void h2_free(h2_matrix* H) { delete H; }

h2_status h2_comm_get_unique_id(void* id128) {
  try {
    H2_REQUIRE(id128, "h2_comm_get_unique_id: NULL id");
    h2::nccl_unique_id(id128);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_comm_init(const void* id128, int32_t rank, int32_t nranks, h2_comm** out) {
  if (!out) return (g_err = "h2_comm_init: out is NULL", H2_ERR_INVALID_ARG);
  *out = nullptr;
  try {
    H2_REQUIRE(id128 && nranks >= 1 && rank >= 0 && rank < nranks, "h2_comm_init: bad argument");
    auto* c = new h2_comm{};
    c->rank = rank;
    c->nranks = nranks;
    c->allgatherv = nullptr;
    c->alltoallv = nullptr;
    c->ctx = nullptr;
    try {
      c->nccl = h2::nccl_comm_init(id128, rank, nranks);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

void h2_comm_free(h2_comm* c) {
  if (!c) return;
  try {
    h2::nccl_comm_free(c->nccl);
  } catch (const Error&) {
  }
  delete c;
}

h2_status h2_comm_allgatherv(const h2_comm* comm, void* buf, const int64_t* counts, const int64_t* displs,
                             void* stream) {
  try {
    H2_REQUIRE(comm && counts && displs && (comm->allgatherv || comm->nccl) && comm->nranks >= 1,
               "h2_comm_allgatherv: bad argument");
    std::vector<int64_t> c(counts, counts + comm->nranks), d(displs, displs + comm->nranks);
    for (int r = 0; r < comm->nranks; ++r) H2_REQUIRE(c[r] >= 0 && d[r] >= 0, "h2_comm_allgatherv: negative segment");
    comm_allgather(comm, buf, c, d, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

h2_status h2_comm_alltoallv(const h2_comm* comm, const void* send, const int64_t* scounts, const int64_t* sdispls,
                            void* recv, const int64_t* rcounts, const int64_t* rdispls, void* stream) {
  try {
    H2_REQUIRE(comm && scounts && sdispls && rcounts && rdispls && comm->nranks >= 1 &&
                   comm->rank >= 0 && comm->rank < comm->nranks,
               "h2_comm_alltoallv: bad argument");
    const int P = comm->nranks;
    std::vector<int64_t> sc(scounts, scounts + P), sd(sdispls, sdispls + P), rc(rcounts, rcounts + P),
        rd(rdispls, rdispls + P);
    for (int r = 0; r < P; ++r)
      H2_REQUIRE(sc[r] >= 0 && sd[r] >= 0 && rc[r] >= 0 && rd[r] >= 0, "h2_comm_alltoallv: negative segment");
    H2_REQUIRE(sc[comm->rank] == rc[comm->rank], "h2_comm_alltoallv: own send and receive segments differ");
    comm_alltoall(comm, send, sc, sd, recv, rc, rd, (cudaStream_t)stream);
    return H2_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

int64_t h2_cache_bytes(void) { return (int64_t)h2::cache_bytes_held(); }
void h2_cache_trim(void) { h2::cache_trim(); }

}  // extern "C"
