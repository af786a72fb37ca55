// batchedID: column-pivoted QR of every panel A_c = (Y^loc_c)^T,
// which is also the convergence test of §III-B (L361, "QR decomposition ... smallest absolute
// value of the diagonal"; reading R12), the ID epilogue (T = R11^{-1} R12, Eq.(3)) and the
// shrink / Omega upsweep (batchedShrink L222/L251, batchedGemm L223/L252).
#include <cooperative_groups.h>

#include "alloc.hpp"
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// (best value, index, second-best value) reduction: ties -> lowest index (R14)
struct Top2 {
  double v;
  int i;
  double s;
};

__device__ __forceinline__ Top2 top2_merge(Top2 a, Top2 b) {
  Top2 r;
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) {
    r.v = b.v;
    r.i = b.i;
    r.s = fmax(b.s, a.v);
  } else {
    r.v = a.v;
    r.i = a.i;
    r.s = fmax(a.s, b.v);
  }
  return r;
}

__device__ __forceinline__ Top2 warp_top2(Top2 t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Top2 u;
    u.v = __shfl_xor_sync(0xffffffffu, t.v, o);
    u.i = __shfl_xor_sync(0xffffffffu, t.i, o);
    u.s = __shfl_xor_sync(0xffffffffu, t.s, o);
    t = top2_merge(t, u);
  }
  return t;
}


// One CTA per cluster.  The panel lives in shared memory (rows padded to LD = d rounded up to
// 8 doubles, LD = 8 mod 16: conflict-free) or, when too large, in W (global, L1/L2 resident).
// Row j = column j of A (a point's d samples).  Residual column norms are RECOMPUTED from the
// updated trailing rows every step (R14); the norm for step i+1 is fused into the reflector
// update of step i (one pass over the trailing panel per step).
// Work split: 8 threads per panel row (thread s of a row handles entries r = s mod 8, then a
// 3-step shuffle reduction), NT/8 rows at a time: the dot / update / norm chains are short and
// independent, instead of one warp per row with 5-step butterflies (latency bound: ~1 flop/clk
// per SM).  Per step: pivot = Top2 over the per-warp candidates recorded by the previous
// trailing update (merged by every thread in the same order); warp 0 swaps and builds the
// reflector; barrier; trailing update; barrier.
constexpr int CQ_TPR = 8;
__host__ __device__ inline int cq_ld(int d) { return ((d + 7) / 8) * 8 + (((d + 7) / 8) % 2 == 0 ? 8 : 0); }

// E > 0 (round 2): a thread's E entries r = sub + 8 q of the reflector v and of the row being
// updated are held in registers for the step (the row is read once and written once instead of
// read twice and written once, v is read once per step instead of twice per row); the same
// operations in the same order as E = 0, so the factorisation is bitwise unchanged.
// HYB (global-panel variant only, round 2): once the ACTIVE part of the panel (rows i.., columns
// i..) fits the dynamic shared memory, it is moved there (rows of later pivots swap their retired
// columns < i0 in W) and the factorisation continues in shared memory; copied back at the end.
// Same operations in the same order: bitwise the all-global factorisation.
template <bool SMEM, int CQ_THREADS, int E = 0, bool HYB = false>
__global__ void __launch_bounds__(CQ_THREADS) cpqr_kernel(CpqrArgs a) {
  constexpr int CQ_WARPS = CQ_THREADS / 32;
  constexpr int RPP = CQ_THREADS / CQ_TPR;      // rows per pass
  extern __shared__ double smem[];
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c];
  const int d = a.d;
  const int LD = SMEM ? cq_ld(d) : d;
  double* v = smem;                       // d
  double* nrm = v + d;                    // m
  int* perm = (int*)(nrm + a.max_m);      // m
  double* spanel = nrm + a.max_m + (a.max_m + 1) / 2;   // m*LD (SMEM variant)
  __shared__ Top2 red[CQ_WARPS];
  __shared__ double s_tau;
  __shared__ int s_abort;   // the level-failure flag as polled by thread 0 in the previous step
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = threadIdx.x & (CQ_TPR - 1), rloc = threadIdx.x / CQ_TPR;
  const int64_t off = a.poff[c];
  double* A = SMEM ? spanel : a.W + off * d;
  // element (j, r) of the work panel at rowp(j)[r], r >= ro: before a HYB switch the panel itself
  // (ro = 0), after it the shared-memory copy of rows / columns >= ro
  double* Ab = A;
  int64_t LDa = LD;
  int ro = 0;
  auto rowp = [&](int j) { return Ab + (int64_t)(j - ro) * LDa - ro; };
  uint32_t dyn_bytes = 0;
  if constexpr (HYB) asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_bytes));
  const int64_t hyb_cap = HYB ? (int64_t)(dyn_bytes / 8) - (int64_t)(spanel - smem) : 0;   // doubles
  if (a.fail_flag) {   // the level already failed (CpqrArgs::fail_cap): skip the discarded panel
    if (threadIdx.x == 0) s_abort = *reinterpret_cast<volatile int*>(a.fail_flag);
    __syncthreads();
    if (s_abort) {
      if (threadIdx.x == 0) a.k[c] = 0;
      return;
    }
  }
  // copy panel rows (Y^loc rows) into the work panel
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += CQ_THREADS) {
    const int64_t j = e / d;
    A[j * LD + (e - j * d)] = a.Y[(off + j) * a.ldy + (e - j * d)];
  }
  for (int j = threadIdx.x; j < m; j += CQ_THREADS) perm[j] = j;
  if (threadIdx.x == 0) s_abort = 0;
  __syncthreads();
  auto row_sum = [&](double x) {   // sum over the 8 threads of a row (fixed order)
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    return x;
  };
  auto warp_best = [&](Top2 t) {    // Top2 over the 4 rows of a warp (lanes of a row agree)
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      Top2 u;
      u.v = __shfl_xor_sync(0xffffffffu, t.v, o);
      u.i = __shfl_xor_sync(0xffffffffu, t.i, o);
      u.s = __shfl_xor_sync(0xffffffffu, t.s, o);
      t = top2_merge(t, u);
    }
    return t;
  };
  {
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    for (int j0 = 0; j0 < m; j0 += RPP) {
      const int j = j0 + rloc;
      double q = 0.0;
      if (j < m)
        for (int r = sub; r < d; r += CQ_TPR) q = fma(A[(int64_t)j * LD + r], A[(int64_t)j * LD + r], q);
      q = row_sum(q);
      if (j < m) {
        const double nj = sqrt(q);
        if (sub == 0) nrm[j] = nj;
        loc = top2_merge(loc, Top2{nj, j, -1.0});
      }
    }
    loc = warp_best(loc);
    if (lane == 0) red[warp] = loc;
  }
  __syncthreads();
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  double min_gap = INFINITY, margin = INFINITY;
  int k = 0;
  bool aborted = false;
  // -DH2_CQ_PROF: cycles per pivot step by phase (clock64), printed for two CTAs
#ifdef H2_CQ_PROF
  long long pr[6] = {0, 0, 0, 0, 0, 0}, tp0 = 0, tp1 = 0;
#define CQP(n) do { tp1 = clock64(); pr[n] += tp1 - tp0; tp0 = tp1; } while (0)
  tp0 = clock64();
#else
#define CQP(n) do { } while (0)
#endif
  for (int i = 0;; ++i) {
    if constexpr (HYB) {
      // all threads passed the previous step's final barrier: move the active part if it fits
      if (ro == 0 && i > 0 && i < m && i < d && (int64_t)(m - i) * cq_ld(d - i) <= hyb_cap) {
        const int LDs = cq_ld(d - i), w = d - i;
        for (int64_t e = threadIdx.x; e < (int64_t)(m - i) * w; e += CQ_THREADS) {
          const int64_t j = e / w;
          spanel[j * LDs + (e - j * w)] = A[(i + j) * (int64_t)LD + i + (e - j * w)];
        }
        __syncthreads();
        Ab = spanel;
        LDa = LDs;
        ro = i;
      }
    }
    // every warp merges the per-warp candidates with one butterfly (same result in all threads)
    Top2 t = lane < CQ_WARPS ? red[lane] : Top2{-1.0, 0x7fffffff, -1.0};
    t = warp_top2(t);
    CQP(0);   // pivot merge
    if (i >= m) break;
    // truncation margin of every decision taken (R13); no decision exists at i = min(d, m)
    // certificates (R13): one thread of the LAST warp (off warp 0's reflector path)
    const bool certthr = threadIdx.x == CQ_THREADS - 32;
    if (certthr && a.eps > 0 && i < kfull) margin = fmin(margin, fabs(t.v - a.eps) / a.eps);
    if (i == kcap || !(t.v > a.eps)) {
      k = i;
      break;
    }
    if (a.fail_flag) {   // adaptive early exit (CpqrArgs::fail_cap): uniform decisions
      if (i == a.fail_cap && m > d) {
        if (threadIdx.x == 0) atomicExch(a.fail_flag, 1);
        k = a.fail_k;
        aborted = true;
        break;
      }
      if (s_abort) {
        k = i;
        aborted = true;
        break;
      }
    }
    if (certthr && t.s >= 0) min_gap = fmin(min_gap, (t.v - t.s) / t.v);
    const int p = t.i;
    double* Ai = rowp(i);
    if (warp == 0) {
      // ---- swap rows i and p of the panel (columns of A)
      if (p != i) {
        double* Ap = rowp(p);
        for (int r = ro + lane; r < d; r += 32) {
          const double x = Ai[r];
          Ai[r] = Ap[r];
          Ap[r] = x;
        }
        if (HYB && ro > 0) {   // their retired columns < ro stay in the panel in W
          double* Gi = A + (int64_t)i * LD;
          double* Gp = A + (int64_t)p * LD;
          for (int r = lane; r < ro; r += 32) {
            const double x = Gi[r];
            Gi[r] = Gp[r];
            Gp[r] = x;
          }
        }
        if (lane == 0) {
          const int q = perm[i];
          perm[i] = perm[p];
          perm[p] = q;
          const double x = nrm[i];
          nrm[i] = nrm[p];
          nrm[p] = x;
        }
        __syncwarp();
      }
      // ---- Householder reflector of A(i:d, i), LAPACK dlarfg convention
      double x2 = 0.0;
      for (int r = i + 1 + lane; r < d; r += 32) x2 = fma(Ai[r], Ai[r], x2);
      x2 = warp_sum(x2);
      const double alpha = Ai[i];
      const double xnorm = sqrt(x2);
      double tau, beta;
      if (xnorm == 0.0) {
        tau = 0.0;
        beta = alpha;
      } else {
        const double h = hypot(alpha, xnorm);
        beta = alpha != 0.0 ? -copysign(h, alpha) : -h;
        tau = (beta - alpha) / beta;
      }
      const double den = alpha - beta;
      __syncwarp();
      // v = x / (alpha - beta): one reciprocal and d multiplications (LAPACK dlarfg scales x by
      // 1 / (alpha - beta) the same way) instead of d FP64 divisions on warp 0's serial path
      const double rden = 1.0 / den;
      for (int r = i + 1 + lane; r < d; r += 32) {
        v[r] = tau != 0.0 ? Ai[r] * rden : 0.0;
        Ai[r] = 0.0;
      }
      if (lane == 0) {
        v[i] = 1.0;
        Ai[i] = beta;
        s_tau = tau;
      }
    }
    CQP(1);   // warp 0: swap + reflector (other warps: arrive)
    __syncthreads();
    CQP(2);   // barrier 1
    const double tau = s_tau;
    // poll the level-failure flag (read by thread 0 now, acted on after the next merge)
    int fl = 0;
    if (a.fail_flag && threadIdx.x == 0) fl = *reinterpret_cast<volatile int*>(a.fail_flag);
    // ---- trailing update of rows j > i (columns of A) + next residual norms + local pivot
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    const int r0 = i + ((sub - i) & (CQ_TPR - 1));   // first r >= i with r = sub mod 8
    if constexpr (E > 0) {
      double vq[E];
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const int r = sub + CQ_TPR * q;
        vq[q] = (r >= r0 && r < d) ? v[r] : 0.0;
      }
      for (int j0 = i + 1; j0 < m; j0 += RPP) {
        const int j = j0 + rloc;
        const bool act = j < m;
        double* Aj = A + (int64_t)(act ? j : i) * LD;
        double x[E];
        double w = 0.0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int r = sub + CQ_TPR * q;
          const bool in = act && r >= r0 && r < d;
          x[q] = in ? Aj[r] : 0.0;
          if (in) w = fma(vq[q], x[q], w);
        }
        w = row_sum(w) * tau;
        double qn = 0.0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int r = sub + CQ_TPR * q;
          if (act && r >= r0 && r < d) {
            const double xx = fma(-w, vq[q], x[q]);
            Aj[r] = xx;
            if (r > i) qn = fma(xx, xx, qn);
          }
        }
        qn = row_sum(qn);
        if (act) {
          const double nj = sqrt(qn);
          if (sub == 0) nrm[j] = nj;
          loc = top2_merge(loc, Top2{nj, j, -1.0});
        }
      }
    } else
    for (int j0 = i + 1; j0 < m; j0 += RPP) {
      const int j = j0 + rloc;
      const bool act = j < m;
      double* Aj = rowp(act ? j : i);
      double w = 0.0;
      if (act)
        for (int r = r0; r < d; r += CQ_TPR) w = fma(v[r], Aj[r], w);
      w = row_sum(w) * tau;
      double q = 0.0;
      if (act)
        for (int r = r0; r < d; r += CQ_TPR) {
          const double x = fma(-w, v[r], Aj[r]);
          Aj[r] = x;
          if (r > i) q = fma(x, x, q);
        }
      q = row_sum(q);
      if (act) {
        const double nj = sqrt(q);
        if (sub == 0) nrm[j] = nj;
        loc = top2_merge(loc, Top2{nj, j, -1.0});
      }
    }
    loc = warp_best(loc);
    if (lane == 0) red[warp] = loc;
    if (a.fail_flag && threadIdx.x == 0) s_abort = fl;
    CQP(3);   // trailing update + local pivot
    __syncthreads();
    CQP(4);   // barrier 2
    k = i + 1;
  }
#ifdef H2_CQ_PROF
  if ((threadIdx.x == 0 || threadIdx.x == 32 * (CQ_WARPS - 1)) && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2))
    printf("[cq prof] blk %d thr %d m %d d %d k %d | merge %lld refl %lld bar1 %lld upd %lld bar2 %lld (cycles/step %lld)\n",
           blockIdx.x, threadIdx.x, m, d, k, pr[0] / max(k, 1), pr[1] / max(k, 1), pr[2] / max(k, 1), pr[3] / max(k, 1),
           pr[4] / max(k, 1), (pr[0] + pr[1] + pr[2] + pr[3] + pr[4]) / max(k, 1));
#endif
#undef CQP
  __syncthreads();
  if (aborted) {   // this round is discarded by the host (the level failed): only k is read
    if (threadIdx.x == 0) a.k[c] = k;
    return;
  }
  if (HYB && ro > 0) {   // the shared-memory part back into the panel in W
    const int w = d - ro;
    for (int64_t e = threadIdx.x; e < (int64_t)(m - ro) * w; e += CQ_THREADS) {
      const int64_t j = e / w;
      A[(ro + j) * (int64_t)LD + ro + (e - j * w)] = spanel[j * LDa + (e - j * w)];
    }
  }
  for (int j = threadIdx.x; j < m; j += CQ_THREADS) a.perm[off + j] = perm[j];
  if (SMEM) {
    double* Wc = a.W + off * d;
    for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += CQ_THREADS) {
      const int64_t j = e / d;
      Wc[e] = A[j * LD + (e - j * d)];
    }
  }
  if (threadIdx.x == 0) a.k[c] = k;
  if (threadIdx.x == CQ_THREADS - 32) {
    a.cert[2 * c] = min_gap;
    a.cert[2 * c + 1] = margin;
  }
}

__host__ __device__ inline size_t cq1_head_doubles(int max_m) { return ((size_t)max_m * 5 + 15) / 16 * 2; }

// One barrier per pivot step (round 2).  Panel rows are never swapped: a pivot row is retired in
// place (its R column is final: entries < i were fixed by earlier reflectors, entry i becomes
// beta one step later, when nobody reads it any more), and the factored panel is written to W in
// pivot order at the end (position q <- row perm[q]; redundant rows in ascending row order).
// Every warp rebuilds the reflector of the pivot row redundantly (same data, same order: the same
// bits in every warp), so no second barrier publishes it: per step one __syncthreads separates
// the trailing update (rows j: w = tau (A(j,i) + <A(p,i+1:), A(j,i+1:)> / den), A(j,i) -= w,
// A(j,r) -= (w / den) A(p,r), next norm from the updated entries, local Top2) from the merge of
// the per-warp pivot candidates.  Decisions as R12-R14 (max recomputed norm, ties -> lowest row,
// dlarfg signs), the certificates as before.  SMEM: panel in shared memory; else in `scratch`
// (global, L1/L2 resident), gathered into W at the end.
template <bool SMEM, int NT>
__global__ void __launch_bounds__(NT) cpqr1_kernel(CpqrArgs a, double* __restrict__ scratch) {
  constexpr int NW = NT / 32;
  constexpr int RPP = NT / CQ_TPR;
  extern __shared__ double smem[];
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c];
  const int d = a.d;
  const int LD = SMEM ? cq_ld(d) : d;
  int* perm = reinterpret_cast<int*>(smem);                          // max_m
  unsigned char* retired = reinterpret_cast<unsigned char*>(perm + a.max_m);
  double* spanel = smem + cq1_head_doubles(a.max_m);                 // after perm + retired
  // per-warp pivot candidates, double buffered by step parity: a fast warp publishing step i's
  // candidates never overwrites the ones a slow warp is still merging from step i - 1
  __shared__ Top2 red2[2][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = threadIdx.x & (CQ_TPR - 1), rloc = threadIdx.x / CQ_TPR;
  const int64_t off = a.poff[c];
  double* A = SMEM ? spanel : scratch + off * d;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += NT) {
    const int64_t j = e / d;
    A[j * LD + (e - j * d)] = a.Y[(off + j) * a.ldy + (e - j * d)];
  }
  for (int j = threadIdx.x; j < m; j += NT) retired[j] = 0;
  __syncthreads();
  auto row_sum = [&](double x) {
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    return x;
  };
  auto warp_best = [&](Top2 t) {
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      Top2 u;
      u.v = __shfl_xor_sync(0xffffffffu, t.v, o);
      u.i = __shfl_xor_sync(0xffffffffu, t.i, o);
      u.s = __shfl_xor_sync(0xffffffffu, t.s, o);
      t = top2_merge(t, u);
    }
    return t;
  };
  {
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    for (int j0 = 0; j0 < m; j0 += RPP) {
      const int j = j0 + rloc;
      double q = 0.0;
      if (j < m)
        for (int r = sub; r < d; r += CQ_TPR) q = fma(A[(int64_t)j * LD + r], A[(int64_t)j * LD + r], q);
      q = row_sum(q);
      if (j < m) loc = top2_merge(loc, Top2{sqrt(q), j, -1.0});
    }
    loc = warp_best(loc);
    if (lane == 0) red2[0][warp] = loc;
  }
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  double min_gap = INFINITY, margin = INFINITY;
  int k = 0, p_prev = -1;
  double beta_prev = 0.0;
  for (int i = 0;; ++i) {
    __syncthreads();
    if (threadIdx.x == 0 && p_prev >= 0) {   // the previous pivot's R diagonal; nobody reads it now
      A[(int64_t)p_prev * LD + (i - 1)] = beta_prev;
      retired[p_prev] = 1;
      perm[i - 1] = p_prev;
    }
    Top2 t = lane < NW ? red2[i & 1][lane] : Top2{-1.0, 0x7fffffff, -1.0};
    t = warp_top2(t);
    if (i >= m) break;
    if (a.eps > 0 && i < kfull) margin = fmin(margin, fabs(t.v - a.eps) / a.eps);
    if (i == kcap || !(t.v > a.eps)) {
      k = i;
      break;
    }
    if (t.s >= 0) min_gap = fmin(min_gap, (t.v - t.s) / t.v);
    const int p = t.i;
    const double* Ap = A + (int64_t)p * LD;
    // Householder reflector of the pivot column (LAPACK dlarfg), rebuilt by every warp
    double x2 = 0.0;
    for (int r = i + 1 + lane; r < d; r += 32) x2 = fma(Ap[r], Ap[r], x2);
    x2 = warp_sum(x2);
    const double alpha = Ap[i];
    const double xnorm = sqrt(x2);
    double tau, beta;
    if (xnorm == 0.0) {
      tau = 0.0;
      beta = alpha;
    } else {
      const double h = hypot(alpha, xnorm);
      beta = alpha != 0.0 ? -copysign(h, alpha) : -h;
      tau = (beta - alpha) / beta;
    }
    const double rden = 1.0 / (alpha - beta);
    // trailing update of the unretired rows (the pivot row p excluded) + next norms + local pivot
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    const int r0 = (i + 1) + ((sub - (i + 1)) & (CQ_TPR - 1));   // first r > i with r = sub mod 8
    for (int j0 = 0; j0 < m; j0 += RPP) {
      const int j = j0 + rloc;
      const bool act = j < m && j != p && j != p_prev && !retired[j];
      double* Aj = A + (int64_t)(act ? j : p) * LD;
      double s = 0.0, aji = 0.0;
      if (act) {
        aji = Aj[i];
        if (tau != 0.0)
          for (int r = r0; r < d; r += CQ_TPR) s = fma(Ap[r], Aj[r], s);
      }
      s = row_sum(s);
      __syncwarp();   // every lane of the row read A(j, i) before it is updated
      double q = 0.0;
      if (act) {
        if (tau != 0.0) {
          const double w = tau * fma(s, rden, aji);
          const double wd = w * rden;
          if (sub == 0) Aj[i] = aji - w;
          for (int r = r0; r < d; r += CQ_TPR) {
            const double x = fma(-wd, Ap[r], Aj[r]);
            Aj[r] = x;
            q = fma(x, x, q);
          }
        } else {
          for (int r = r0; r < d; r += CQ_TPR) q = fma(Aj[r], Aj[r], q);
        }
      }
      q = row_sum(q);
      if (act) loc = top2_merge(loc, Top2{sqrt(q), j, -1.0});
    }
    loc = warp_best(loc);
    if (lane == 0) red2[(i + 1) & 1][warp] = loc;
    p_prev = p;
    beta_prev = beta;
    k = i + 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int q = k;   // redundant rows after the pivots, ascending row index
    for (int j = 0; j < m; ++j)
      if (!retired[j]) perm[q++] = j;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += NT) a.perm[off + j] = perm[j];
  double* Wc = a.W + off * d;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += NT) {
    const int64_t q = e / d;
    Wc[e] = A[(int64_t)perm[q] * LD + (e - q * d)];
  }
  if (threadIdx.x == 0) {
    a.k[c] = k;
    a.cert[2 * c] = min_gap;
    a.cert[2 * c + 1] = margin;
  }
}

// cpqr2 (round 2, opt-in H2_CQ2=1): one barrier per pivot step and NO serial
// reflector warp.  profiles/r2_cpqr2.md: in cpqr_kernel 15 warps waited at a barrier (36 % of
// all stall samples) while warp 0 swapped the pivot row, reduced its norm and divided d entries
// by alpha - beta.  Here
//   * x2 = sum_{r > i} A(p, r)^2 of the next pivot is a by-product of the previous trailing update
//     (each row keeps S2_j = sum_{r >= i+2} x_r^2 beside its norm^2 = x_{i+1}^2 + S2_j), so every
//     warp derives the reflector scalars (alpha, beta, tau, 1/(alpha - beta)) redundantly in O(1)
//     from shared memory -- same data, same order, the same bits in every warp;
//   * rows are never swapped: the pivot row is retired in place (its R column is final except
//     R(i, i) = beta, written one step later when nobody reads the row), the active rows are a
//     list (double-buffered in shared memory; warp 0 writes the next step's list, the pivot
//     swap-removed, while every warp reads the current one), so the update loop visits only the
//     m - i - 1 active rows;
//   * v is never materialised: the update reads the pivot row and scales by 1/(alpha - beta)
//     (LAPACK dlarfg scales x by 1/(alpha - beta) too).
// Decisions as R12-R14 (max recomputed norm, ties -> lowest row index, dlarfg signs); the norms
// are recomputed from the updated entries every step (no downdating); certificates as before.
// The factored panel is written to W in pivot order, redundant rows in ascending row index.
__host__ __device__ inline size_t cq2_head_doubles(int max_m) {
  // x2s (max_m doubles) + lists (2 max_m int) + retired flags (max_m bytes), 16-byte aligned
  return (size_t)max_m + ((size_t)max_m * 9 + 15) / 16 * 2;
}

template <bool SMEM, int NT>
__global__ void __launch_bounds__(NT) cpqr2_kernel(CpqrArgs a, double* __restrict__ scratch) {
  constexpr int NW = NT / 32;
  constexpr int RPP = NT / CQ_TPR;
  extern __shared__ double smem[];
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c];
  const int d = a.d;
  const int LD = SMEM ? cq_ld(d) : d;
  double* x2s = smem;                                                 // max_m
  int* lst = reinterpret_cast<int*>(smem + a.max_m);                  // 2 x max_m
  unsigned char* retired = reinterpret_cast<unsigned char*>(lst + 2 * a.max_m);   // max_m
  double* spanel = smem + cq2_head_doubles(a.max_m);
  __shared__ Top2 red2[2][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = threadIdx.x & (CQ_TPR - 1), rloc = threadIdx.x / CQ_TPR;
  const int64_t off = a.poff[c];
  int* gperm = a.perm + off;
  double* A = SMEM ? spanel : scratch + off * d;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += NT) {
    const int64_t j = e / d;
    A[j * LD + (e - j * d)] = a.Y[(off + j) * a.ldy + (e - j * d)];
  }
  for (int j = threadIdx.x; j < m; j += NT) {
    lst[j] = j;
    retired[j] = 0;
  }
  __syncthreads();
  auto row_sum = [&](double x) {
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    return x;
  };
  auto warp_best = [&](Top2 t) {
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      Top2 u;
      u.v = __shfl_xor_sync(0xffffffffu, t.v, o);
      u.i = __shfl_xor_sync(0xffffffffu, t.i, o);
      u.s = __shfl_xor_sync(0xffffffffu, t.s, o);
      t = top2_merge(t, u);
    }
    return t;
  };
  {
    // initial norms over r >= 0 and S2 over r >= 1
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    for (int j0 = 0; j0 < m; j0 += RPP) {
      const int j = j0 + rloc;
      double s2 = 0.0, x0 = 0.0;
      if (j < m) {
        for (int r = sub; r < d; r += CQ_TPR) {
          const double x = A[(int64_t)j * LD + r];
          if (r == 0) x0 = x;
          else s2 = fma(x, x, s2);
        }
      }
      s2 = row_sum(s2);
      x0 = row_sum(x0);
      if (j < m) {
        if (sub == 0) x2s[j] = s2;
        loc = top2_merge(loc, Top2{sqrt(fma(x0, x0, s2)), j, -1.0});
      }
    }
    loc = warp_best(loc);
    if (lane == 0) red2[0][warp] = loc;
  }
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  double min_gap = INFINITY, margin = INFINITY;
  int k = 0, p_prev = -1;
  double beta_prev = 0.0;
  for (int i = 0;; ++i) {
    __syncthreads();
    if (p_prev >= 0) {   // finalize the previous pivot row: R(i-1, i-1) = beta, zeros below
      double* Aq = A + (int64_t)p_prev * LD;
      for (int r = i + threadIdx.x; r < d; r += NT) Aq[r] = 0.0;
      if (threadIdx.x == 0) {
        Aq[i - 1] = beta_prev;
        retired[p_prev] = 1;
        gperm[i - 1] = p_prev;
      }
    }
    Top2 t = lane < NW ? red2[i & 1][lane] : Top2{-1.0, 0x7fffffff, -1.0};
    t = warp_top2(t);
    if (i >= m) break;
    if (a.eps > 0 && i < kfull) margin = fmin(margin, fabs(t.v - a.eps) / a.eps);
    if (i == kcap || !(t.v > a.eps)) {
      k = i;
      break;
    }
    if (t.s >= 0) min_gap = fmin(min_gap, (t.v - t.s) / t.v);
    const int p = t.i;
    const double* Ap = A + (int64_t)p * LD;
    // Householder reflector of the pivot column (LAPACK dlarfg) from shared scalars
    const double alpha = Ap[i];
    const double x2 = x2s[p];
    const double xnorm = sqrt(x2);
    double tau, beta;
    if (xnorm == 0.0) {
      tau = 0.0;
      beta = alpha;
    } else {
      const double h = hypot(alpha, xnorm);
      beta = alpha != 0.0 ? -copysign(h, alpha) : -h;
      tau = (beta - alpha) / beta;
    }
    const double rden = 1.0 / (alpha - beta);
    const int cnt = m - i;                       // active rows (incl. p) in lst[i & 1]
    const int* L = lst + (i & 1) * a.max_m;
    if (warp == 0) {                             // next step's list: p swap-removed
      int* Ln = lst + ((i + 1) & 1) * a.max_m;
      const int last = L[cnt - 1];
      for (int q = lane; q < cnt - 1; q += 32) {
        const int v = L[q];
        Ln[q] = v == p ? last : v;
      }
    }
    // trailing update of the active rows (p excluded) + next norms, S2 and local pivot
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    const int r0 = (i + 1) + ((sub - (i + 1)) & (CQ_TPR - 1));   // first r > i with r = sub mod 8
    for (int q0 = 0; q0 < cnt; q0 += RPP) {
      const int q = q0 + rloc;
      const int j = q < cnt ? L[q] : p;
      const bool act = j != p;
      double* Aj = A + (int64_t)j * LD;
      double s = 0.0, aji = 0.0;
      if (act) {
        aji = Aj[i];
        if (tau != 0.0)
          for (int r = r0; r < d; r += CQ_TPR) s = fma(Ap[r], Aj[r], s);
      }
      s = row_sum(s);
      __syncwarp();   // every lane of the row read A(j, i) before it is updated
      double s2 = 0.0, x1 = 0.0;
      if (act) {
        if (tau != 0.0) {
          const double w = tau * fma(s, rden, aji);
          const double wd = w * rden;
          if (sub == 0) Aj[i] = aji - w;
          for (int r = r0; r < d; r += CQ_TPR) {
            const double x = fma(-wd, Ap[r], Aj[r]);
            Aj[r] = x;
            if (r == i + 1) x1 = x;
            else s2 = fma(x, x, s2);
          }
        } else {
          for (int r = r0; r < d; r += CQ_TPR) {
            const double x = Aj[r];
            if (r == i + 1) x1 = x;
            else s2 = fma(x, x, s2);
          }
        }
      }
      s2 = row_sum(s2);
      x1 = row_sum(x1);   // one owner, exact zeros elsewhere
      if (act) {
        if (sub == 0) x2s[j] = s2;
        loc = top2_merge(loc, Top2{sqrt(fma(x1, x1, s2)), j, -1.0});
      }
    }
    loc = warp_best(loc);
    if (lane == 0) red2[(i + 1) & 1][warp] = loc;
    p_prev = p;
    beta_prev = beta;
    k = i + 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int q = k;   // redundant rows after the pivots, ascending row index
    for (int j = 0; j < m; ++j)
      if (!retired[j]) gperm[q++] = j;
  }
  __syncthreads();
  double* Wc = a.W + off * d;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += NT) {
    const int64_t q = e / d;
    Wc[e] = A[(int64_t)gperm[q] * LD + (e - q * d)];
  }
  if (threadIdx.x == 0) {
    a.k[c] = k;
    a.cert[2 * c] = min_gap;
    a.cert[2 * c + 1] = margin;
  }
}

template <bool SMEM, int NT>
static void cpqr2_launch(const CpqrArgs& a, size_t sm, double* scratch, cudaStream_t st) {
  H2_CUDA(cudaFuncSetAttribute(cpqr2_kernel<SMEM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cpqr2_kernel<SMEM, NT><<<a.nclusters, NT, sm, st>>>(a, scratch);
}

template <bool SMEM, int NT>
static void cpqr1_launch(const CpqrArgs& a, size_t sm, double* scratch, cudaStream_t st) {
  H2_CUDA(cudaFuncSetAttribute(cpqr1_kernel<SMEM, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cpqr1_kernel<SMEM, NT><<<a.nclusters, NT, sm, st>>>(a, scratch);
}

template <bool SMEM, int NT, int E = 0, bool HYB = false>
static void cpqr_launch_e(const CpqrArgs& a, size_t sm, cudaStream_t st) {
  if (sm > 48 * 1024)
    H2_CUDA(cudaFuncSetAttribute(cpqr_kernel<SMEM, NT, E, HYB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cpqr_kernel<SMEM, NT, E, HYB><<<a.nclusters, NT, sm, st>>>(a);
}

// register-cached variant when every thread's entries fit E (d <= 8 E): on every level
// (H2_CQ_REG=1) measured slower at C2 (33.5 vs 30.4 ms: 128 registers x 512 threads leave one
// CTA per SM on the global-panel levels, which ran two); on the levels with at most one panel
// per SM only (default) slightly faster
template <bool SMEM, int NT>
static void cpqr_launch(const CpqrArgs& a, size_t sm, cudaStream_t st) {
  // H2_CQ_REG: 0 off, 1 every block panel, 2 shared-memory panels only (one CTA per SM there
  // anyway, so the 128 registers cost no occupancy)
  // 3: global-panel levels with at most one panel per SM (the L2-latency-bound upper levels:
  // all E row loads of a pass in flight at once); 4: 2 + 3
  const int regm = env_int("H2_CQ_REG", 3);   // default 3: 29.4 vs 30.0 ms at C2 (bitwise)
  const bool few = !SMEM && a.nclusters <= 148;
  const bool reg = regm == 1 || (regm == 2 && SMEM) || (regm == 3 && few) || (regm == 4 && (SMEM || few));
  const int need = (a.d + CQ_TPR - 1) / CQ_TPR;
  if (reg && need <= 8) cpqr_launch_e<SMEM, NT, 8>(a, sm, st);
  else if (reg && need <= 16) cpqr_launch_e<SMEM, NT, 16>(a, sm, st);
  else if (reg && need <= 20) cpqr_launch_e<SMEM, NT, 20>(a, sm, st);
  else if (reg && need <= 24) cpqr_launch_e<SMEM, NT, 24>(a, sm, st);
  else cpqr_launch_e<SMEM, NT, 0>(a, sm, st);
}

// Small panels (m <= 64 rows, the leaf level): one WARP per panel, 4 panels per CTA, no block
// barriers.  Lane l owns panel rows l and l + 32 (row-major in shared memory, odd row stride:
// conflict-free column walks); the pivot is a warp Top2 butterfly, the reflector is built by
// the whole warp, the trailing update of a row is a sequential dot / update / norm over its
// columns (two accumulators).  Same decisions as the block kernel (max recomputed norm, ties ->
// lowest index, LAPACK dlarfg), same certificates.
constexpr int CW_WPB = 4;
__host__ __device__ inline int cw_ld(int d) { return d | 1; }
__host__ __device__ inline size_t cw_warp_doubles(int d) { return (size_t)64 * cw_ld(d) + d + 64 + 32; }

__global__ void __launch_bounds__(32 * CW_WPB) cpqr_warp_kernel(CpqrArgs a) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ci = blockIdx.x * CW_WPB + warp;
  if (ci >= a.nclusters) return;
  const int c = a.c_begin + ci;
  const int m = a.m[c], d = a.d, LD = cw_ld(d);
  double* A = smem + (size_t)warp * cw_warp_doubles(d);
  double* v = A + (size_t)64 * LD;
  double* nrm = v + d;
  int* perm = reinterpret_cast<int*>(nrm + 64);
  const int64_t off = a.poff[c];
  if (a.fail_flag && __shfl_sync(0xffffffffu, lane == 0 ? *reinterpret_cast<volatile int*>(a.fail_flag) : 0, 0)) {
    if (lane == 0) a.k[c] = 0;   // the level already failed: skip the discarded panel
    return;
  }
  for (int j = 0; j < m; ++j)
    for (int r = lane; r < d; r += 32) A[j * LD + r] = a.Y[(off + j) * a.ldy + r];
  __syncwarp();
  for (int q = 0; q < 2; ++q) {
    const int j = lane + 32 * q;
    if (j < m) {
      double s0 = 0.0, s1 = 0.0;
      int r = 0;
      for (; r + 1 < d; r += 2) {
        s0 = fma(A[j * LD + r], A[j * LD + r], s0);
        s1 = fma(A[j * LD + r + 1], A[j * LD + r + 1], s1);
      }
      if (r < d) s0 = fma(A[j * LD + r], A[j * LD + r], s0);
      nrm[j] = sqrt(s0 + s1);
      perm[j] = j;
    }
  }
  __syncwarp();
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  double min_gap = INFINITY, margin = INFINITY;
  int k = 0;
  bool aborted = false;
  int fl = 0;   // level-failure flag polled by lane 0 in the previous step
  for (int i = 0;; ++i) {
    Top2 t{-1.0, 0x7fffffff, -1.0};
    for (int q = 0; q < 2; ++q) {
      const int j = lane + 32 * q;
      if (j >= i && j < m) t = top2_merge(t, Top2{nrm[j], j, -1.0});
    }
    t = warp_top2(t);
    if (i >= m) break;
    if (a.eps > 0 && i < kfull) margin = fmin(margin, fabs(t.v - a.eps) / a.eps);
    if (i == kcap || !(t.v > a.eps)) {
      k = i;
      break;
    }
    if (a.fail_flag) {   // adaptive early exit (CpqrArgs::fail_cap)
      if (i == a.fail_cap && m > d) {
        if (lane == 0) atomicExch(a.fail_flag, 1);
        k = a.fail_k;
        aborted = true;
        break;
      }
      if (__shfl_sync(0xffffffffu, fl, 0)) {
        k = i;
        aborted = true;
        break;
      }
      if (lane == 0) fl = *reinterpret_cast<volatile int*>(a.fail_flag);
    }
    if (t.s >= 0) min_gap = fmin(min_gap, (t.v - t.s) / t.v);
    const int p = t.i;
    double* Ai = A + i * LD;
    if (p != i) {
      double* Ap = A + p * LD;
      for (int r = lane; r < d; r += 32) {
        const double x = Ai[r];
        Ai[r] = Ap[r];
        Ap[r] = x;
      }
      if (lane == 0) {
        const int q = perm[i];
        perm[i] = perm[p];
        perm[p] = q;
        const double x = nrm[i];
        nrm[i] = nrm[p];
        nrm[p] = x;
      }
      __syncwarp();
    }
    // Householder reflector of A(i:d, i), LAPACK dlarfg convention
    double x2 = 0.0;
    for (int r = i + 1 + lane; r < d; r += 32) x2 = fma(Ai[r], Ai[r], x2);
    x2 = warp_sum(x2);
    const double alpha = Ai[i];
    const double xnorm = sqrt(x2);
    double tau, beta;
    if (xnorm == 0.0) {
      tau = 0.0;
      beta = alpha;
    } else {
      const double h = hypot(alpha, xnorm);
      beta = alpha != 0.0 ? -copysign(h, alpha) : -h;
      tau = (beta - alpha) / beta;
    }
    const double den = alpha - beta;
    __syncwarp();
    const double rden = 1.0 / den;   // dlarfg: x scaled by 1 / (alpha - beta)
    for (int r = i + 1 + lane; r < d; r += 32) {
      v[r] = tau != 0.0 ? Ai[r] * rden : 0.0;
      Ai[r] = 0.0;
    }
    if (lane == 0) {
      v[i] = 1.0;
      Ai[i] = beta;
    }
    __syncwarp();
    // trailing update of this lane's rows j > i + next residual norms
    for (int q = 0; q < 2; ++q) {
      const int j = lane + 32 * q;
      if (j <= i || j >= m) continue;
      double* Aj = A + j * LD;
      double w0 = 0.0, w1 = 0.0;
      int r = i;
      for (; r + 1 < d; r += 2) {
        w0 = fma(v[r], Aj[r], w0);
        w1 = fma(v[r + 1], Aj[r + 1], w1);
      }
      if (r < d) w0 = fma(v[r], Aj[r], w0);
      const double w = (w0 + w1) * tau;
      double q0 = 0.0, q1 = 0.0;
      Aj[i] = fma(-w, v[i], Aj[i]);
      for (r = i + 1; r + 1 < d; r += 2) {
        const double x0 = fma(-w, v[r], Aj[r]);
        const double x1 = fma(-w, v[r + 1], Aj[r + 1]);
        Aj[r] = x0;
        Aj[r + 1] = x1;
        q0 = fma(x0, x0, q0);
        q1 = fma(x1, x1, q1);
      }
      if (r < d) {
        const double x0 = fma(-w, v[r], Aj[r]);
        Aj[r] = x0;
        q0 = fma(x0, x0, q0);
      }
      nrm[j] = sqrt(q0 + q1);
    }
    __syncwarp();
    k = i + 1;
  }
  __syncwarp();
  if (aborted) {   // this round is discarded by the host (the level failed): only k is read
    if (lane == 0) a.k[c] = k;
    return;
  }
  for (int j = lane; j < m; j += 32) a.perm[off + j] = perm[j];
  double* Wc = a.W + off * d;
  for (int j = 0; j < m; ++j)
    for (int r = lane; r < d; r += 32) Wc[(int64_t)j * d + r] = A[j * LD + r];
  if (lane == 0) {
    a.k[c] = k;
    a.cert[2 * c] = min_gap;
    a.cert[2 * c + 1] = margin;
  }
}

// ------------------------------------------------------------------------------------------
// CTA-cluster CPQR (round 2) for panels too large for one CTA's shared memory (m * d at the
// upper depths: 180-240 rows x 160 samples = 230-320 KB), which the one-CTA kernel otherwise
// streams from global memory every pivot step (L2-latency bound: 18-33 k cycles per step).
// One cluster of CL CTAs per panel: panel row j lives in CTA j % CL (local row j / CL) in shared
// memory, so each CTA updates 1/CL of the rows.  Rows never move: a pivot row is retired in
// place and the positions are tracked (pos[row], rowat[position], replicated in every CTA), so
// each row's arithmetic is exactly the one-CTA kernel's (same 8-thread row split, same fixed-order
// reductions, same dlarfg reflector) and the pivot candidates carry (position << 16 | row): ties
// go to the lowest POSITION as in the row-swapping kernels.  The result is bitwise theirs.
// Per step: (A) cluster barrier -> every warp merges the NW x CL candidates (one per lane) ->
// the owner CTA's warp 0 builds the reflector from its local pivot row and writes v, tau into
// every CTA (distributed shared memory); thread 0 of every CTA swaps the two positions;
// (B) cluster barrier -> trailing update of the local active rows (position > i), next norms,
// per-warp candidates written into every CTA.  Early exit (CpqrArgs::fail_cap) as the one-CTA
// kernel, with the polled flag broadcast by CTA 0 so that every CTA of the cluster decides alike.
// ------------------------------------------------------------------------------------------
namespace cgx = cooperative_groups;
__host__ __device__ inline size_t cqc_head_bytes(int d, int max_m) {
  return (((size_t)d * 8 + 32 * 8 * 2 + 32 * 4 + (size_t)max_m * 8 + 8) + 127) / 128 * 128;
}
template <int CL, int NT>
__global__ void __launch_bounds__(NT) cpqr_cluster_kernel(CpqrArgs a) {
  constexpr int NW = NT / 32;
  static_assert(NW * CL <= 32, "one pivot candidate per lane of the merge");
  constexpr int RPP = NT / CQ_TPR;
  cgx::cluster_group cl = cgx::this_cluster();
  const int crank = (int)cl.block_rank();
  const int c = a.c_begin + blockIdx.x / CL;
  const int m = a.m[c], d = a.d, LD = cq_ld(d);
  const int mloc = (m - crank + CL - 1) / CL;
  extern __shared__ __align__(128) unsigned char cq_smem[];
  double* v = reinterpret_cast<double*>(cq_smem);          // d
  double* cv = v + d;                                      // 32 candidate values
  double* cs = cv + 32;                                    // 32 second-best values
  int* ci = reinterpret_cast<int*>(cs + 32);               // 32 packed indices
  int* pos = ci + 32;                                      // max_m
  int* rowat = pos + a.max_m;                              // max_m
  double* P = reinterpret_cast<double*>(cq_smem + cqc_head_bytes(d, a.max_m));   // mloc x LD
  __shared__ double s_tau;
  __shared__ int s_abort;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = tid & (CQ_TPR - 1), rloc = tid / CQ_TPR;
  const int64_t off = a.poff[c];
  double* vr[CL];
  double* cvr[CL];
  double* csr[CL];
  int* cir[CL];
  double* taur[CL];
  int* abr[CL];
#pragma unroll
  for (int q = 0; q < CL; ++q) {
    vr[q] = cl.map_shared_rank(v, q);
    cvr[q] = cl.map_shared_rank(cv, q);
    csr[q] = cl.map_shared_rank(cs, q);
    cir[q] = cl.map_shared_rank(ci, q);
    taur[q] = cl.map_shared_rank(&s_tau, q);
    abr[q] = cl.map_shared_rank(&s_abort, q);
  }
  if (tid == 0) s_abort = 0;
  cl.sync();   // every CTA of the cluster runs before any distributed shared memory access
  if (a.fail_flag) {   // the level already failed: skip the discarded panel (cluster-uniform)
    if (crank == 0 && tid == 0) {
      const int f = *reinterpret_cast<volatile int*>(a.fail_flag);
#pragma unroll
      for (int q = 0; q < CL; ++q) *abr[q] = f;
    }
    cl.sync();
    if (s_abort) {
      if (crank == 0 && tid == 0) a.k[c] = 0;
      return;
    }
  }
  for (int64_t e = tid; e < (int64_t)mloc * d; e += NT) {
    const int64_t jl = e / d;
    P[jl * LD + (e - jl * d)] = a.Y[(off + crank + CL * jl) * a.ldy + (e - jl * d)];
  }
  for (int j = tid; j < m; j += NT) {
    pos[j] = j;
    rowat[j] = j;
  }
  __syncthreads();
  auto row_sum = [&](double x) {
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 4);
    return x;
  };
  auto warp_best = [&](Top2 t) {
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      Top2 u;
      u.v = __shfl_xor_sync(0xffffffffu, t.v, o);
      u.i = __shfl_xor_sync(0xffffffffu, t.i, o);
      u.s = __shfl_xor_sync(0xffffffffu, t.s, o);
      t = top2_merge(t, u);
    }
    return t;
  };
  auto publish = [&](Top2 t) {   // this warp's candidate into slot crank * NW + warp of every CTA
    if (lane == 0) {
      const int slot = crank * NW + warp;
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        cvr[q][slot] = t.v;
        csr[q][slot] = t.s;
        cir[q][slot] = t.i;
      }
    }
  };
  {
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    for (int jl0 = 0; jl0 < mloc; jl0 += RPP) {
      const int jl = jl0 + rloc;
      double q = 0.0;
      if (jl < mloc)
        for (int r = sub; r < d; r += CQ_TPR) q = fma(P[(int64_t)jl * LD + r], P[(int64_t)jl * LD + r], q);
      q = row_sum(q);
      if (jl < mloc) {
        const int j = crank + CL * jl;
        loc = top2_merge(loc, Top2{sqrt(q), (j << 16) | j, -1.0});
      }
    }
    publish(warp_best(loc));
  }
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  double min_gap = INFINITY, margin = INFINITY;
  int k = 0;
  bool aborted = false;
#ifdef H2_CQ_PROF
  long long pr[6] = {0, 0, 0, 0, 0, 0}, tp0 = clock64(), tp1 = 0;
#define CQC(n) do { tp1 = clock64(); pr[n] += tp1 - tp0; tp0 = tp1; } while (0)
#else
#define CQC(n) do { } while (0)
#endif
  for (int i = 0;; ++i) {
    CQC(4);   // publish
    cl.sync();   // (A) the candidates of step i (and the polled flag) are visible
    CQC(0);   // barrier A
    Top2 t = lane < NW * CL ? Top2{cv[lane], ci[lane], cs[lane]} : Top2{-1.0, 0x7fffffff, -1.0};
    t = warp_top2(t);
    CQC(1);   // merge
    if (i >= m) break;
    const bool certthr = crank == 0 && tid == NT - 32;   // certificates (R13) off warp 0's path
    if (certthr && a.eps > 0 && i < kfull) margin = fmin(margin, fabs(t.v - a.eps) / a.eps);
    if (i == kcap || !(t.v > a.eps)) {
      k = i;
      break;
    }
    if (a.fail_flag) {
      if (i == a.fail_cap && m > d) {
        if (crank == 0 && tid == 0) atomicExch(a.fail_flag, 1);
        k = a.fail_k;
        aborted = true;
        break;
      }
      if (s_abort) {
        k = i;
        aborted = true;
        break;
      }
    }
    if (certthr && t.s >= 0) min_gap = fmin(min_gap, (t.v - t.s) / t.v);
    const int ppos = t.i >> 16, prow = t.i & 0xffff;
    if (crank == prow % CL && warp == 0) {
      // ---- Householder reflector of the pivot row's entries r >= i (dlarfg, as cpqr_kernel)
      double* Ai = P + (int64_t)(prow / CL) * LD;
      double x2 = 0.0;
      for (int r = i + 1 + lane; r < d; r += 32) x2 = fma(Ai[r], Ai[r], x2);
      x2 = warp_sum(x2);
      const double alpha = Ai[i];
      const double xnorm = sqrt(x2);
      double tau, beta;
      if (xnorm == 0.0) {
        tau = 0.0;
        beta = alpha;
      } else {
        const double h = hypot(alpha, xnorm);
        beta = alpha != 0.0 ? -copysign(h, alpha) : -h;
        tau = (beta - alpha) / beta;
      }
      const double den = alpha - beta;
      __syncwarp();
      const double rden = 1.0 / den;
      for (int r = i + 1 + lane; r < d; r += 32) {
        const double x = tau != 0.0 ? Ai[r] * rden : 0.0;
#pragma unroll
        for (int q = 0; q < CL; ++q) vr[q][r] = x;
        Ai[r] = 0.0;
      }
      if (lane == 0) {
#pragma unroll
        for (int q = 0; q < CL; ++q) {
          vr[q][i] = 1.0;
          *taur[q] = tau;
        }
        Ai[i] = beta;
      }
    }
    if (tid == 0) {   // positions i and ppos exchange their rows (identical in every CTA)
      const int r0w = rowat[i];
      rowat[i] = prow;
      rowat[ppos] = r0w;
      pos[r0w] = ppos;
      pos[prow] = i;
    }
    CQC(2);   // reflector (owner warp 0) + swap
    cl.sync();   // (B) v, tau and the positions are visible
    CQC(5);   // barrier B
    // poll the level-failure flag (global load hidden behind the update; broadcast before (A))
    int fl = 0;
    if (a.fail_flag && crank == 0 && tid == NT - 32) fl = *reinterpret_cast<volatile int*>(a.fail_flag);
    const double tau = s_tau;
    Top2 loc{-1.0, 0x7fffffff, -1.0};
    const int r0 = i + ((sub - i) & (CQ_TPR - 1));
    for (int jl0 = 0; jl0 < mloc; jl0 += RPP) {
      const int jl = jl0 + rloc;
      const int j = crank + CL * jl;
      const bool act = jl < mloc && pos[j] > i;
      double* Aj = P + (int64_t)(act ? jl : 0) * LD;
      double w = 0.0;
      if (act)
        for (int r = r0; r < d; r += CQ_TPR) w = fma(v[r], Aj[r], w);
      w = row_sum(w) * tau;
      double q = 0.0;
      if (act)
        for (int r = r0; r < d; r += CQ_TPR) {
          const double x = fma(-w, v[r], Aj[r]);
          Aj[r] = x;
          if (r > i) q = fma(x, x, q);
        }
      q = row_sum(q);
      if (act) loc = top2_merge(loc, Top2{sqrt(q), (pos[j] << 16) | j, -1.0});
    }
    CQC(3);   // update
    publish(warp_best(loc));
    if (a.fail_flag && crank == 0 && tid == NT - 32) {
#pragma unroll
      for (int q = 0; q < CL; ++q) *abr[q] = fl;
    }
    k = i + 1;
  }
#ifdef H2_CQ_PROF
  if ((tid == 0 || tid == NT - 32) && blockIdx.x < CL && !aborted)
    printf("[cqc prof] cta %d thr %d m %d d %d k %d | barA %lld merge %lld refl %lld upd %lld publ %lld barB %lld (cycles/step)\n",
           crank, tid, m, d, k, pr[0] / max(k, 1), pr[1] / max(k, 1), pr[2] / max(k, 1), pr[3] / max(k, 1),
           pr[4] / max(k, 1), pr[5] / max(k, 1));
#endif
#undef CQC
  // no distributed shared memory access after the last (A): every CTA may leave
  if (aborted) {
    if (crank == 0 && tid == 0) a.k[c] = k;
    return;
  }
  for (int64_t e = tid; e < (int64_t)mloc * d; e += NT) {
    const int64_t jl = e / d;
    const int j = crank + CL * (int)jl;
    a.W[(off + pos[j]) * d + (e - jl * d)] = P[jl * LD + (e - jl * d)];
  }
  if (crank == 0) {
    for (int q = tid; q < m; q += NT) a.perm[off + q] = rowat[q];
    if (tid == 0) a.k[c] = k;
    if (tid == NT - 32) {
      a.cert[2 * c] = min_gap;
      a.cert[2 * c + 1] = margin;
    }
  }
}

template <int CL, int NT>
static void cpqr_cluster_launch(const CpqrArgs& a, size_t sm, cudaStream_t st) {
  auto kfn = cpqr_cluster_kernel<CL, NT>;
  H2_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)a.nclusters * CL);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  H2_CUDA(cudaLaunchKernelEx(&cfg, kfn, a));
}

// shared memory per CTA of the cluster kernel with CL CTAs per panel
static size_t cqc_smem(const CpqrArgs& a, int CL) {
  const int mloc = (a.max_m + CL - 1) / CL;
  return cqc_head_bytes(a.d, a.max_m) + sizeof(double) * (size_t)mloc * cq_ld(a.d);
}

static int forced_variant() {
  const char* v = getenv("H2_CQ_VARIANT");
  if (!v) return 0;
  const std::string s(v);
  return s == "warp" ? H2_CQ_V_WARP : s == "smem" ? H2_CQ_V_SMEM : s == "global" ? H2_CQ_V_GLOBAL
       : s == "cluster" ? H2_CQ_V_CLUSTER : 0;
}

int launch_cpqr(const CpqrArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return 0;
  const int force = forced_variant();
  const size_t wsm = sizeof(double) * cw_warp_doubles(a.d) * CW_WPB;
  if (a.max_m <= 64 && wsm <= 200 * 1024 && env_int("H2_CQ_WARP", 1) != 0 && (force == 0 || force == H2_CQ_V_WARP)) {
    // per launch: the attribute is per device (a process may drive several GPUs)
    H2_CUDA(cudaFuncSetAttribute(cpqr_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cpqr_warp_kernel<<<div_up(a.nclusters, CW_WPB), 32 * CW_WPB, wsm, st>>>(a);
    H2_CHECK_LAUNCH();
    return H2_CQ_V_WARP;
  }
  // cpqr2 (opt-in H2_CQ2=1): x2 by-product, in-place retirement, active-row list, one barrier per
  // step -- measured slower at C2 (33.2 vs 30.3 ms summed kernel time, ncu launch lists
  // profiles/r2_cpqr2.md): the shorter critical path does not pay for the extra shuffles and the
  // list indirection; the big (global-panel) levels are L2-latency bound either way
  const int cq2 = env_int("H2_CQ2", 0);   // per launch (tests switch it)
  if (cq2 != 0 && env_int("H2_CQ_ONEBAR", 0) == 0) {
    size_t sm = sizeof(double) * cq2_head_doubles(a.max_m);
    const size_t panel = sizeof(double) * (size_t)a.max_m * cq_ld(a.d);
    const int NTsel = a.max_m > 64 && a.nclusters < 148 ? 1024 : (a.max_m > 32 ? 512 : 256);
    if (sm + panel <= 200 * 1024 && force != H2_CQ_V_GLOBAL) {
      sm += panel;
      if (NTsel == 1024) cpqr2_launch<true, 1024>(a, sm, nullptr, st);
      else if (NTsel == 512) cpqr2_launch<true, 512>(a, sm, nullptr, st);
      else cpqr2_launch<true, 256>(a, sm, nullptr, st);
      H2_CHECK_LAUNCH();
      return H2_CQ_V_SMEM;
    }
    double* scr = static_cast<double*>(cache_alloc(sizeof(double) * std::max<int64_t>(a.rows * a.d, 1), st));
    if (NTsel == 1024) cpqr2_launch<false, 1024>(a, sm, scr, st);
    else if (NTsel == 512) cpqr2_launch<false, 512>(a, sm, scr, st);
    else cpqr2_launch<false, 256>(a, sm, scr, st);
    H2_CHECK_LAUNCH();
    cache_free(scr, st);
    return H2_CQ_V_GLOBAL;
  }
  static const int onebar = env_int("H2_CQ_ONEBAR", 0);
  // 1: every block-panel level (measured slower at C2: 33.6 vs 30.4 ms); 2: only levels with fewer
  // panels than SMs (the latency-bound upper levels, 1024 threads per panel)
  if (onebar == 1 || (onebar == 2 && a.nclusters < 148)) {
    // one-barrier kernel: perm + retired flags + (SMEM) the padded panel
    size_t sm = sizeof(double) * cq1_head_doubles(a.max_m);
    const size_t panel = sizeof(double) * (size_t)a.max_m * cq_ld(a.d);
    // threads: 8 per panel row pass; 1024 when few panels leave SMs idle (upper levels)
    const int NTsel = a.max_m > 64 && a.nclusters < 148 ? 1024 : (a.max_m > 32 ? 512 : 256);
    if (sm + panel <= 200 * 1024 && force != H2_CQ_V_GLOBAL) {
      sm += panel;
      if (NTsel == 1024) cpqr1_launch<true, 1024>(a, sm, nullptr, st);
      else if (NTsel == 512) cpqr1_launch<true, 512>(a, sm, nullptr, st);
      else cpqr1_launch<true, 256>(a, sm, nullptr, st);
      H2_CHECK_LAUNCH();
      return H2_CQ_V_SMEM;
    }
    double* scr = static_cast<double*>(cache_alloc(sizeof(double) * std::max<int64_t>(a.rows * a.d, 1), st));
    if (NTsel == 1024) cpqr1_launch<false, 1024>(a, sm, scr, st);
    else if (NTsel == 512) cpqr1_launch<false, 512>(a, sm, scr, st);
    else cpqr1_launch<false, 256>(a, sm, scr, st);
    H2_CHECK_LAUNCH();
    cache_free(scr, st);
    return H2_CQ_V_GLOBAL;
  }
  size_t sm = sizeof(double) * (a.d + a.max_m + (a.max_m + 1) / 2);
  size_t panel = sizeof(double) * (size_t)a.max_m * cq_ld(a.d);
  // rows per pass = threads / 8 (32 or 64); 512 threads once a panel has more than 32 rows
  const bool big = a.max_m > 32;
  int used;
  // CTA-cluster kernel (H2_CQ_CLUSTER, default 1: the panels that do not fit one CTA's shared
  // memory on levels with at most 74 panels; 2: every such level; 0 off): 2 CTAs x 512 threads,
  // or 4 x 256 when half a panel does not fit either
  const int clus = env_int("H2_CQ_CLUSTER", 1);
  const bool fits1 = sm + panel <= 200 * 1024;
  // measured at C2 (ncu, profiles/r2_cpqr_cluster.md): faster on levels with few panels (32 / 64:
  // 1.17 -> 0.76, 1.31 -> 0.93 ms), slower once 2 CTAs per panel exceed the SMs (128-1024 panels)
  const bool few_panels = 2 * a.nclusters <= 148;
  if ((force == H2_CQ_V_CLUSTER || (force == 0 && clus != 0 && !fits1 && (few_panels || clus >= 2))) &&
      a.max_m >= 2) {
    // H2_CQ_CLUSTER=4 (A/B): 4 CTAs x 256 threads per panel on every level it is used (smaller
    // CTAs: several clusters per SM on the many-panel levels)
    // default: 4 x 256 when the level's clusters fit twice over the SMs (<= 74 panels: depths 5-6
    // of C2, 0.73 -> 0.57 / 0.90 -> 0.79 ms), else 2 x 512
    if ((clus == 4 || (clus == 1 && force == 0 && 4 * a.nclusters <= 2 * 148)) && cqc_smem(a, 4) <= 210 * 1024) {
      cpqr_cluster_launch<4, 256>(a, cqc_smem(a, 4), st);
      H2_CHECK_LAUNCH();
      return H2_CQ_V_CLUSTER;
    }
    if (cqc_smem(a, 2) <= 210 * 1024) {
      cpqr_cluster_launch<2, 512>(a, cqc_smem(a, 2), st);
      H2_CHECK_LAUNCH();
      return H2_CQ_V_CLUSTER;
    }
    if (cqc_smem(a, 4) <= 210 * 1024) {
      cpqr_cluster_launch<4, 256>(a, cqc_smem(a, 4), st);
      H2_CHECK_LAUNCH();
      return H2_CQ_V_CLUSTER;
    }
  }
  if (sm + panel <= 200 * 1024 && force != H2_CQ_V_GLOBAL) {
    sm += panel;
    if (big) cpqr_launch<true, 512>(a, sm, st);
    else cpqr_launch<true, 256>(a, sm, st);
    used = H2_CQ_V_SMEM;
  } else {
    // H2_CQ_HYB = shared memory (KB) per CTA for the global-panel variant's switch to shared
    // memory once the active part fits (0: off)
    const int hyb = env_int("H2_CQ_HYB", 0);
    if (hyb > 0) {
      const size_t smh = std::max(sm, (size_t)std::min(hyb, 200) * 1024);
      if (big) cpqr_launch_e<false, 512, 0, true>(a, smh, st);
      else cpqr_launch_e<false, 256, 0, true>(a, smh, st);
    } else if (big) cpqr_launch<false, 512>(a, sm, st);
    else cpqr_launch<false, 256>(a, sm, st);
    used = H2_CQ_V_GLOBAL;
  }
  H2_CHECK_LAUNCH();
  return used;
}

// ------------------------------------------------------------------------------------------
// ID epilogue.  W row j holds column j of the factored A: R(0:k, j) in its first k entries.
// X (m x k row-major): X(J[i], :) = e_i, X(Rhat[c], :) = T(:, c)^T, T = R11^{-1} R12 (R15: back
// substitution, rows k-1 -> 0).
// CTA (cluster, 32 redundant columns), 256 threads; B = R12(:, cols) (k x 32) lives in shared
// memory and is overwritten by T.  Blocked right-looking back substitution over 32-row blocks
// (from the bottom): warp 0 solves the 32 x 32 diagonal block (lane = column, left-looking,
// ascending j), then all threads apply the rank-32 update to the rows above.  The previous
// version (one thread per column, serial k^2/2 loop reading T from global memory) took 5 ms
// per launch at the top levels (32 clusters, k ~ 210).
// ------------------------------------------------------------------------------------------
constexpr int ID_CB = 32;
__global__ void __launch_bounds__(256) id_kernel(IdArgs a, double* __restrict__ gpanel) {
  extern __shared__ double smB[];          // k x ID_CB, row stride ID_CB + 1
  // ranks beyond the shared-memory panel (k > ~770) use a per-CTA panel in global memory
  double* sB = gpanel ? gpanel + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * a.max_k * (ID_CB + 1) : smB;
  __shared__ double sD[ID_CB][ID_CB + 1];  // diagonal block R(i0:i1, i0:i1)
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c], k = a.k[c], d = a.d;
  const int64_t off = a.poff[c];
  const double* A = a.W + off * d;
  const int* perm = a.perm + off;
  double* X = a.X + a.xoff[c];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.y == 0) {
    for (int i = warp; i < k; i += 8) {
      double* row = X + (int64_t)perm[i] * k;
      for (int q = lane; q < k; q += 32) row[q] = (q == i) ? 1.0 : 0.0;
      if (lane == 0) a.skel[a.roff[c] + i] = a.ibar[off + perm[i]];
    }
  }
  const int cc0 = blockIdx.y * ID_CB;
  const int ncc = min(ID_CB, m - k - cc0);
  if (ncc <= 0 || k == 0) return;
  constexpr int LD = ID_CB + 1;
  // B(i, cc) = R(i, k + cc0 + cc) = W row (k + cc0 + cc), entry i
  for (int e = tid; e < k * ID_CB; e += 256) {
    const int cc = e / k, i = e - cc * k;
    sB[i * LD + cc] = cc < ncc ? A[(int64_t)(k + cc0 + cc) * d + i] : 0.0;
  }
  for (int i1 = k; i1 > 0; i1 -= ID_CB) {
    const int i0 = max(0, i1 - ID_CB), nb = i1 - i0;
    __syncthreads();
    for (int e = tid; e < nb * nb; e += 256) {
      const int jj = e / nb, ii = e - jj * nb;       // R(i0+ii, i0+jj) = W row i0+jj, entry i0+ii
      sD[ii][jj] = A[(int64_t)(i0 + jj) * d + i0 + ii];
    }
    __syncthreads();
    if (warp == 0) {
      // column `lane`: t_i = (b_i - sum_{j>i, j<i1} R(i,j) t_j) / R(i,i), ascending j
      for (int ii = nb - 1; ii >= 0; --ii) {
        double s = sB[(i0 + ii) * LD + lane];
        for (int jj = ii + 1; jj < nb; ++jj) s -= sD[ii][jj] * sB[(i0 + jj) * LD + lane];
        sB[(i0 + ii) * LD + lane] = s / sD[ii][ii];
      }
    }
    __syncthreads();
    // rows r < i0: b_r -= sum_{j in [i0,i1)} R(r, j) t_j   (ascending j)
    for (int e = tid; e < i0 * ID_CB; e += 256) {
      const int r = e / ID_CB, cc = e - r * ID_CB;
      double s = sB[r * LD + cc];
      for (int jj = 0; jj < nb; ++jj) s -= A[(int64_t)(i0 + jj) * d + r] * sB[(i0 + jj) * LD + cc];
      sB[r * LD + cc] = s;
    }
  }
  __syncthreads();
  // X(Rhat[cc0 + cc], :) = T(:, cc0 + cc)^T
  for (int cc = warp; cc < ncc; cc += 8) {
    double* row = X + (int64_t)perm[k + cc0 + cc] * k;
    for (int i = lane; i < k; i += 32) row[i] = sB[i * LD + cc];
  }
}

void launch_id(const IdArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  const int ny = std::max(1, div_up(a.max_red, ID_CB));
  const size_t smem = sizeof(double) * (size_t)std::max(a.max_k, 1) * (ID_CB + 1);
  // static sD + dynamic may exceed 48 KB for any k > 150; per launch (the attribute is per device)
  H2_CUDA(cudaFuncSetAttribute(id_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  if (smem <= 200 * 1024) {
    id_kernel<<<dim3(a.nclusters, ny), 256, smem, st>>>(a, nullptr);
    H2_CHECK_LAUNCH();
  } else {
    double* g = static_cast<double*>(cache_alloc(smem * (size_t)a.nclusters * ny, st));
    id_kernel<<<dim3(a.nclusters, ny), 256, 0, st>>>(a, g);
    H2_CHECK_LAUNCH();
    cache_free(g, st);
  }
}

// ------------------------------------------------------------------------------------------
// shrink + project for columns [c0, c1):  Yp(roff+i) = Yl(poff+J[i]),
// Op(roff+i) = Ol(poff+J[i]) + sum_cc T(i,cc) Ol(poff+Rhat[cc])   (= X^T Ol, identity rows exact)
// ------------------------------------------------------------------------------------------
// CTA = (cluster, 32 skeleton rows i, 32 columns): Op(i, :) = Ol(J_i, :) + sum_cc T(i, cc)
// Ol(Rhat_cc, :) as a shared-memory tiled product over 32-deep cc slabs (the interpolation rows
// X(Rhat_cc, i) and the sample rows Ol(Rhat_cc, :) staged once per slab and reused 32 times);
// each thread 4 rows of one column, cc ascending from Ol(J_i) (the order of the scalar version).
constexpr int SP_T = 32;
__global__ void __launch_bounds__(256) shrink_project_kernel(ShrinkArgs a) {
  __shared__ double sX[SP_T][SP_T + 1];   // [cc][i]
  __shared__ double sO[SP_T][SP_T + 1];   // [cc][col]
  __shared__ int sR[SP_T];
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c], k = a.k[c];
  const int i0 = blockIdx.y * SP_T;
  const int cb0 = a.c0 + blockIdx.z * SP_T;
  const int nc = min(SP_T, a.c1 - cb0);
  if (i0 >= k || nc <= 0) return;
  const int64_t off = a.poff[c];
  const int* perm = a.perm + off;
  const double* X = a.X + a.xoff[c];
  const int tid = threadIdx.x, col = tid & 31, ib = (tid >> 5) * 4;
  double acc[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + ib + r;
    acc[r] = 0.0;
    if (i < k && col < nc) {
      const int64_t src = off + perm[i];
      a.Yp[(a.roff[c] + i) * a.ldp + cb0 + col] = a.Yl[src * a.ld + cb0 + col];   // batchedShrink
      acc[r] = a.Ol[src * a.ld + cb0 + col];
    }
  }
  for (int cc0 = 0; cc0 < m - k; cc0 += SP_T) {
    const int nt = min(SP_T, m - k - cc0);
    __syncthreads();
    if (tid < SP_T) sR[tid] = tid < nt ? perm[k + cc0 + tid] : 0;
    __syncthreads();
    for (int e = tid; e < SP_T * SP_T; e += 256) {
      const int t = e >> 5, x = e & 31;
      const bool ok = t < nt;
      sX[t][x] = (ok && i0 + x < k) ? X[(int64_t)sR[t] * k + i0 + x] : 0.0;
      sO[t][x] = (ok && x < nc) ? a.Ol[(off + sR[t]) * a.ld + cb0 + x] : 0.0;
    }
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
      const double o = sO[t][col];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fma(sX[t][ib + r], o, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int i = i0 + ib + r;
    if (i < k && col < nc) a.Op[(a.roff[c] + i) * a.ldp + cb0 + col] = acc[r];
  }
}

void launch_shrink_project(const ShrinkArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0 || a.c1 <= a.c0) return;
  const dim3 grid(a.nclusters, div_up(std::max(a.max_k, 1), SP_T), div_up(a.c1 - a.c0, SP_T));
  shrink_project_kernel<<<grid, 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

}  // namespace h2
