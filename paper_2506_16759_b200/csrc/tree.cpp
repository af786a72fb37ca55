// Host-side KD-tree and dual-tree traversal (§II-A) -> per-depth CSR batch
// descriptors (§IV-A).  Readings R1-R6 of DESIGN.md.  Built once per tree,
// before h2_build (the partition is an input of Algorithm 1).
// Compiled with -ffp-contract=off: the admissibility arithmetic must not be contracted.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <thread>

#include "alloc.hpp"
#include "common.cuh"
#include "tree.hpp"

namespace {

int leaf_depth_for(int64_t n, int leaf) {
  int d = 0;
  while ((n + (int64_t(1) << d) - 1) / (int64_t(1) << d) > leaf) ++d;
  return d;
}

struct BBox {
  double lo[3], hi[3];
};

double diameter(const BBox& b) {  // R2: bbox diagonal, left-to-right sum
  double acc = 0.0;
  for (int d = 0; d < 3; ++d) {
    double e = b.hi[d] - b.lo[d];
    acc = acc + e * e;
  }
  return std::sqrt(acc);
}

double distance(const BBox& s, const BBox& t, int rule) {  // R1
  double acc = 0.0;
  for (int d = 0; d < 3; ++d) {
    double g;
    if (rule == H2_DIST_CENTER) {
      g = (s.lo[d] + s.hi[d]) * 0.5 - (t.lo[d] + t.hi[d]) * 0.5;
    } else {
      g = std::max(0.0, std::max(t.lo[d] - s.hi[d], s.lo[d] - t.hi[d]));
    }
    acc = acc + g * g;
  }
  return std::sqrt(acc);
}

void make_csr(PairCSR& C, std::vector<std::pair<int32_t, int32_t>>& pairs, int32_t nrows, bool strict) {
  // counting sort by row, then each (short) row sorted: O(nnz) instead of a global sort
  C.ptr.assign(nrows + 1, 0);
  for (auto& p : pairs) C.ptr[p.first + 1]++;
  for (int32_t r = 0; r < nrows; ++r) C.ptr[r + 1] += C.ptr[r];
  C.idx.resize(pairs.size());
  {
    std::vector<int32_t> fill(C.ptr.begin(), C.ptr.end() - 1);
    for (auto& p : pairs) C.idx[fill[p.first]++] = p.second;
  }
  // per-row work split over threads for large row counts (rows are independent; deterministic)
  auto par_rows = [nrows](auto&& fn) {
    const int nt = nrows >= 4096 ? (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency())) : 1;
    if (nt <= 1) {
      fn(0, nrows);
      return;
    }
    std::vector<std::thread> th;
    for (int q = 0; q < nt; ++q)
      th.emplace_back([&fn, q, nt, nrows] { fn((int32_t)((int64_t)nrows * q / nt), (int32_t)((int64_t)nrows * (q + 1) / nt)); });
    for (auto& x : th) x.join();
  };
  par_rows([&](int32_t r0, int32_t r1) {
    for (int32_t r = r0; r < r1; ++r) std::sort(C.idx.begin() + C.ptr[r], C.idx.begin() + C.ptr[r + 1]);
  });
  // unique pairs (s, b), s <= b (s < b if strict), sorted by (s, b): row s's partners b >= s
  std::vector<int64_t> uoff(nrows + 1, 0);
  std::vector<int32_t> first(nrows);   // position in row s of its first partner b >= s (b > s)
  for (int32_t r = 0; r < nrows; ++r) {
    const int32_t* b0 = C.idx.data() + C.ptr[r];
    const int32_t* b1 = C.idx.data() + C.ptr[r + 1];
    const int32_t* f = strict ? std::upper_bound(b0, b1, r) : std::lower_bound(b0, b1, r);
    first[r] = (int32_t)(f - b0);
    uoff[r + 1] = uoff[r] + (b1 - f);
  }
  C.us.resize(uoff[nrows]);
  C.ub.resize(uoff[nrows]);
  C.uidx.resize(pairs.size());
  for (int32_t r = 0; r < nrows; ++r)
    for (int32_t e = C.ptr[r] + first[r], q = 0; e < C.ptr[r + 1]; ++e, ++q) {
      C.us[uoff[r] + q] = r;
      C.ub[uoff[r] + q] = C.idx[e];
    }
  par_rows([&](int32_t r0, int32_t r1) {
    for (int32_t r = r0; r < r1; ++r)
      for (int32_t e = C.ptr[r]; e < C.ptr[r + 1]; ++e) {
        const int32_t b = C.idx[e];
        const int32_t a = std::min(r, b), c = std::max(r, b);
        // position of c among row a's partners >= a (rows are sorted; the symmetric set holds (a, c))
        const int32_t* b0 = C.idx.data() + C.ptr[a] + first[a];
        const int32_t* b1 = C.idx.data() + C.ptr[a + 1];
        C.uidx[e] = (int32_t)(uoff[a] + (std::lower_bound(b0, b1, c) - b0));
      }
  });
}

}  // namespace

void tree_build_host(h2_tree& T, const double* X, int64_t n, int dim, int leaf, double eta, int rule) {
  tree_build_order(T, X, n, dim, leaf, eta, rule);
  tree_build_partition(T);
}

// The KD ordering (R4) and the tree-order coordinates: everything the dense sketch needs.
void tree_build_order(h2_tree& T, const double* X, int64_t n, int dim, int leaf, double eta, int rule) {
  H2_REQUIRE(n >= 1 && n < (int64_t(1) << 31), "h2_tree_build: need 1 <= n < 2^31");
  H2_REQUIRE(dim >= 1 && dim <= 3, "h2_tree_build: dim must be 1, 2 or 3");
  H2_REQUIRE(leaf >= 2, "h2_tree_build: leaf_size >= 2");
  H2_REQUIRE(eta > 0, "h2_tree_build: eta > 0");
  H2_REQUIRE(rule == H2_DIST_CENTER || rule == H2_DIST_BOX, "h2_tree_build: bad dist_rule");
  for (int64_t i = 0; i < n * dim; ++i) H2_REQUIRE(std::isfinite(X[i]), "h2_tree_build: non-finite coordinate");
  T.n = n;
  T.dim = dim;
  T.leaf_size = leaf;
  T.eta = eta;
  T.rule = rule;
  const int Dl = T.Dl = leaf_depth_for(n, leaf);
  auto coord = [&](int64_t orig, int ax) { return X[orig * dim + ax]; };
  const bool trace = getenv("H2_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[h2 tree] %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };

  // ---- KD-tree (R4): median split of the longest bbox axis, key (coordinate, original index).
  // The points move as 32-byte records (coordinates + original index): partitions stream through
  // contiguous memory instead of gathering coordinates through the permutation.
  struct Pt {
    double c[3];
    int64_t orig;
  };
  std::vector<Pt> pts(n);
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) pts[i].c[a] = a < dim ? coord(i, a) : 0.0;
    pts[i].orig = i;
  }
  lap("kd records");
  T.begin.assign(Dl + 1, {});
  T.end.assign(Dl + 1, {});
  T.begin[0] = {0};
  T.end[0] = {n};
  const int nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  for (int t = 0; t < Dl; ++t) {
    const int64_t nn = int64_t(1) << t;
    T.begin[t + 1].resize(2 * nn);
    T.end[t + 1].resize(2 * nn);
    // the nodes of a depth own disjoint segments: split them over threads (deterministic)
    auto nodes = [&](int64_t c0, int64_t c1) {
      for (int64_t c = c0; c < c1; ++c) {
        const int64_t b = T.begin[t][c], e = T.end[t][c], m = e - b;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t q = b; q < e; ++q)
          for (int a = 0; a < dim; ++a) {
            lo[a] = std::min(lo[a], pts[q].c[a]);
            hi[a] = std::max(hi[a], pts[q].c[a]);
          }
        int axis = 0;
        double best = hi[0] - lo[0];
        for (int a = 1; a < dim; ++a)
          if (hi[a] - lo[a] > best) {
            best = hi[a] - lo[a];
            axis = a;
          }
        auto less = [axis](const Pt& p, const Pt& q) {
          return p.c[axis] < q.c[axis] || (p.c[axis] == q.c[axis] && p.orig < q.orig);
        };
        const int64_t left = (m + 1) / 2;
        if (t == Dl - 1) {
          std::sort(pts.begin() + b, pts.begin() + e, less);   // leaf order = sorted (R4)
        } else if (m > 1) {
          std::nth_element(pts.begin() + b, pts.begin() + b + left, pts.begin() + e, less);
        }
        T.begin[t + 1][2 * c] = b;
        T.end[t + 1][2 * c] = b + left;
        T.begin[t + 1][2 * c + 1] = b + left;
        T.end[t + 1][2 * c + 1] = e;
      }
    };
    const int nt = (int)std::min<int64_t>(nthreads, nn);
    if (nt <= 1) {
      nodes(0, nn);
    } else {
      std::vector<std::thread> th;
      for (int q = 0; q < nt; ++q) th.emplace_back(nodes, nn * q / nt, nn * (q + 1) / nt);
      for (auto& x : th) x.join();
    }
    if (trace && t < 4) lap("kd depth");
  }
  T.perm.resize(n);
  for (int64_t i = 0; i < n; ++i) T.perm[i] = pts[i].orig;
  lap("kd-tree");
  T.xt.resize(n);
  T.yt.resize(n);
  T.zt.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    T.xt[i] = pts[i].c[0];
    T.yt[i] = pts[i].c[1];
    T.zt[i] = pts[i].c[2];
  }
  {
    double lo[3] = {1e308, 1e308, 1e308}, hi[3] = {-1e308, -1e308, -1e308};
    for (int64_t i = 0; i < n; ++i) {
      const double v[3] = {T.xt[i], T.yt[i], T.zt[i]};
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], v[a]);
        hi[a] = std::max(hi[a], v[a]);
      }
    }
    T.diam = n > 0 ? std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                               (hi[2] - lo[2]) * (hi[2] - lo[2]))
                   : 0.0;
  }

  lap("coords");
}

// tree_build_order on the GPU (kd_gpu.cu): identical ordering, node ranges from the sizes alone
void tree_build_order_gpu(h2_tree& T, const double* X, int64_t n, int dim, int leaf, double eta, int rule) {
  H2_REQUIRE(n >= 1 && n < (int64_t(1) << 31), "h2_tree_build: need 1 <= n < 2^31");
  H2_REQUIRE(dim >= 1 && dim <= 3, "h2_tree_build: dim must be 1, 2 or 3");
  H2_REQUIRE(leaf >= 2, "h2_tree_build: leaf_size >= 2");
  H2_REQUIRE(eta > 0, "h2_tree_build: eta > 0");
  H2_REQUIRE(rule == H2_DIST_CENTER || rule == H2_DIST_BOX, "h2_tree_build: bad dist_rule");
  for (int64_t i = 0; i < n * dim; ++i) H2_REQUIRE(std::isfinite(X[i]), "h2_tree_build: non-finite coordinate");
  T.n = n;
  T.dim = dim;
  T.leaf_size = leaf;
  T.eta = eta;
  T.rule = rule;
  const int Dl = T.Dl = leaf_depth_for(n, leaf);
  T.begin.assign(Dl + 1, {});
  T.end.assign(Dl + 1, {});
  T.begin[0] = {0};
  T.end[0] = {n};
  std::vector<int> seg_all;
  for (int t = 0; t < Dl; ++t) {
    const int64_t nn = int64_t(1) << t;
    T.begin[t + 1].resize(2 * nn);
    T.end[t + 1].resize(2 * nn);
    for (int64_t c = 0; c < nn; ++c) {
      const int64_t b = T.begin[t][c], e = T.end[t][c], left = (e - b + 1) / 2;
      seg_all.push_back((int)b);
      T.begin[t + 1][2 * c] = b;
      T.end[t + 1][2 * c] = b + left;
      T.begin[t + 1][2 * c + 1] = b + left;
      T.end[t + 1][2 * c + 1] = e;
    }
    seg_all.push_back((int)n);
  }
  const bool trace = getenv("H2_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[h2 tree] %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  lap("gpu setup");
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  cudaStream_t st;
  H2_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double box[6];
  try {
    h2::kd_order_device(X, n, dim, Dl, seg_all, &T.d_perm, &T.d_x, &T.d_y, &T.d_z, &T.d_iota, box, st);
  } catch (...) {
    cudaStreamDestroy(st);
    throw;
  }
  cudaStreamDestroy(st);
  lap("gpu kd");
  T.device = dev;
  {
    std::vector<int64_t> lb(T.begin[Dl]);
    lb.push_back(n);
    T.d_leaf_begin = static_cast<int64_t*>(h2::cache_alloc(lb.size() * sizeof(int64_t), nullptr));
    H2_CUDA(cudaMemcpy(T.d_leaf_begin, lb.data(), lb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    std::vector<int32_t> ls(T.begin[Dl].size());
    for (size_t c = 0; c < ls.size(); ++c) ls[c] = (int32_t)(T.end[Dl][c] - T.begin[Dl][c]);
    T.d_leaf_size = static_cast<int32_t*>(h2::cache_alloc(std::max<size_t>(ls.size(), 1) * sizeof(int32_t), nullptr));
    H2_CUDA(cudaMemcpy(T.d_leaf_size, ls.data(), ls.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  // the bounding-box diagonal as the host computes it (tree-order coordinates, zero-padded to 3D)
  {
    double lo[3] = {1e308, 1e308, 1e308}, hi[3] = {-1e308, -1e308, -1e308};
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], box[a]);
      hi[a] = std::max(hi[a], box[3 + a]);
    }
    T.diam = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                       (hi[2] - lo[2]) * (hi[2] - lo[2]));
  }
}

// host copies of the GPU ordering (perm, tree-order coordinates) for the partition / exports
void tree_download_order(h2_tree& T) {
  if (!T.d_perm || !T.perm.empty()) return;
  H2_CUDA(cudaSetDevice(T.device));
  std::vector<int32_t> p(T.n);
  T.xt.resize(T.n);
  T.yt.resize(T.n);
  T.zt.resize(T.n);
  H2_CUDA(cudaMemcpy(p.data(), T.d_perm, sizeof(int32_t) * T.n, cudaMemcpyDeviceToHost));
  H2_CUDA(cudaMemcpy(T.xt.data(), T.d_x, sizeof(double) * T.n, cudaMemcpyDeviceToHost));
  H2_CUDA(cudaMemcpy(T.yt.data(), T.d_y, sizeof(double) * T.n, cudaMemcpyDeviceToHost));
  H2_CUDA(cudaMemcpy(T.zt.data(), T.d_z, sizeof(double) * T.n, cudaMemcpyDeviceToHost));
  T.perm.assign(p.begin(), p.end());
  // d_perm stays until the tree is freed: cudaFree would synchronise the device (this thread runs
  // while the first sketch pass does)
}

// The block partition of an ordered tree (bounding boxes, dual traversal, CSR batch descriptors,
// unique D offsets).  Synchronous in h2_tree_build; on a host thread in h2_tree_build_async.
void tree_build_partition(h2_tree& T) {
  const int Dl = T.Dl;
  const double eta = T.eta;
  const int rule = T.rule;
  const bool trace = getenv("H2_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[h2 tree] %-12s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  // ---- bounding boxes per depth (tree order, zero padded)
  std::vector<std::vector<BBox>> box(Dl + 1);
  for (int t = Dl; t >= 0; --t) {
    const int64_t nn = int64_t(1) << t;
    box[t].resize(nn);
    for (int64_t c = 0; c < nn; ++c) {
      BBox& B = box[t][c];
      if (t == Dl) {
        for (int a = 0; a < 3; ++a) {
          B.lo[a] = INFINITY;
          B.hi[a] = -INFINITY;
        }
        for (int64_t q = T.begin[t][c]; q < T.end[t][c]; ++q) {
          double v[3] = {T.xt[q], T.yt[q], T.zt[q]};
          for (int a = 0; a < 3; ++a) {
            B.lo[a] = std::min(B.lo[a], v[a]);
            B.hi[a] = std::max(B.hi[a], v[a]);
          }
        }
      } else {
        const BBox &L = box[t + 1][2 * c], &R = box[t + 1][2 * c + 1];
        for (int a = 0; a < 3; ++a) {
          B.lo[a] = std::min(L.lo[a], R.lo[a]);
          B.hi[a] = std::max(L.hi[a], R.hi[a]);
        }
      }
    }
  }

  lap("bboxes");
  // ---- dual-tree traversal (L127), depth by depth
  std::vector<std::pair<int32_t, int32_t>> cur{{0, 0}}, nxt, near;
  T.far.assign(Dl + 1, PairCSR{});
  T.top = -1;
  T.csp = 0;
  std::vector<std::vector<double>> diam(Dl + 1);
  for (int t = 0; t <= Dl; ++t) {
    diam[t].resize(box[t].size());
    for (size_t c = 0; c < box[t].size(); ++c) diam[t][c] = diameter(box[t][c]);
  }
  // the pairs of a depth are split into contiguous ranges over threads; the per-thread lists are
  // concatenated in range order, so the result is identical to the serial traversal
  const int nthr = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  // the CSR of a depth's far pairs is built on its own thread while the traversal descends
  std::vector<std::vector<std::pair<int32_t, int32_t>>> far_lists(Dl + 1);
  std::vector<std::thread> csr_threads;
  for (int t = 0; t <= Dl; ++t) {
    const int64_t np = (int64_t)cur.size();
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthr, np / 4096));
    std::vector<std::vector<std::pair<int32_t, int32_t>>> far_t(nt), nxt_t(nt), near_t(nt);
    auto work = [&](int q) {
      for (int64_t e = np * q / nt; e < np * (q + 1) / nt; ++e) {
        const auto& p = cur[e];
        const int32_t s = p.first, u = p.second;
        bool adm = false;
        if (s != u) {
          const double dist = distance(box[t][s], box[t][u], rule);
          adm = (diam[t][s] + diam[t][u]) * 0.5 <= eta * dist;   // Eq.(1)
        }
        if (adm) far_t[q].push_back(p);
        else if (t == Dl) near_t[q].push_back(p);
        else
          for (int a = 0; a < 2; ++a)
            for (int bb = 0; bb < 2; ++bb) nxt_t[q].push_back({2 * s + a, 2 * u + bb});
      }
    };
    if (nt == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int q = 0; q < nt; ++q) th.emplace_back(work, q);
      for (auto& x : th) x.join();
    }
    std::vector<std::pair<int32_t, int32_t>>& far = far_lists[t];
    nxt.clear();
    for (int q = 0; q < nt; ++q) {
      far.insert(far.end(), far_t[q].begin(), far_t[q].end());
      nxt.insert(nxt.end(), nxt_t[q].begin(), nxt_t[q].end());
      near.insert(near.end(), near_t[q].begin(), near_t[q].end());
    }
    if (!far.empty() && T.top < 0) T.top = t;
    csr_threads.emplace_back([&T, &far, t] { make_csr(T.far[t], far, 1 << t, true); });
    cur.swap(nxt);
  }
  lap("traversal");
  make_csr(T.near, near, 1 << Dl, false);
  for (auto& x : csr_threads) x.join();
  for (int t = 0; t <= Dl; ++t)
    for (int64_t r = 0; r < (int64_t(1) << t); ++r) {
      int row = T.far[t].ptr[r + 1] - T.far[t].ptr[r];
      if (t == Dl) row += T.near.ptr[r + 1] - T.near.ptr[r];
      T.csp = std::max(T.csp, row);
    }
  // unique D block offsets (s <= b), row-major m_s x m_b
  T.D_off.assign(T.near.nuniq() + 1, 0);
  for (int64_t q = 0; q < T.near.nuniq(); ++q) {
    int64_t ms = T.end[Dl][T.near.us[q]] - T.begin[Dl][T.near.us[q]];
    int64_t mb = T.end[Dl][T.near.ub[q]] - T.begin[Dl][T.near.ub[q]];
    T.D_off[q + 1] = T.D_off[q] + ms * mb;
  }
  lap("near csr");
}

// h2_tree_import: a partition built elsewhere (e.g. the CPU oracle), so that both paths consume
// the SAME tree ("a hierarchical partitioning" is an input of
// Algorithm 1).  Checked: perm is a permutation; the cluster ranges form a complete binary tree
// (children split their parent contiguously); pair indices in range, no duplicates, symmetric
// sets, no (s, s) far pair; the blocks' areas sum to n^2 (a necessary covering condition).
void tree_import_host(h2_tree& T, const h2_tree_desc& D) {
  const int64_t n = D.n;
  const int dim = D.dim, Dl = D.leaf_depth;
  H2_REQUIRE(n >= 1 && n < (int64_t(1) << 31), "h2_tree_import: need 1 <= n < 2^31");
  H2_REQUIRE(dim >= 1 && dim <= 3, "h2_tree_import: dim must be 1, 2 or 3");
  H2_REQUIRE(Dl >= 0 && Dl < 31 && (int64_t(1) << Dl) <= n, "h2_tree_import: need 0 <= leaf_depth, 2^leaf_depth <= n");
  H2_REQUIRE(D.coords && D.perm && D.begin && D.end && D.near_pairs && D.far_nnz, "h2_tree_import: NULL array");
  for (int64_t i = 0; i < n * dim; ++i) H2_REQUIRE(std::isfinite(D.coords[i]), "h2_tree_import: non-finite coordinate");
  T.n = n;
  T.dim = dim;
  T.Dl = Dl;
  T.eta = 0.0;
  T.rule = -1;   // imported: admissibility rule unknown
  {
    std::vector<char> seen(n, 0);
    T.perm.assign(D.perm, D.perm + n);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t p = T.perm[i];
      H2_REQUIRE(p >= 0 && p < n && !seen[p], "h2_tree_import: perm is not a permutation of 0..n-1");
      seen[p] = 1;
    }
  }
  T.begin.assign(Dl + 1, {});
  T.end.assign(Dl + 1, {});
  for (int t = 0; t <= Dl; ++t) {
    const int64_t nn = int64_t(1) << t;
    T.begin[t].assign(D.begin + (nn - 1), D.begin + (2 * nn - 1));
    T.end[t].assign(D.end + (nn - 1), D.end + (2 * nn - 1));
  }
  H2_REQUIRE(T.begin[0][0] == 0 && T.end[0][0] == n, "h2_tree_import: the root must hold [0, n)");
  for (int t = 0; t < Dl; ++t)
    for (int64_t c = 0; c < (int64_t(1) << t); ++c) {
      const int64_t b = T.begin[t][c], e = T.end[t][c];
      const int64_t m1 = T.end[t + 1][2 * c];
      H2_REQUIRE(T.begin[t + 1][2 * c] == b && T.begin[t + 1][2 * c + 1] == m1 && T.end[t + 1][2 * c + 1] == e &&
                     b <= m1 && m1 <= e,
                 "h2_tree_import: children must split their parent's index range contiguously");
    }
  T.leaf_size = 0;
  for (int64_t c = 0; c < (int64_t(1) << Dl); ++c)
    T.leaf_size = std::max<int32_t>(T.leaf_size, (int32_t)(T.end[Dl][c] - T.begin[Dl][c]));
  T.xt.resize(n);
  T.yt.resize(n);
  T.zt.resize(n);
  double lo[3] = {1e308, 1e308, 1e308}, hi[3] = {-1e308, -1e308, -1e308};
  for (int64_t i = 0; i < n; ++i) {
    double v[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < dim; ++a) v[a] = D.coords[T.perm[i] * dim + a];
    T.xt[i] = v[0];
    T.yt[i] = v[1];
    T.zt[i] = v[2];
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], v[a]);
      hi[a] = std::max(hi[a], v[a]);
    }
  }
  T.diam = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                     (hi[2] - lo[2]) * (hi[2] - lo[2]));
  auto size_of = [&](int t, int64_t c) { return T.end[t][c] - T.begin[t][c]; };
  long double area = 0;
  auto load = [&](const int32_t* pr, int64_t nnz, int t, bool strict, PairCSR& C) {
    const int64_t nn = int64_t(1) << t;
    std::vector<std::pair<int32_t, int32_t>> pairs(nnz);
    for (int64_t e = 0; e < nnz; ++e) {
      const int32_t s = pr[2 * e], b = pr[2 * e + 1];
      H2_REQUIRE(s >= 0 && s < nn && b >= 0 && b < nn, "h2_tree_import: pair index out of range");
      H2_REQUIRE(!strict || s != b, "h2_tree_import: an admissible pair (s, s)");
      pairs[e] = {s, b};
      area += (long double)size_of(t, s) * (long double)size_of(t, b);
    }
    make_csr(C, pairs, (int32_t)nn, strict);
    for (int64_t r = 0; r < nn; ++r)
      for (int32_t e = C.ptr[r]; e < C.ptr[r + 1]; ++e) {
        H2_REQUIRE(e == C.ptr[r] || C.idx[e] > C.idx[e - 1], "h2_tree_import: duplicate pair");
        const int32_t b = C.idx[e];
        auto it = std::lower_bound(C.idx.begin() + C.ptr[b], C.idx.begin() + C.ptr[b + 1], (int32_t)r);
        H2_REQUIRE(it != C.idx.begin() + C.ptr[b + 1] && *it == (int32_t)r, "h2_tree_import: pair set not symmetric");
      }
  };
  load(D.near_pairs, D.near_nnz, Dl, false, T.near);
  T.far.assign(Dl + 1, PairCSR{});
  T.top = -1;
  for (int t = 0; t <= Dl; ++t) {
    const int64_t nnz = D.far_nnz[t];
    H2_REQUIRE(nnz >= 0 && (nnz == 0 || (D.far_pairs && D.far_pairs[t])), "h2_tree_import: far pairs missing");
    load(nnz ? D.far_pairs[t] : nullptr, nnz, t, true, T.far[t]);
    if (nnz > 0 && T.top < 0) T.top = t;
  }
  H2_REQUIRE(area == (long double)n * (long double)n, "h2_tree_import: the blocks do not tile the n x n matrix");
  T.csp = 0;
  for (int t = 0; t <= Dl; ++t)
    for (int64_t r = 0; r < (int64_t(1) << t); ++r) {
      int row = T.far[t].ptr[r + 1] - T.far[t].ptr[r];
      if (t == Dl) row += T.near.ptr[r + 1] - T.near.ptr[r];
      T.csp = std::max(T.csp, row);
    }
  T.D_off.assign(T.near.nuniq() + 1, 0);
  for (int64_t q = 0; q < T.near.nuniq(); ++q)
    T.D_off[q + 1] = T.D_off[q] + size_of(Dl, T.near.us[q]) * size_of(Dl, T.near.ub[q]);
}

namespace {
template <class V>
typename V::value_type* upload(const V& v) {
  // the tree's device arrays live in libh2's block cache: no cudaMalloc / cudaFree (device-
  // synchronising, latency varying by 1-20 ms) per tree once the cache holds the sizes
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(typename V::value_type);
  auto* p = static_cast<typename V::value_type*>(h2::cache_alloc(bytes, nullptr));
  if (!v.empty()) H2_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(typename V::value_type), cudaMemcpyHostToDevice));
  return p;
}
DeviceCSR upload_csr(const PairCSR& C) {
  DeviceCSR d;
  d.ptr = upload(C.ptr);
  d.idx = upload(C.idx);
  d.uidx = upload(C.uidx);
  d.us = upload(C.us);
  d.ub = upload(C.ub);
  return d;
}
void free_csr(DeviceCSR& d) {
  for (void* p : {(void*)d.ptr, (void*)d.idx, (void*)d.uidx, (void*)d.us, (void*)d.ub}) h2::cache_free(p, nullptr);
  d = DeviceCSR{};
}
}  // namespace

void tree_upload(h2_tree& T) {
  tree_upload_order(T);
  tree_upload_partition(T);
}

void tree_upload_order(h2_tree& T) {
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  T.d_x = upload(T.xt);
  T.d_y = upload(T.yt);
  T.d_z = upload(T.zt);
  std::vector<int32_t> iota(T.n);
  std::iota(iota.begin(), iota.end(), 0);
  T.d_iota = upload(iota);
  std::vector<int64_t> lb(T.begin[T.Dl]);
  lb.push_back(T.n);
  T.d_leaf_begin = upload(lb);
  std::vector<int32_t> ls(T.begin[T.Dl].size());
  for (size_t c = 0; c < ls.size(); ++c) ls[c] = (int32_t)(T.end[T.Dl][c] - T.begin[T.Dl][c]);
  T.d_leaf_size = upload(ls);
  T.device = dev;
}

void tree_upload_partition(h2_tree& T) {
  T.d_D_off = upload(T.D_off);
  T.d_near = upload_csr(T.near);
  T.d_far.resize(T.Dl + 1);
  for (int t = 0; t <= T.Dl; ++t) T.d_far[t] = upload_csr(T.far[t]);
  T.part_uploaded = true;
}

void h2_tree::wait_partition() {
  std::lock_guard<std::mutex> g(part_mu);
  if (part_thread.joinable()) part_thread.join();
  if (!part_error.empty()) throw h2::Error(H2_ERR_INVALID_ARG, part_error);
}

h2_tree::~h2_tree() {
  if (part_thread.joinable()) part_thread.join();
  if (device < 0) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  // every device array of the tree comes from the block cache: back to it, no device sync
  for (void* p : {(void*)d_x, (void*)d_y, (void*)d_z, (void*)d_iota, (void*)d_perm, (void*)d_leaf_begin,
                  (void*)d_leaf_size, (void*)d_D_off})
    h2::cache_free(p, nullptr);
  free_csr(d_near);
  for (auto& f : d_far) free_csr(f);
  for (void* p : {(void*)d_nl_ptr, (void*)d_nl_chunk, (void*)d_nl_mask}) h2::cache_free(p, nullptr);
  cudaSetDevice(prev);
}
