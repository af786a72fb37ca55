// Host-side KD-tree and dual-tree traversal (§II-A) -> per-depth CSR batch
// descriptors (§IV-A).  Readings R1-R6 of DESIGN.md.  Built once per tree,
// before h2_build (the partition is an input of Algorithm 1).
// Compiled with -ffp-contract=off: the admissibility arithmetic must not be contracted.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

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
  std::sort(pairs.begin(), pairs.end());
  C.ptr.assign(nrows + 1, 0);
  C.idx.resize(pairs.size());
  for (size_t q = 0; q < pairs.size(); ++q) {
    C.ptr[pairs[q].first + 1]++;
    C.idx[q] = pairs[q].second;
  }
  for (int32_t r = 0; r < nrows; ++r) C.ptr[r + 1] += C.ptr[r];
  C.us.clear();
  C.ub.clear();
  for (auto& p : pairs)
    if (strict ? p.first < p.second : p.first <= p.second) {
      C.us.push_back(p.first);
      C.ub.push_back(p.second);
    }
  C.uidx.resize(pairs.size());
  for (size_t q = 0; q < pairs.size(); ++q) {
    int32_t a = std::min(pairs[q].first, pairs[q].second), b = std::max(pairs[q].first, pairs[q].second);
    // unique list is sorted by (s, b): binary search
    size_t lo = 0, hi = C.us.size();
    while (lo < hi) {
      size_t mid = (lo + hi) / 2;
      if (C.us[mid] < a || (C.us[mid] == a && C.ub[mid] < b)) lo = mid + 1;
      else hi = mid;
    }
    C.uidx[q] = (int32_t)lo;
  }
}

}  // namespace

void tree_build_host(h2_tree& T, const double* X, int64_t n, int dim, int leaf, double eta, int rule) {
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

  // ---- KD-tree (R4): median split of the longest bbox axis, key (coordinate, original index)
  T.perm.resize(n);
  std::iota(T.perm.begin(), T.perm.end(), int64_t(0));
  T.begin.assign(Dl + 1, {});
  T.end.assign(Dl + 1, {});
  T.begin[0] = {0};
  T.end[0] = {n};
  for (int t = 0; t < Dl; ++t) {
    const int64_t nn = int64_t(1) << t;
    T.begin[t + 1].resize(2 * nn);
    T.end[t + 1].resize(2 * nn);
    for (int64_t c = 0; c < nn; ++c) {
      int64_t b = T.begin[t][c], e = T.end[t][c], m = e - b;
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t q = b; q < e; ++q)
        for (int a = 0; a < dim; ++a) {
          double v = coord(T.perm[q], a);
          lo[a] = std::min(lo[a], v);
          hi[a] = std::max(hi[a], v);
        }
      int axis = 0;
      double best = hi[0] - lo[0];
      for (int a = 1; a < dim; ++a)
        if (hi[a] - lo[a] > best) {
          best = hi[a] - lo[a];
          axis = a;
        }
      auto less = [&](int64_t p, int64_t q) {
        double cp = coord(p, axis), cq = coord(q, axis);
        return cp < cq || (cp == cq && p < q);
      };
      int64_t left = (m + 1) / 2;
      if (t == Dl - 1) {
        std::sort(T.perm.begin() + b, T.perm.begin() + e, less);   // leaf order = sorted (R4)
      } else if (m > 1) {
        std::nth_element(T.perm.begin() + b, T.perm.begin() + b + left, T.perm.begin() + e, less);
      }
      T.begin[t + 1][2 * c] = b;
      T.end[t + 1][2 * c] = b + left;
      T.begin[t + 1][2 * c + 1] = b + left;
      T.end[t + 1][2 * c + 1] = e;
    }
  }
  T.xt.assign(n, 0.0);
  T.yt.assign(n, 0.0);
  T.zt.assign(n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    T.xt[i] = coord(T.perm[i], 0);
    if (dim > 1) T.yt[i] = coord(T.perm[i], 1);
    if (dim > 2) T.zt[i] = coord(T.perm[i], 2);
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
  for (int t = 0; t <= Dl; ++t) {
    std::vector<std::pair<int32_t, int32_t>> far;
    nxt.clear();
    for (auto& p : cur) {
      int32_t s = p.first, u = p.second;
      bool adm = false;
      if (s != u) {
        double dist = distance(box[t][s], box[t][u], rule);
        adm = (diam[t][s] + diam[t][u]) * 0.5 <= eta * dist;   // Eq.(1)
      }
      if (adm) far.push_back(p);
      else if (t == Dl) near.push_back(p);
      else
        for (int a = 0; a < 2; ++a)
          for (int bb = 0; bb < 2; ++bb) nxt.push_back({2 * s + a, 2 * u + bb});
    }
    if (!far.empty() && T.top < 0) T.top = t;
    make_csr(T.far[t], far, 1 << t, true);
    cur.swap(nxt);
  }
  make_csr(T.near, near, 1 << Dl, false);
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
}

namespace {
template <class V>
typename V::value_type* upload(const V& v) {
  typename V::value_type* p = nullptr;
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(typename V::value_type);
  H2_CUDA(cudaMalloc(&p, bytes));
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
  cudaFree(d.ptr);
  cudaFree(d.idx);
  cudaFree(d.uidx);
  cudaFree(d.us);
  cudaFree(d.ub);
  d = DeviceCSR{};
}
}  // namespace

void tree_upload(h2_tree& T) {
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
  T.d_D_off = upload(T.D_off);
  T.d_near = upload_csr(T.near);
  T.d_far.resize(T.Dl + 1);
  for (int t = 0; t <= T.Dl; ++t) T.d_far[t] = upload_csr(T.far[t]);
  T.device = dev;
}

h2_tree::~h2_tree() {
  if (device < 0) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaFree(d_x);
  cudaFree(d_y);
  cudaFree(d_z);
  cudaFree(d_iota);
  cudaFree(d_leaf_begin);
  cudaFree(d_leaf_size);
  cudaFree(d_D_off);
  free_csr(d_near);
  for (auto& f : d_far) free_csr(f);
  cudaSetDevice(prev);
}
