// KD ordering (R4, §II-A) on the GPU for h2_tree_build_async (round 2): the
// same tree as the host ordering of tree.cpp, built on the device where the host needs ~17 ms at
// N = 2^18 -- the prefix of the end-to-end build before the first sketch pass can start.  Depth
// by depth, with every node a contiguous segment of the current order:
//   1. every node's bounding box (exact min / max) -> longest axis, ties -> lowest axis (as the
//      host), and every point's node id;
//   2. two STABLE global radix sorts starting from the original order: by the orderable bit
//      pattern of the point's node-axis coordinate, then by node id -- i.e. the order (node,
//      coordinate, original index) of the host comparator inside every node; the lower ceil(m/2)
//      points of a node form its left child.
// The host takes nth_element at inner depths (only the SETS of the children are defined there)
// and a full sort at depth Dl - 1 (the leaf order); sorting fully at every depth yields the same
// sets and the same final order.  Node ranges depend on the sizes only (host arrays).
#include <cub/device/device_radix_sort.cuh>

#include <vector>

#include "alloc.hpp"
#include "common.cuh"

namespace h2 {
namespace {

// order-preserving map of a finite double to uint64 (-0.0 and +0.0 compare equal, as in C++)
__device__ __forceinline__ uint64_t ord_key(double x) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  if (b == 0x8000000000000000ull) b = 0;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// one CTA per segment (grid-stride): bounding box -> axis of the segment
__global__ void __launch_bounds__(256) kd_level_kernel(const double* __restrict__ X, int dim,
                                                       const int* __restrict__ seg, int nseg,
                                                       const int* __restrict__ idx, int* __restrict__ axis_out,
                                                       double* __restrict__ box) {
  __shared__ double slo[3][8], shi[3][8];
  __shared__ int s_axis;   // (kept for the root call's single segment)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = blockIdx.x; c < nseg; c += gridDim.x) {
    const int b = seg[c], e = seg[c + 1];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int p = b + threadIdx.x; p < e; p += blockDim.x) {
      const double* x = X + (int64_t)idx[p] * dim;
      for (int a = 0; a < dim; ++a) {
        lo[a] = fmin(lo[a], x[a]);
        hi[a] = fmax(hi[a], x[a]);
      }
    }
    for (int a = 0; a < dim; ++a) {   // min / max: exact, order-free
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
        hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
      }
      if (lane == 0) {
        slo[a][warp] = lo[a];
        shi[a][warp] = hi[a];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double L[3] = {INFINITY, INFINITY, INFINITY}, Hh[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int a = 0; a < dim; ++a)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          L[a] = fmin(L[a], slo[a][w]);
          Hh[a] = fmax(Hh[a], shi[a][w]);
        }
      int axis = 0;
      double best = Hh[0] - L[0];
      for (int a = 1; a < dim; ++a)
        if (Hh[a] - L[a] > best) {
          best = Hh[a] - L[a];
          axis = a;
        }
      s_axis = axis;
      if (axis_out) axis_out[c] = axis;
      if (box) {   // the root box (diameter of the point set), zero-padded to 3D
        for (int a = 0; a < 3; ++a) {
          box[a] = a < dim ? L[a] : 0.0;
          box[3 + a] = a < dim ? Hh[a] : 0.0;
        }
      }
    }
    __syncthreads();
  }
}

// node id of every position (the nodes of a depth are contiguous position ranges, found by binary
// search over the offsets): segid of the point at position p, written at its ORIGINAL index
__global__ void kd_segid_kernel(const int* __restrict__ seg, int nseg, const int* __restrict__ idx, int n,
                                int* __restrict__ segid_orig) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    int lo = 0, hi = nseg;   // seg[lo] <= p < seg[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (seg[mid] <= p) lo = mid;
      else hi = mid;
    }
    segid_orig[idx[p]] = lo;
  }
}

// two-stage node boxes for depths with few, large nodes: CTA (s, c) reduces slice s of node c to a
// partial box (exact min / max, order-free) ...
__global__ void __launch_bounds__(256) kd_box_partial_kernel(const double* __restrict__ X, int dim,
                                                             const int* __restrict__ seg, const int* __restrict__ idx,
                                                             int S, double* __restrict__ part) {
  __shared__ double slo[3][8], shi[3][8];
  const int c = blockIdx.y, sl = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = seg[c], e0 = seg[c + 1];
  const int64_t len = e0 - b0;
  const int b = b0 + (int)(len * sl / S), e = b0 + (int)(len * (sl + 1) / S);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int p = b + threadIdx.x; p < e; p += blockDim.x) {
    const double* x = X + (int64_t)idx[p] * dim;
    for (int a = 0; a < dim; ++a) {
      lo[a] = fmin(lo[a], x[a]);
      hi[a] = fmax(hi[a], x[a]);
    }
  }
  for (int a = 0; a < dim; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) {
      slo[a][warp] = lo[a];
      shi[a][warp] = hi[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int a = threadIdx.x;
    double L = INFINITY, H = -INFINITY;
    if (a < dim)
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        L = fmin(L, slo[a][w]);
        H = fmax(H, shi[a][w]);
      }
    double* o = part + ((int64_t)c * S + sl) * 6;
    o[a] = L;
    o[3 + a] = H;
  }
}

// ... and one thread per node merges its S partials and picks the axis (as the host)
__global__ void kd_axis_kernel(const double* __restrict__ part, int nseg, int S, int dim, int* __restrict__ axis_out,
                               double* __restrict__ box) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nseg; c += gridDim.x * blockDim.x) {
    double L[3] = {INFINITY, INFINITY, INFINITY}, Hh[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int sl = 0; sl < S; ++sl) {
      const double* o = part + ((int64_t)c * S + sl) * 6;
      for (int a = 0; a < dim; ++a) {
        L[a] = fmin(L[a], o[a]);
        Hh[a] = fmax(Hh[a], o[3 + a]);
      }
    }
    int axis = 0;
    double best = Hh[0] - L[0];
    for (int a = 1; a < dim; ++a)
      if (Hh[a] - L[a] > best) {
        best = Hh[a] - L[a];
        axis = a;
      }
    if (axis_out) axis_out[c] = axis;
    if (box)
      for (int a = 0; a < 3; ++a) {
        box[a] = a < dim ? L[a] : 0.0;
        box[3 + a] = a < dim ? Hh[a] : 0.0;
      }
  }
}

// keys in ORIGINAL order: the coordinate of point o on its node's axis; values o
__global__ void kd_keys_kernel(const double* __restrict__ X, int dim, const int* __restrict__ segid_orig,
                               const int* __restrict__ axis, int n, uint64_t* __restrict__ keys, int* __restrict__ vals) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    keys[o] = ord_key(X[(int64_t)o * dim + axis[segid_orig[o]]]);
    vals[o] = o;
  }
}

// node ids in the coordinate order (key of the second, stable, sort)
__global__ void kd_gather_segid_kernel(const int* __restrict__ segid_orig, const int* __restrict__ vals, int n,
                                       unsigned* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) out[p] = (unsigned)segid_orig[vals[p]];
}

__global__ void kd_finish_kernel(const double* __restrict__ X, int dim, const int* __restrict__ idx, int n,
                                 double* __restrict__ xt, double* __restrict__ yt, double* __restrict__ zt,
                                 int* __restrict__ iota) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const double* x = X + (int64_t)idx[p] * dim;
    xt[p] = x[0];
    yt[p] = dim > 1 ? x[1] : 0.0;
    zt[p] = dim > 2 ? x[2] : 0.0;
    iota[p] = p;
  }
}

__global__ void kd_iota_kernel(int* v, int n) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) v[p] = p;
}

}  // namespace

// Device KD ordering.  X: host coordinates (n x dim, original order); seg_all: the node ranges of
// depths 0..Dl-1 concatenated (depth t: 2^t + 1 offsets).  Outputs (cudaMalloc'd, owned by the
// caller): perm_dev (tree index -> original index), xt / yt / zt (tree order, zero-padded),
// iota_dev, from the block cache (free them with cache_free); root_box[6] (host) = the bounding box.
void kd_order_device(const double* X, int64_t n64, int dim, int Dl, const std::vector<int>& seg_all, int** perm_dev,
                     double** xt, double** yt, double** zt, int** iota_dev, double* root_box, cudaStream_t st) {
  const int n = (int)n64;
  double* dX = static_cast<double*>(cache_alloc(sizeof(double) * (size_t)n * dim, st));
  H2_CUDA(cudaMemcpyAsync(dX, X, sizeof(double) * (size_t)n * dim, cudaMemcpyHostToDevice, st));
  int* seg = static_cast<int*>(cache_alloc(sizeof(int) * std::max<size_t>(seg_all.size(), 1), st));
  if (!seg_all.empty())
    H2_CUDA(cudaMemcpyAsync(seg, seg_all.data(), sizeof(int) * seg_all.size(), cudaMemcpyHostToDevice, st));
  int* idx = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)n, st));      // current order
  int* val[2];
  uint64_t* key[2];
  unsigned* sk[2];
  for (int q = 0; q < 2; ++q) {
    val[q] = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)n, st));
    key[q] = static_cast<uint64_t*>(cache_alloc(sizeof(uint64_t) * (size_t)n, st));
    sk[q] = static_cast<unsigned*>(cache_alloc(sizeof(unsigned) * (size_t)n, st));
  }
  int* segid = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)n, st));
  int* axis = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)(Dl > 0 ? 1 << (Dl - 1) : 1), st));
  double* dbox = static_cast<double*>(cache_alloc(sizeof(double) * 6, st));
  const int grid1 = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  kd_iota_kernel<<<grid1, 256, 0, st>>>(idx, n);
  H2_CHECK_LAUNCH();
  size_t tmp_bytes = 0;   // CUB scratch, grown to the largest requirement met
  void* tmp = nullptr;
  auto scratch = [&](size_t need) {
    if (tmp && need <= tmp_bytes) return;
    if (tmp) cache_free(tmp, st);
    tmp_bytes = std::max<size_t>(need, 16);
    tmp = cache_alloc(tmp_bytes, st);
  };
  // node boxes -> axes: one CTA per node when there are many nodes, else S CTAs per node and a
  // merge (the top depths hold few nodes of up to n points)
  const int SMAX = 296;
  double* part = static_cast<double*>(cache_alloc(sizeof(double) * 6 * SMAX, st));
  auto boxes = [&](const int* sg, int nseg, int* ax, double* box) {
    if (nseg >= 148) {
      kd_level_kernel<<<std::min(nseg, 148 * 8), 256, 0, st>>>(dX, dim, sg, nseg, idx, ax, box);
    } else {
      const int S = SMAX / nseg;
      kd_box_partial_kernel<<<dim3(S, nseg), 256, 0, st>>>(dX, dim, sg, idx, S, part);
      H2_CHECK_LAUNCH();
      kd_axis_kernel<<<1, 256, 0, st>>>(part, nseg, S, dim, ax, box);
    }
    H2_CHECK_LAUNCH();
  };
  {   // the root box (the diameter; also the only "level" when Dl = 0)
    std::vector<int> root{0, n};
    int* rseg = static_cast<int*>(cache_alloc(sizeof(int) * 2, st));
    H2_CUDA(cudaMemcpyAsync(rseg, root.data(), sizeof(int) * 2, cudaMemcpyHostToDevice, st));
    boxes(rseg, 1, nullptr, dbox);
    cache_free(rseg, st);
  }
  size_t off = 0;
  for (int t = 0; t < Dl; ++t) {
    const int nseg = 1 << t;
    const int* sg = seg + off;
    boxes(sg, nseg, axis, nullptr);   // (1) axes
    kd_segid_kernel<<<grid1, 256, 0, st>>>(sg, nseg, idx, n, segid);
    H2_CHECK_LAUNCH();
    kd_keys_kernel<<<grid1, 256, 0, st>>>(dX, dim, segid, axis, n, key[0], val[0]);
    H2_CHECK_LAUNCH();
    // (2) stable by coordinate from the original order, then stable by node id
    size_t tb = 0;
    H2_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key[0], key[1], val[0], val[1], n, 0, 64, st));
    scratch(tb);
    H2_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key[0], key[1], val[0], val[1], n, 0, 64, st));
    kd_gather_segid_kernel<<<grid1, 256, 0, st>>>(segid, val[1], n, sk[0]);
    H2_CHECK_LAUNCH();
    const int bits = t == 0 ? 1 : t;
    tb = 0;
    H2_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, sk[0], sk[1], val[1], idx, n, 0, bits, st));
    scratch(tb);
    H2_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, sk[0], sk[1], val[1], idx, n, 0, bits, st));
    off += (size_t)nseg + 1;
  }
  // the tree's order arrays come from the block cache (h2_tree::order_cached): no cudaMalloc /
  // cudaFree per tree (their driver latency varied by 1-20 ms in the end-to-end loop)
  *perm_dev = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)std::max(n, 1), st));
  *xt = static_cast<double*>(cache_alloc(sizeof(double) * (size_t)std::max(n, 1), st));
  *yt = static_cast<double*>(cache_alloc(sizeof(double) * (size_t)std::max(n, 1), st));
  *zt = static_cast<double*>(cache_alloc(sizeof(double) * (size_t)std::max(n, 1), st));
  *iota_dev = static_cast<int*>(cache_alloc(sizeof(int) * (size_t)std::max(n, 1), st));
  H2_CUDA(cudaMemcpyAsync(*perm_dev, idx, sizeof(int) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  kd_finish_kernel<<<grid1, 256, 0, st>>>(dX, dim, idx, n, *xt, *yt, *zt, *iota_dev);
  H2_CHECK_LAUNCH();
  H2_CUDA(cudaMemcpyAsync(root_box, dbox, sizeof(double) * 6, cudaMemcpyDeviceToHost, st));
  H2_CUDA(cudaStreamSynchronize(st));
  if (tmp) cache_free(tmp, st);
  for (int q = 0; q < 2; ++q) {
    cache_free(val[q], st);
    cache_free(key[q], st);
    cache_free(sk[q], st);
  }
  cache_free(idx, st);
  cache_free(segid, st);
  cache_free(axis, st);
  cache_free(dbox, st);
  cache_free(part, st);
  cache_free(seg, st);
  cache_free(dX, st);
}

}  // namespace h2
