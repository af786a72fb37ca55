// Host-side cluster tree + block partition (§II-A) and their flattened
// per-level CSR batch descriptors (§IV-A "stored contiguously level by level").
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/h2.h"

struct PairCSR {
  // ordered pairs (row s, col b) of one depth, sorted (s, b); symmetric set
  std::vector<int32_t> ptr;    // 2^t + 1
  std::vector<int32_t> idx;    // partner b per ordered pair
  std::vector<int32_t> uidx;   // index of {min(s,b), max(s,b)} in the unique list
  std::vector<int32_t> us, ub; // unique pairs (s <= b for near, s < b for far), sorted
  int64_t nnz() const { return (int64_t)idx.size(); }
  int64_t nuniq() const { return (int64_t)us.size(); }
};

struct DeviceCSR {
  int32_t *ptr = nullptr, *idx = nullptr, *uidx = nullptr, *us = nullptr, *ub = nullptr;
};

struct h2_tree {
  int64_t n = 0;
  int32_t dim = 0, leaf_size = 0, Dl = 0, top = -1, rule = 0, csp = 0;
  double eta = 0;
  std::vector<int64_t> perm;                       // tree index -> original index
  std::vector<std::vector<int64_t>> begin, end;    // per depth
  std::vector<double> xt, yt, zt;                  // tree-order coordinates (zero padded to 3D)
  double diam = 0;                                 // bounding-box diagonal of all points
  double rmin = -1;                                // min distance of distinct points (near pairs), -1 = not computed
  PairCSR near;                                    // leaf depth
  std::vector<PairCSR> far;                        // per depth
  std::vector<int64_t> D_off;                      // unique near pair offsets (m_s*m_b prefix)

  // asynchronous partition (h2_tree_build_async): the KD ordering and tree-order coordinates are
  // ready at return, the block partition (boxes, dual traversal, CSR, D offsets) is built on a
  // host thread; every reader of the partition calls wait_partition() first (it rethrows a
  // partition error).  The first dense-sketch pass of h2_build runs before that wait.
  std::thread part_thread;
  std::mutex part_mu;
  std::string part_error;
  bool part_uploaded = false;
  void wait_partition();

  // near-field chunk lists of the tensor-core leaf subtraction (api.cpp ensure_near_chunks):
  // per leaf, the 128-j chunks holding its near leaves + 2-bit half masks; state 0 = not built,
  // 1 = built (leaves of exactly 64 points at multiples of 64), -1 = tree not eligible
  int nl_state = 0;
  int32_t *d_nl_ptr = nullptr, *d_nl_chunk = nullptr;
  uint8_t* d_nl_mask = nullptr;

  // device mirrors (current device at build time)
  int device = -1;
  double *d_x = nullptr, *d_y = nullptr, *d_z = nullptr;
  int32_t* d_iota = nullptr;                       // 0..n-1
  int32_t* d_perm = nullptr;                       // GPU KD ordering: perm until the partition thread
                                                   // downloads it (then freed)
  int64_t* d_leaf_begin = nullptr;                 // 2^Dl + 1 (last = n)
  int32_t* d_leaf_size = nullptr;
  int64_t* d_D_off = nullptr;
  DeviceCSR d_near;
  std::vector<DeviceCSR> d_far;

  ~h2_tree();
};

void tree_build_host(h2_tree& T, const double* coords, int64_t n, int dim, int leaf, double eta, int rule);
void tree_build_order(h2_tree& T, const double* coords, int64_t n, int dim, int leaf, double eta, int rule);
// the same ordering on the current CUDA device (kd_gpu.cu); device arrays ready at return, the host
// copies (perm, xt/yt/zt) filled by tree_download_order (the partition thread calls it first)
void tree_build_order_gpu(h2_tree& T, const double* coords, int64_t n, int dim, int leaf, double eta, int rule);
void tree_download_order(h2_tree& T);
namespace h2 {
void kd_order_device(const double* X, int64_t n, int dim, int Dl, const std::vector<int>& seg_all, int** perm_dev,
                     double** xt, double** yt, double** zt, int** iota_dev, double* root_box, cudaStream_t st);
}
void tree_build_partition(h2_tree& T);
void tree_upload_order(h2_tree& T);
void tree_upload_partition(h2_tree& T);
void tree_import_host(h2_tree& T, const h2_tree_desc& desc);
void tree_upload(h2_tree& T);
