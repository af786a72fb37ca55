// H^2 matvec pieces (upward pass x^ = U^T x / E^T x^, downward pass y = U y^ / E y^), used by
// h2_matvec for verification (PAPER.md L440 uses an H^2 matvec as K_blk; L447 error check).
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// Upward / downward passes: per cluster small dense products X^T xin (k x q) and X yh (m x q).
// CTA = (cluster, 32 output rows); lanes = right-hand-side columns (coalesced), each warp 4
// output rows with 4 independent accumulators (the X entries are warp-uniform broadcasts).  The
// top levels hold few clusters with k ~ 200-600: spreading the rows over CTAs fills the GPU
// (one CTA per cluster before: 62 -> 36 ms per 32-column matvec of an N = 2^18 H^2 at 1e-8).
constexpr int MV_ROWS = 32;

// xh(roff+i, q) = sum_j X(j, i) xin(ioff+j, q)
__global__ void __launch_bounds__(256) upward_kernel(UpArgs a) {
  const int c = blockIdx.x;
  const int m = a.m[c], k = a.k[c];
  const int i0 = blockIdx.y * MV_ROWS + (threadIdx.x >> 5) * 4;
  if (blockIdx.y * MV_ROWS >= k) return;
  const double* X = a.X + a.xoff[c];
  const double* xin = a.xin + a.ioff[c] * a.ldi;
  double* xh = a.xh + a.roff[c] * a.ldh;
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < a.q; q += 32) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int j = 0; j < m; ++j) {
      const double x = xin[(int64_t)j * a.ldi + q];
      const double* Xj = X + (int64_t)j * k + i0;
      if (i0 < k) s0 = fma(Xj[0], x, s0);
      if (i0 + 1 < k) s1 = fma(Xj[1], x, s1);
      if (i0 + 2 < k) s2 = fma(Xj[2], x, s2);
      if (i0 + 3 < k) s3 = fma(Xj[3], x, s3);
    }
    if (i0 < k) xh[(int64_t)i0 * a.ldh + q] = s0;
    if (i0 + 1 < k) xh[(int64_t)(i0 + 1) * a.ldh + q] = s1;
    if (i0 + 2 < k) xh[(int64_t)(i0 + 2) * a.ldh + q] = s2;
    if (i0 + 3 < k) xh[(int64_t)(i0 + 3) * a.ldh + q] = s3;
  }
}

void launch_upward(const UpArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  const int rows = a.max_out > 0 ? a.max_out : 1024;
  upward_kernel<<<dim3(a.nclusters, div_up(rows, MV_ROWS)), 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

// yout(ioff+j, q) (+)= alpha * sum_i X(j, i) yh(roff+i, q)
__global__ void __launch_bounds__(256) downward_kernel(DownArgs a) {
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c], k = a.k[c];
  const int j0 = blockIdx.y * MV_ROWS + (threadIdx.x >> 5) * 4;
  if (blockIdx.y * MV_ROWS >= m) return;
  const double* X = a.X + a.xoff[c];
  const double* yh = a.yh + a.roff[c] * a.ldh;
  double* y = a.yout + a.ioff[c] * a.ldo;
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < a.q; q += 32) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < k; ++i) {
      const double h = yh[(int64_t)i * a.ldh + q];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (j0 + r < m) s[r] = fma(X[(int64_t)(j0 + r) * k + i], h, s[r]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (j0 + r >= m) continue;
      double* o = y + (int64_t)(j0 + r) * a.ldo + q;
      *o = a.accumulate ? fma(a.alpha, s[r], *o) : a.alpha * s[r];
    }
  }
}

void launch_downward(const DownArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  const int rows = a.max_out > 0 ? a.max_out : 1024;
  downward_kernel<<<dim3(a.nclusters, div_up(rows, MV_ROWS)), 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

__global__ void scale_kernel(double* y, int64_t n, int64_t ld, int q, double beta) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * q; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / q;
    double* p = y + r * ld + (e - r * q);
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

void launch_scale(double* y, int64_t n, int64_t ld, int q, double beta, cudaStream_t st) {
  if (n <= 0 || q <= 0) return;
  int grid = (int)std::min<int64_t>((n * q + 255) / 256, 148 * 16);
  scale_kernel<<<grid, 256, 0, st>>>(y, n, ld, q, beta);
  H2_CHECK_LAUNCH();
}


// Row gather / scatter of a row-major panel (the halo exchange of the sharded construction,
// S§8(e)): packed row e <-> panel row rows[e], ncols columns.  dir 0: out[e] = P[rows[e]]
// (pack for sending), dir 1: P[rows[e]] = in[e] (unpack after receiving).
__global__ void __launch_bounds__(256) rows_move_kernel(double* __restrict__ P, int64_t ld, const int32_t* __restrict__ rows,
                                                        int64_t nrows, int ncols, double* __restrict__ buf, int dir) {
  const int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / ncols;
    const int c = (int)(e - r * ncols);
    double* p = P + (int64_t)rows[r] * ld + c;
    if (dir == 0) buf[e] = *p;
    else *p = buf[e];
  }
}

void launch_rows_move(double* P, int64_t ld, const int32_t* rows, int64_t nrows, int ncols, double* buf, int dir,
                      cudaStream_t st) {
  if (nrows <= 0 || ncols <= 0) return;
  const int64_t total = nrows * ncols;
  rows_move_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, st>>>(P, ld, rows, nrows, ncols, buf,
                                                                                        dir);
  H2_CHECK_LAUNCH();
}

}  // namespace h2
