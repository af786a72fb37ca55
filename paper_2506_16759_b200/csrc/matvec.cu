// H^2 matvec pieces (upward pass x^ = U^T x / E^T x^, downward pass y = U y^ / E y^), used by
// h2_matvec for verification (PAPER.md L440 uses an H^2 matvec as K_blk; L447 error check).
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// xh(roff+i, q) = sum_j X(j, i) xin(ioff+j, q); one CTA per cluster, thread per (i, q)
__global__ void __launch_bounds__(256) upward_kernel(UpArgs a) {
  const int c = blockIdx.x;
  const int m = a.m[c], k = a.k[c];
  const double* X = a.X + a.xoff[c];
  const double* xin = a.xin + a.ioff[c] * a.ldi;
  double* xh = a.xh + a.roff[c] * a.ldh;
  for (int e = threadIdx.x; e < k * a.q; e += blockDim.x) {
    const int i = e / a.q, q = e % a.q;
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(X[(int64_t)j * k + i], xin[(int64_t)j * a.ldi + q], s);
    xh[(int64_t)i * a.ldh + q] = s;
  }
}

void launch_upward(const UpArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  upward_kernel<<<a.nclusters, 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

// yout(ioff+j, q) (+)= alpha * sum_i X(j, i) yh(roff+i, q)
__global__ void __launch_bounds__(256) downward_kernel(DownArgs a) {
  const int c = blockIdx.x;
  const int m = a.m[c], k = a.k[c];
  const double* X = a.X + a.xoff[c];
  const double* yh = a.yh + a.roff[c] * a.ldh;
  double* y = a.yout + a.ioff[c] * a.ldo;
  for (int e = threadIdx.x; e < m * a.q; e += blockDim.x) {
    const int j = e / a.q, q = e % a.q;
    double s = 0.0;
    for (int i = 0; i < k; ++i) s = fma(X[(int64_t)j * k + i], yh[(int64_t)i * a.ldh + q], s);
    double* o = y + (int64_t)j * a.ldo + q;
    *o = a.accumulate ? fma(a.alpha, s, *o) : a.alpha * s;
  }
}

void launch_downward(const DownArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  downward_kernel<<<a.nclusters, 256, 0, st>>>(a);
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

}  // namespace h2
