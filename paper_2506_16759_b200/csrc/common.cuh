// Internal helpers of libh2 (CUDA path only; never shared with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/h2.h"

namespace h2 {

// ---------------------------------------------------------------------------------------
// error plumbing: internal code throws h2::Error, the C ABI converts it to a status code
// ---------------------------------------------------------------------------------------
struct Error : std::runtime_error {
  h2_status status;
  Error(h2_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define H2_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::h2::Error(e_ == cudaErrorMemoryAllocation ? H2_ERR_OOM : H2_ERR_CUDA,         \
                        std::string(#call) + ": " + cudaGetErrorString(e_) + " @" __FILE__ \
                        ":" + std::to_string(__LINE__));                                   \
  } while (0)

void count_launch();  // api.cpp: per-thread kernel launch counter (h2_build_stats.launches)
#define H2_CHECK_LAUNCH()     \
  do {                        \
    ::h2::count_launch();     \
    H2_CUDA(cudaGetLastError()); \
  } while (0)

#define H2_REQUIRE(cond, msg) \
  do {                        \
    if (!(cond)) throw ::h2::Error(H2_ERR_INVALID_ARG, msg); \
  } while (0)

// ---------------------------------------------------------------------------------------
// built-in kernels (§V-A): K(x,y) as a function of r^2 = |x-y|^2
// ---------------------------------------------------------------------------------------
struct KernelParams {
  int kind;
  double param;   // l (exp) or k (helmholtz)
  double inv;     // 1/l for exp
  double rmax;    // upper bound of the scaled distance over the point set (|x-y|/l, k|x-y|); 0 = unknown
  double rmin;    // minimum distance of distinct points (unscaled; Helmholtz fixed-point scale); 0 = unknown
  double l2;      // param^2 (rational test kernel)
};

inline KernelParams make_kernel(const h2_kernel& k, double diam = -1.0, double rmin = 0.0) {
  KernelParams p;
  p.kind = k.kind;
  p.param = k.param;
  p.inv = 1.0 / k.param;
  p.rmax = diam >= 0 ? diam * (k.kind == H2_K_EXP ? p.inv : k.param) : 0.0;
  p.rmin = rmin;
  p.l2 = k.param * k.param;
  return p;
}

// Rational test kernel K = 1 / (1 + r^2 / l^2), r^2 = (dx*dx + dy*dy) + dz*dz, every operation
// correctly rounded and never contracted (explicit _rn intrinsics): bitwise the value the C
// oracle computes (DESIGN.md §3 exact-order specification; H2_K_RATIONAL).
__device__ __forceinline__ double r2_exact(double xi, double yi, double zi, double xj, double yj, double zj) {
  const double dx = __dadd_rn(xi, -xj), dy = __dadd_rn(yi, -yj), dz = __dadd_rn(zi, -zj);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}
__device__ __forceinline__ double k_rational(double r2, double l2) {
  return __ddiv_rn(1.0, __dadd_rn(1.0, __ddiv_rn(r2, l2)));
}

// exp(x) for x <= 0 in ~10 FP64 pipe operations (libdevice exp costs ~2.5x more, measured):
// x = (n/64) ln2 + g with n = rint(64 x / ln2) (shifter trick), Cody-Waite 2-term reduction
// (fdlibm ln2 split; |n| < 2^17 keeps kf*hi exact), |g| <= ln2/128, e^g by the degree-5 Taylor
// polynomial (truncation 3.5e-17 relative), 2^(j/64) from a 64-entry table `tab`, 2^(n>>6) by
// exponent arithmetic.  Max error ~1.5 ulp.  x < -700 -> 0 (true value < 1e-304).
// The non-short constants are passed as register values (ExpNegC) that a kernel loads ONCE from
// shared memory (exp_neg_consts_fill / _load): as literals, the compiler rematerialises each
// 64-bit constant with two integer MOVs (or an LDC) per evaluation, and the batchedGen loop was
// issue-bound on them.
struct ExpNegC {
  double c[6];
};
__device__ __forceinline__ void exp_neg_consts_fill(double* sk) {
  const double v[6] = {92.332482616893656,        // 64/ln2
                       -0.01083042469326756,      // ln2_hi/64 (fdlibm 0x3fe62e42fee00000)
                       -2.9815858269852933e-12,   // ln2_lo/64 (fdlibm 0x3dea39ef35793c76)
                       1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0};
  if (threadIdx.x < 6) sk[threadIdx.x] = v[threadIdx.x];
}
__device__ __forceinline__ ExpNegC exp_neg_consts_load(const double* sk) {
  ExpNegC k;
#pragma unroll
  for (int i = 0; i < 6; ++i) k.c[i] = sk[i];
  return k;
}
__device__ __forceinline__ double exp_neg(double x, const double* __restrict__ tab, const ExpNegC& k) {
  const double SH = 6755399441055744.0;                 // 1.5 * 2^52
  double t = fma(x, k.c[0], SH);
  double kf = t - SH;
  int n = __double2loint(t);
  double g = fma(kf, k.c[1], x);
  g = fma(kf, k.c[2], g);
  double p = fma(g, k.c[3], k.c[4]);
  p = fma(p, g, k.c[5]);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
  double r = tab[n & 63] * p;
  r = __hiloint2double(__double2hiint(r) + ((n >> 6) << 20), __double2loint(r));
  return x < -700.0 ? 0.0 : r;
}

// ---------------------------------------------------------------------------------------
// Sketch-path evaluation in SCALED coordinates x' = x*cs (cs = 1/l for exp, k for Helmholtz),
// so r' = |x'-y'| is the kernel argument directly.  FP64-pipe cost per entry (SASS):
//   r'^2: 6 (3 DADD, DMUL, 2 DFMA);  1/r' : MUFU.RSQ64H + 4 (one cubic correction, ~1 ulp,
//   as libdevice rsqrt);  r' = r'^2/r': 1;  exp(-r'): 7 (shifter, 1-term Cody-Waite, degree-4
//   polynomial on |g| <= ln2/512, 256-entry table, exponent arithmetic).
// Absolute error <= ~2e-16 for exp entries (the 1-term reduction error kf*d(ln2/256) is damped
// by e^{-r'}); the sketch only needs rounding-level accuracy in absolute terms.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y * y, 1.0);
  double p = fma(e, 0.375, 0.5);
  return fma(p, y * e, y);
}

// exp(-r) for r >= 0 with a 256-entry table of 2^(j/256)
__device__ __forceinline__ double exp_neg256(double r, const double* __restrict__ tab) {
  const double SH = 6755399441055744.0;                  // 1.5 * 2^52
  double t = fma(r, -369.32993046757464, SH);            // -256/ln2
  double kf = t - SH;
  int n = __double2loint(t);                             // n = rint(-256 r / ln2) <= 0
  double g = fma(kf, -0.0027076061740622863, -r);        // -r - kf ln2/256, |g| <= ln2/512
  double p = fma(g, 1.0 / 24.0, 1.0 / 6.0);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
  double v = tab[n & 255] * p;
  v = __hiloint2double(__double2hiint(v) + ((n >> 8) << 20), __double2loint(v));
  return n < -256 * 1000 ? 0.0 : v;
}

__device__ __forceinline__ void fill_exp_table256(double* tab) {
  for (int j = threadIdx.x; j < 256; j += blockDim.x) tab[j] = exp2((double)j * (1.0 / 256.0));
}

// K(r') in scaled coordinates; r2 = r'^2.  exp: e^{-r'};  Helmholtz: k cos(r')/r' (0 at r' = 0)
template <int KIND>
__device__ __forceinline__ double kernel_scaled(double r2, double k, const double* __restrict__ tab) {
  const bool zero = __double2hiint(r2) < 0x00100000;     // r2 < 2^-1022 (incl. 0): integer test
  double y = rsqrt_fast(zero ? 1.0 : r2);
  if (KIND == H2_K_EXP) {
    double r = zero ? 0.0 : r2 * y;
    return exp_neg256(r, tab);
  } else {
    double r = r2 * y;
    return zero ? 0.0 : k * cos(r) * y;
  }
}

// 2^(j/64), j < 64, filled once per CTA (libdevice exp2, < 1 ulp)
__device__ __forceinline__ void fill_exp_table(double* tab) {
  for (int j = threadIdx.x; j < 64; j += blockDim.x) tab[j] = exp2((double)j * (1.0 / 64.0));
}

template <int KIND>
__device__ __forceinline__ double kernel_of_r2(double r2, double param, double inv, const double* tab,
                                               const ExpNegC& ek) {
  if (KIND == H2_K_EXP) {
    // exp(-|x-y|/l)  (PAPER.md Eq. cov)
    return exp_neg(-sqrt(r2) * inv, tab, ek);
  } else {
    double r = sqrt(r2);
    return r2 > 0.0 ? cos(param * r) / r : 0.0;
  }
}

template <int KIND>
__device__ __forceinline__ double kernel_of_r2(double r2, double param, double inv) {
  if (KIND == H2_K_EXP) {
    // exp(-|x-y|/l)  (PAPER.md Eq. cov)
    return exp(-sqrt(r2) * inv);
  } else {
    // cos(k|x-y|)/|x-y|, 0 at x = y  (PAPER.md Eq. ie; R20)
    double r = sqrt(r2);
    return r2 > 0.0 ? cos(param * r) / r : 0.0;
  }
}

__device__ __forceinline__ double dist2(double xi, double yi, double zi, double xj, double yj, double zj) {
  double dx = xi - xj, dy = yi - yj, dz = zi - zj;
  return fma(dz, dz, fma(dy, dy, dx * dx));
}

// ---------------------------------------------------------------------------------------
// FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a; no tcgen05 .kind::f64 exists)
// A: 8x4 row, one element per lane: A[lane>>2][lane&3]
// B: 4x8 col, one element per lane: B[lane&3][lane>>2]
// C: 8x8, two elements per lane: C[lane>>2][2*(lane&3) + {0,1}]
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace h2
