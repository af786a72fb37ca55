// Exact-order mode (h2_build_opts.exact_order; SURVEY §8(c) parity contract 2):
// kernels that perform every floating-point operation of Algorithm 1 in the
// order the exact-order specification states -- sequential fma chains, correctly rounded
// division / sqrt, no tensor cores, no tree reductions -- so that with the rational test kernel
// and the exactly representable Omega stream the H^2 matrix (ranks, skeletons, U/E, B, D,
// certificates) is bitwise the one the CPU reference computes.  Compiled with --fmad=false: no
// multiply-add is ever contracted; every fused operation is an explicit fma().
// The production kernels (sketch_tc.cu, gen_bsr.cu, cpqr.cu) compute the same quantities with
// tensor cores and parallel reductions; this file is the bit-reproducible path, slow by design
// (one thread per output element, sequential inner loops), meant for N <= a few thousand.
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

template <int KIND>
__device__ __forceinline__ double k_exact(double xi, double yi, double zi, double xj, double yj, double zj,
                                          double param, double l2) {
  const double r2 = r2_exact(xi, yi, zi, xj, yj, zj);
  if (KIND == H2_K_RATIONAL) return k_rational(r2, l2);
  if (KIND == H2_K_EXP) return exp(-sqrt(r2) / param);
  if (r2 == 0.0) return 0.0;
  const double r = sqrt(r2);
  return cos(param * r) / r;
}

// Y(i - row0, j) = fma-chain over k = 0..n-1 of K(i, k) Om(k, j), from 0 (one thread per entry)
template <int KIND>
__global__ void __launch_bounds__(128) exact_sketch_kernel(const double* __restrict__ X, const double* __restrict__ Yc,
                                                           const double* __restrict__ Zc, int64_t n, int64_t row0,
                                                           int64_t row1, const double* __restrict__ Om, int64_t ldo,
                                                           int nc, double* __restrict__ Y, int64_t ldy, double param,
                                                           double l2) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (row1 - row0) * nc) return;
  const int64_t i = row0 + t / nc;
  const int j = (int)(t % nc);
  const double xi = X[i], yi = Yc[i], zi = Zc[i];
  double s = 0.0;
  for (int64_t k = 0; k < n; ++k) s = fma(k_exact<KIND>(xi, yi, zi, X[k], Yc[k], Zc[k], param, l2), Om[k * ldo + j], s);
  Y[(i - row0) * ldy + j] = s;
}

void launch_exact_sketch(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                         int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Y, int64_t ldy,
                         cudaStream_t st) {
  if (row1 <= row0 || ncols <= 0) return;
  const int64_t tot = (row1 - row0) * ncols;
  const int grid = div_up(tot, 128);
  if (kp.kind == H2_K_RATIONAL)
    exact_sketch_kernel<H2_K_RATIONAL><<<grid, 128, 0, st>>>(X, Yc, Zc, n, row0, row1, Om, ldo, ncols, Y, ldy, kp.param, kp.l2);
  else if (kp.kind == H2_K_EXP)
    exact_sketch_kernel<H2_K_EXP><<<grid, 128, 0, st>>>(X, Yc, Zc, n, row0, row1, Om, ldo, ncols, Y, ldy, kp.param, kp.l2);
  else
    exact_sketch_kernel<H2_K_HELMHOLTZ><<<grid, 128, 0, st>>>(X, Yc, Zc, n, row0, row1, Om, ldo, ncols, Y, ldy, kp.param,
                                                             kp.l2);
  H2_CHECK_LAUNCH();
}

// ||Y||_F^2: per leaf c, p_c = fma-chain over rows ascending, columns ascending of y^2
__global__ void exact_sumsq_leaf_kernel(const double* __restrict__ Y, const int64_t* __restrict__ leaf_begin, int cb,
                                        int ce, int64_t ld, int c0, int c1, double* __restrict__ part) {
  const int c = cb + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ce) return;
  double p = 0.0;
  for (int64_t i = leaf_begin[c]; i < leaf_begin[c + 1]; ++i)
    for (int j = c0; j < c1; ++j) p = fma(Y[i * ld + j], Y[i * ld + j], p);
  part[c] = p;
}
// draw total = ((p_0 + p_1) + ...) over leaves ascending; acc = acc + total
__global__ void exact_sumsq_total_kernel(const double* __restrict__ part, int nleaf, double* acc, int* flag) {
  double tot = 0.0;
  for (int c = 0; c < nleaf; ++c) tot = tot + part[c];
  acc[0] = acc[0] + tot;
  if (!isfinite(tot)) *flag = 1;
}

void launch_exact_sumsq_leaf(const double* Y, const int64_t* leaf_begin, int cb, int ce, int64_t ld, int c0, int c1,
                             double* part, cudaStream_t st) {
  if (ce <= cb || c1 <= c0) return;
  exact_sumsq_leaf_kernel<<<div_up(ce - cb, 128), 128, 0, st>>>(Y, leaf_begin, cb, ce, ld, c0, c1, part);
  H2_CHECK_LAUNCH();
}
void launch_exact_sumsq_total(const double* part, int nleaf, double* acc, int* nonfinite, cudaStream_t st) {
  exact_sumsq_total_kernel<<<1, 1, 0, st>>>(part, nleaf, acc, nonfinite);
  H2_CHECK_LAUNCH();
}

// BSR: Y(i, j) = Y(i, j) - s_b for partners b ascending, s_b = fma-chain over k ascending of
// Blk(i, k) Om(k, j) from 0.  CTA per cluster, thread per (row, column).
__global__ void __launch_bounds__(256) exact_bsr_kernel(BsrArgs a) {
  const int c = a.c_begin + blockIdx.x;
  const int mc = a.cnt[c];
  for (int e = threadIdx.x; e < mc * a.ncols; e += blockDim.x) {
    const int i = e / a.ncols, j = a.c0 + e % a.ncols;
    double* yp = a.Y + (a.yoff[c] + i) * a.ldy + j;
    double y = *yp;
    for (int q = a.ptr[c]; q < a.ptr[c + 1]; ++q) {
      const int b = a.idx[q];
      const int u = a.uidx ? a.uidx[q] : q;
      const bool direct = a.tmode == 0 ? a.us[u] == c : a.tmode == 1;
      const int mb = a.kcnt ? a.kcnt[b] : a.cnt[b];
      const double* B = a.blk + a.blk_off[u];
      const double* om = a.Om + a.ooff[b] * a.ldo + j;
      double s = 0.0;
      for (int k = 0; k < mb; ++k) s = fma(direct ? B[(int64_t)i * mb + k] : B[(int64_t)k * mc + i], om[k * a.ldo], s);
      y = y - s;
    }
    *yp = y;
  }
}

void launch_exact_bsr(const BsrArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0 || a.ncols <= 0) return;
  exact_bsr_kernel<<<a.nclusters, 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

// CPQR of A = (Y^loc)^T (R12-R14) in the stated order; CTA per panel, the panel in W (row j =
// column j of A, ld = d).  Sequential decisions (pivot, reflector) by thread 0; per-column
// chains (norms, reflector application) by one thread each.
__global__ void __launch_bounds__(128) exact_cpqr_kernel(CpqrArgs a) {
  extern __shared__ double sm[];
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c], d = a.d;
  double* nrm = sm;                       // max_m
  double* v = nrm + a.max_m;              // d
  int* perm = (int*)(v + d);              // max_m
  __shared__ double s_tau, s_den, s_beta, s_gap, s_margin;
  __shared__ int s_stop, s_piv, s_k;
  const int64_t off = a.poff[c];
  double* A = a.W + off * d;
  for (int64_t e = threadIdx.x; e < (int64_t)m * d; e += blockDim.x) {
    const int64_t j = e / d;
    A[e] = a.Y[(off + j) * a.ldy + (e - j * d)];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    double q = 0.0;
    for (int r = 0; r < d; ++r) q = fma(A[(int64_t)j * d + r], A[(int64_t)j * d + r], q);
    nrm[j] = sqrt(q);
    perm[j] = j;
  }
  if (threadIdx.x == 0) {
    s_gap = INFINITY;
    s_margin = INFINITY;
    s_k = 0;
  }
  __syncthreads();
  const int kfull = min(d, m);
  const int kcap = a.kmax > 0 ? min(kfull, a.kmax) : kfull;
  for (int i = 0;; ++i) {
    if (i >= m) break;
    if (threadIdx.x == 0) {
      double bv = -1.0, sv = -1.0;
      int bi = i;
      for (int j = i; j < m; ++j) {
        if (nrm[j] > bv) {
          sv = fmax(sv, bv);
          bv = nrm[j];
          bi = j;
        } else {
          sv = fmax(sv, nrm[j]);
        }
      }
      if (a.eps > 0 && i < kfull) s_margin = fmin(s_margin, fabs(bv - a.eps) / a.eps);
      s_stop = (i == kcap || !(bv > a.eps)) ? 1 : 0;
      if (s_stop) {
        s_k = i;
      } else {
        if (sv >= 0) s_gap = fmin(s_gap, (bv - sv) / bv);
        s_piv = bi;
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int p = s_piv;
    double* Ai = A + (int64_t)i * d;
    if (p != i) {
      double* Ap = A + (int64_t)p * d;
      for (int r = threadIdx.x; r < d; r += blockDim.x) {
        const double x = Ai[r];
        Ai[r] = Ap[r];
        Ap[r] = x;
      }
      if (threadIdx.x == 0) {
        const int q = perm[i];
        perm[i] = perm[p];
        perm[p] = q;
        const double x = nrm[i];
        nrm[i] = nrm[p];
        nrm[p] = x;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double x2 = 0.0;
      for (int r = i + 1; r < d; ++r) x2 = fma(Ai[r], Ai[r], x2);
      const double alpha = Ai[i];
      const double xnorm = sqrt(x2);
      double tau, beta;
      if (xnorm == 0.0) {
        tau = 0.0;
        beta = alpha;
      } else {
        const double h = sqrt(fma(alpha, alpha, x2));
        beta = alpha < 0.0 ? h : -h;
        tau = (beta - alpha) / beta;
      }
      s_tau = tau;
      s_beta = beta;
      s_den = alpha - beta;
    }
    __syncthreads();
    const double tau = s_tau, den = s_den;
    for (int r = i + 1 + threadIdx.x; r < d; r += blockDim.x) {
      v[r] = tau != 0.0 ? Ai[r] / den : 0.0;
      Ai[r] = 0.0;
    }
    if (threadIdx.x == 0) {
      v[i] = 1.0;
      Ai[i] = s_beta;
    }
    __syncthreads();
    for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) {
      double* Aj = A + (int64_t)j * d;
      double w = 0.0;
      for (int r = i; r < d; ++r) w = fma(v[r], Aj[r], w);
      w = w * tau;
      double q = 0.0;
      for (int r = i; r < d; ++r) {
        const double x = fma(-w, v[r], Aj[r]);
        Aj[r] = x;
        if (r > i) q = fma(x, x, q);
      }
      nrm[j] = sqrt(q);
    }
    if (threadIdx.x == 0) s_k = i + 1;
    __syncthreads();
  }
  __syncthreads();
  for (int j = threadIdx.x; j < m; j += blockDim.x) a.perm[off + j] = perm[j];
  if (threadIdx.x == 0) {
    a.k[c] = s_k;
    a.cert[2 * c] = s_gap;
    a.cert[2 * c + 1] = s_margin;
  }
}

void launch_exact_cpqr(const CpqrArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  const size_t sm = sizeof(double) * (a.max_m + a.d) + sizeof(int) * a.max_m;
  H2_CUDA(cudaFuncSetAttribute(exact_cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  H2_REQUIRE(sm <= 200 * 1024, "exact-order CPQR: panel too large for the exact-order mode");
  exact_cpqr_kernel<<<a.nclusters, 128, sm, st>>>(a);
  H2_CHECK_LAUNCH();
}

// ID (R15): T(:, cc) by back substitution in the stated order, written in place into the basis
// row X(Rhat_cc, :); identity rows X(J_i, :) = e_i; skeletons I~ = Ibar[J]
__global__ void __launch_bounds__(128) exact_id_kernel(IdArgs a) {
  const int c = a.c_begin + blockIdx.x;
  const int m = a.m[c], k = a.k[c], d = a.d;
  const int64_t off = a.poff[c];
  const double* A = a.W + off * d;        // R(i, j) = A[j * d + i]
  const int* perm = a.perm + off;
  double* X = a.X + a.xoff[c];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, q = e % k;
    X[(int64_t)perm[i] * k + q] = q == i ? 1.0 : 0.0;
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) a.skel[a.roff[c] + i] = a.ibar[off + perm[i]];
  for (int cc = threadIdx.x; cc < m - k; cc += blockDim.x) {
    double* row = X + (int64_t)perm[k + cc] * k;
    for (int i = k - 1; i >= 0; --i) {
      double s = A[(int64_t)(k + cc) * d + i];
      for (int j = i + 1; j < k; ++j) s = fma(-A[(int64_t)j * d + i], row[j], s);
      row[i] = s / A[(int64_t)i * d + i];
    }
  }
}

void launch_exact_id(const IdArgs& a, cudaStream_t st) {
  if (a.nclusters <= 0) return;
  exact_id_kernel<<<a.nclusters, 128, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

}  // namespace h2
