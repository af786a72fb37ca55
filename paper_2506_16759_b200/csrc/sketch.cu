// batchedRand (PAPER.md L203/L216/L246, L384 "generated in a single kernel") and the built-in
// dense-kernel sketch Y = K Omega (Algorithm 1 line 1 with K_blk = the dense kernel matrix,
// BASELINE configs[1]); plus the sketch-norm reduction used by the tolerance rule (R10).
#include <cublas_v2.h>
#include <mutex>

#include "common.cuh"
#include "alloc.hpp"
#include "kernels.hpp"

#include <cstdlib>

namespace h2 {

// ------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11) -> two centred-binomial entries (R8)
// counter = (row, column pair q, stream id, 0), key = (seed lo, seed hi)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__global__ void omega_kernel(uint2 key, uint32_t sid, int64_t row0, int64_t nrows, int col0, int ncols,
                             double* __restrict__ out, int64_t ld) {
  const int q0 = col0 >> 1;
  const int nq = ((col0 + ncols + 1) >> 1) - q0;
  const int64_t total = nrows * nq;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t / nq;
    int q = q0 + (int)(t - r * nq);
    uint4 w = philox4x32_10(make_uint4((uint32_t)(row0 + r), (uint32_t)q, sid, 0u), key);
    // centred binomial (R8): (popcount of 64 random bits - 32) / 4, exact in FP64 and int8
    const double g0 = (double)(__popc(w.x) + __popc(w.y) - 32) * 0.25;
    const double g1 = (double)(__popc(w.z) + __popc(w.w) - 32) * 0.25;
    int j0 = 2 * q - col0;  // column within the output block
    double* o = out + r * ld;
    if (j0 >= 0 && j0 < ncols) o[j0] = g0;
    if (j0 + 1 >= 0 && j0 + 1 < ncols) o[j0 + 1] = g1;
  }
}

void launch_omega(uint64_t seed, uint32_t sid, int64_t row0, int64_t nrows, int col0, int ncols, double* out,
                  int64_t ld, cudaStream_t st) {
  if (nrows <= 0 || ncols <= 0) return;
  uint2 key = make_uint2((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  int64_t work = nrows * ((ncols + 2) / 2);
  int grid = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
  omega_kernel<<<grid, 256, 0, st>>>(key, sid, row0, nrows, col0, ncols, out, ld);
  H2_CHECK_LAUNCH();
}

// ------------------------------------------------------------------------------------------
// Dense sketch: Y(i, c0:c0+32) = sum_{j in [jb,je)} K(x_i, x_j) Omega(j, c0:c0+32)
// CTA = 4 warps x (8 MB) rows; columns in one 32-wide chunk (4 DMMA n-blocks).  K entries are
// generated in registers directly in the DMMA A-fragment layout (each lane evaluates exactly
// the entries it contributes: no K tile ever touches shared memory or HBM); Omega rows and
// the x_j coordinates are staged in shared memory per 32-row j-chunk (cp.async double buffer).
// The j range may be split over gridDim.y slices (partial sums combined in a fixed order by
// sketch_combine_kernel) to fill the last wave; accumulation order is fixed -> deterministic.
// ------------------------------------------------------------------------------------------
constexpr int SK_JT = 32;       // j rows per smem stage
constexpr int SK_LD = 36;       // padded Omega row stride (doubles), conflict-free B fragments

template <int KIND, int MB, int MINB, int UNR>
__global__ void __launch_bounds__(128, MINB)
    dense_sketch_kernel(const double* __restrict__ X, const double* __restrict__ Yc, const double* __restrict__ Zc,
                        int64_t n, int64_t row0, int64_t row1, const double* __restrict__ Om, int64_t ldo, int ncols,
                        double* __restrict__ Yout, int64_t ldy, int64_t split_stride, double param, double inv,
                        bool aligned) {
  constexpr int WR = 8 * MB;                       // rows per warp
  __shared__ __align__(16) double sOm[2][SK_JT * SK_LD];
  __shared__ double sx[2][SK_JT], sy[2][SK_JT], sz[2][SK_JT];
  __shared__ double tab[256];
  fill_exp_table256(tab);
  // scaled coordinates x' = cs x: the kernel argument is |x'-y'| directly (cs = 1/l or k)
  const double cs = KIND == H2_K_EXP ? inv : param;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rbase = row0 + (int64_t)blockIdx.x * (4 * WR) + warp * WR;
  // j slice of this CTA
  const int64_t nch_all = (n + SK_JT - 1) / SK_JT;
  const int64_t ch_b = nch_all * blockIdx.y / gridDim.y, ch_e = nch_all * (blockIdx.y + 1) / gridDim.y;
  double xi[MB], yi[MB], zi[MB];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    int64_t i = rbase + mb * 8 + (lane >> 2);
    if (i < row1) {
      xi[mb] = X[i] * cs;
      yi[mb] = Yc[i] * cs;
      zi[mb] = Zc[i] * cs;
    } else {
      xi[mb] = yi[mb] = zi[mb] = 0.0;
    }
  }
  double acc[MB][4][2];
#pragma unroll
  for (int a = 0; a < MB; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  auto stage = [&](int64_t ch, int buf) {
    int64_t j0 = ch * SK_JT;
    for (int e = threadIdx.x; e < SK_JT * 16; e += 128) {
      int r = e >> 4, c2 = (e & 15) * 2;
      double* dst = &sOm[buf][r * SK_LD + c2];
      int64_t j = j0 + r;
      if (aligned && j < n && c2 + 1 < ncols) {
        const double* src = Om + j * ldo + c2;
        unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(src));
      } else {
        dst[0] = (j < n && c2 < ncols) ? Om[j * ldo + c2] : 0.0;
        dst[1] = (j < n && c2 + 1 < ncols) ? Om[j * ldo + c2 + 1] : 0.0;
      }
    }
    if (threadIdx.x < SK_JT) {
      int64_t j = j0 + threadIdx.x;
      sx[buf][threadIdx.x] = j < n ? X[j] * cs : 0.0;
      sy[buf][threadIdx.x] = j < n ? Yc[j] * cs : 0.0;
      sz[buf][threadIdx.x] = j < n ? Zc[j] * cs : 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  if (ch_b < ch_e) stage(ch_b, 0);
  for (int64_t ch = ch_b; ch < ch_e; ++ch) {
    const int buf = (int)((ch - ch_b) & 1);
    if (ch + 1 < ch_e) {
      stage(ch + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const int64_t j0 = ch * SK_JT;
    const bool full = j0 + SK_JT <= n;
#pragma unroll UNR
    for (int ks = 0; ks < SK_JT / 4; ++ks) {
      const int jl = ks * 4 + (lane & 3);
      const double xj = sx[buf][jl], yj = sy[buf][jl], zj = sz[buf][jl];
      const bool jvalid = full || (j0 + jl) < n;
      double a[MB];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        double r2 = dist2(xi[mb], yi[mb], zi[mb], xj, yj, zj);
        double v = kernel_scaled<KIND>(r2, param, tab);
        a[mb] = jvalid ? v : 0.0;
      }
      double b[4];
#pragma unroll
      for (int nb = 0; nb < 4; ++nb) b[nb] = sOm[buf][(ks * 4 + (lane & 3)) * SK_LD + nb * 8 + (lane >> 2)];
#pragma unroll
      for (int mb = 0; mb < MB; ++mb)
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) dmma_8x8x4(acc[mb][nb][0], acc[mb][nb][1], a[mb], b[nb]);
    }
    __syncthreads();
  }
  double* Yo = Yout + blockIdx.y * split_stride;
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    int64_t i = rbase + mb * 8 + (lane >> 2);
    if (i >= row1) continue;
    double* y = Yo + (i - row0) * ldy;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      int c = nb * 8 + 2 * (lane & 3);
      if (c < ncols) y[c] = acc[mb][nb][0];
      if (c + 1 < ncols) y[c + 1] = acc[mb][nb][1];
    }
  }
}

// Y(i, c) = sum_{s < S} P_s(i, c), s ascending (fixed order)
__global__ void sketch_combine_kernel(const double* __restrict__ P, int S, int64_t rows, int ncols,
                                      double* __restrict__ Y, int64_t ldy) {
  const int64_t total = rows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / ncols;
    int c = (int)(e - r * ncols);
    double s = P[e];
    for (int q = 1; q < S; ++q) s += P[q * total + e];
    Y[r * ldy + c] = s;
  }
}

void launch_sketch_combine(const double* P, int S, int64_t rows, int ncols, double* Y, int64_t ldy, cudaStream_t st) {
  int g = (int)std::min<int64_t>((rows * ncols + 255) / 256, (int64_t)148 * 16);
  sketch_combine_kernel<<<g, 256, 0, st>>>(P, S, rows, ncols, Y, ldy);
  H2_CHECK_LAUNCH();
}

int env_int(const char* name, int def) {
  const char* v = getenv(name);
  return v ? atoi(v) : def;
}

namespace {

template <int KIND, int MB, int MINB, int UNR>
void sketch_variant(dim3 grid, cudaStream_t st, const double* X, const double* Yc, const double* Zc, int64_t n,
                    int64_t row0, int64_t row1, const double* Om, int64_t ldo, int nc, double* Yo, int64_t ldy,
                    int64_t sstride, const KernelParams& kp, bool aligned) {
  dense_sketch_kernel<KIND, MB, MINB, UNR><<<grid, 128, 0, st>>>(X, Yc, Zc, n, row0, row1, Om, ldo, nc, Yo, ldy,
                                                                 sstride, kp.param, kp.inv, aligned);
}

// (rows-per-lane MB, min CTAs/SM, k-step unroll) variants; index from H2_SK_VAR (tuning)
struct SkVar {
  int rows, occ;   // rows per CTA, resident CTAs per SM
};
constexpr SkVar SK_VARS[] = {{128, 3}, {128, 3}, {128, 4}, {128, 4}, {64, 4}, {64, 5}, {64, 6}};
constexpr int SK_DEFAULT_VAR = 1;

template <int KIND>
void sketch_dispatch(int var, dim3 grid, cudaStream_t st, const double* X, const double* Yc, const double* Zc,
                     int64_t n, int64_t row0, int64_t row1, const double* Om, int64_t ldo, int nc, double* Yo,
                     int64_t ldy, int64_t sstride, const KernelParams& kp, bool aligned) {
#define H2_SKV(MB, MINB, UNR) \
  sketch_variant<KIND, MB, MINB, UNR>(grid, st, X, Yc, Zc, n, row0, row1, Om, ldo, nc, Yo, ldy, sstride, kp, aligned)
  switch (var) {
    case 1: H2_SKV(4, 3, 1); break;
    case 2: H2_SKV(4, 4, 1); break;
    case 3: H2_SKV(4, 4, 2); break;
    case 4: H2_SKV(2, 4, 2); break;
    case 5: H2_SKV(2, 5, 1); break;
    case 6: H2_SKV(2, 6, 1); break;
    default: H2_SKV(4, 3, 2); break;
  }
#undef H2_SKV
}
}  // namespace

void launch_dense_sketch(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                         int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Yout,
                         int64_t ldy, bool omega_quarters, cudaStream_t st) {
  if (row1 <= row0 || ncols <= 0) return;
  if (kp.kind == H2_K_RATIONAL) {   // the exact-order test kernel has only the exact-order sketch
    launch_exact_sketch(kp, X, Yc, Zc, n, row0, row1, Om, ldo, ncols, Yout, ldy, st);
    return;
  }
  // exp kernel with Omega in quarters (the h2 stream): exact int8 tensor-core contraction
  // (sketch_tc.cu); any other Omega, or H2_SK_TC=0, takes the DMMA path
  if (omega_quarters && sketch_tc_supported(kp) && env_int("H2_SK_TC", 1) != 0) {
    if (launch_dense_sketch_tc(kp, X, Yc, Zc, n, row0, row1, Om, ldo, ncols, Yout, ldy, st)) return;
    // a Helmholtz entry exceeded the fixed-point scale: recompute on the FP64 DMMA path
  }
  int var = env_int("H2_SK_VAR", SK_DEFAULT_VAR);
  if (var < 0 || var > 6) var = SK_DEFAULT_VAR;
  const int occ = SK_VARS[var].occ;               // resident CTAs / SM (registers)
  const int64_t rows = row1 - row0;
  const int tiles = div_up(rows, SK_VARS[var].rows);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // j-split S: fill the last wave (efficiency = units / (slots * ceil(units / slots)))
  int S = env_int("H2_SK_SPLIT", 0);
  if (S <= 0) {
    const int slots = sms * occ;
    double best = 0;
    S = 1;
    // chosen from n only (as if all rows were computed): the row shards of a multi-GPU build
    // then split j identically and produce bitwise the same rows as one GPU
    const int64_t tiles_n = div_up(n, SK_VARS[var].rows * 8);   // the 8-GPU row shard (as sketch_tc.cu)
    for (int s = 1; s <= 4; ++s) {
      int64_t units = tiles_n * s;
      if (n / s < 4096 && s > 1) break;
      double eff = (double)units / ((double)slots * ((units + slots - 1) / slots)) - 0.01 * (s - 1);
      if (eff > best + 1e-9) {
        best = eff;
        S = s;
      }
    }
  }
  double* part = nullptr;
  if (S > 1) part = static_cast<double*>(cache_alloc(sizeof(double) * rows * 32 * S, st));
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    int nc = std::min(32, ncols - c0);
    // 16-byte cp.async staging needs 16-byte aligned Omega rows
    const bool aligned = ((uintptr_t)(Om + c0) % 16 == 0) && (ldo % 2 == 0);
    dim3 grid(tiles, S);
    double* yo = S > 1 ? part : Yout + c0;
    const int64_t ld = S > 1 ? nc : ldy;
    const int64_t sstride = S > 1 ? rows * nc : 0;
    if (kp.kind == H2_K_EXP)
      sketch_dispatch<H2_K_EXP>(var, grid, st, X, Yc, Zc, n, row0, row1, Om + c0, ldo, nc, yo, ld, sstride, kp, aligned);
    else
      sketch_dispatch<H2_K_HELMHOLTZ>(var, grid, st, X, Yc, Zc, n, row0, row1, Om + c0, ldo, nc, yo, ld, sstride, kp,
                                      aligned);
    H2_CHECK_LAUNCH();
    if (S > 1) {
      int g = (int)std::min<int64_t>((rows * nc + 255) / 256, (int64_t)sms * 16);
      sketch_combine_kernel<<<g, 256, 0, st>>>(part, S, rows, nc, Yout + c0, ldy);
      H2_CHECK_LAUNCH();
    }
  }
  if (part) cache_free(part, st);
}

// ------------------------------------------------------------------------------------------
// sum of squares of Y(:, c0:c1) (R10: rho^2 N = ||Y||_F^2, accumulated over the draws)
// ------------------------------------------------------------------------------------------
__global__ void sumsq_final_kernel(const double* __restrict__ part, int np, double* __restrict__ out, int* flag) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      out[0] += v;
      if (!isfinite(v)) *flag = 1;
    }
  }
}

// per-leaf partials: every leaf is summed by one CTA (its owner under multi-GPU), and the total
// is taken over the leaves in order, so the result is bitwise independent of the GPU count.
__global__ void sumsq_leaf_kernel(const double* __restrict__ Y, const int64_t* __restrict__ leaf_begin, int cb,
                                  int64_t ld, int c0, int c1, double* __restrict__ part) {
  __shared__ double red[32];
  const int c = cb + blockIdx.x;
  const int64_t r0 = leaf_begin[c], r1 = leaf_begin[c + 1];
  const int w = c1 - c0;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < (r1 - r0) * w; e += blockDim.x) {
    const double v = Y[(r0 + e / w) * ld + c0 + e % w];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[c] = v;
  }
}

void launch_sumsq_leaf(const double* Y, const int64_t* leaf_begin, int cb, int ce, int64_t ld, int c0, int c1,
                       double* part, cudaStream_t st) {
  if (ce <= cb || c1 <= c0) return;
  sumsq_leaf_kernel<<<ce - cb, 256, 0, st>>>(Y, leaf_begin, cb, ld, c0, c1, part);
  H2_CHECK_LAUNCH();
}

void launch_sumsq_total(const double* part, int nleaf, double* accum, int* nonfinite, cudaStream_t st) {
  sumsq_final_kernel<<<1, 1024, 0, st>>>(part, nleaf, accum, nonfinite);
  H2_CHECK_LAUNCH();
}


// Y (rows x ncols, row-major, ldy) = A(rows, :) (row-major, lda) Omega (n x ncols, row-major, ldo):
// in column-major terms Y^T = Omega^T A(rows,:)^T, one DGEMM.
void dense_matrix_sketch(const double* A, int64_t lda, int64_t n, int64_t row0, int64_t row1, const double* Om,
                         int64_t ldo, int ncols, double* Y, int64_t ldy, cudaStream_t st, bool trans) {
  if (row1 <= row0 || ncols <= 0) return;
  static std::mutex mu;
  static cublasHandle_t handles[64] = {};
  int dev = 0;
  H2_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  cublasHandle_t& h = handles[dev & 63];
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw Error(H2_ERR_CUDA, "cublasCreate failed");
  cublasSetStream(h, st);
  cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);   // FP64 (DMMA tensor cores when profitable), no reduced precision
  const double one = 1.0, zero = 0.0;
  // column-major view: Y^T = Om^T A(rows,:)^T;  trans: Y^T = Om^T A(:,rows)
  const cublasStatus_t r =
      trans ? cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, ncols, (int)(row1 - row0), (int)n, &one, Om, (int)ldo,
                          A + row0, (int)lda, &zero, Y, (int)ldy)
            : cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, ncols, (int)(row1 - row0), (int)n, &one, Om, (int)ldo,
                          A + row0 * lda, (int)lda, &zero, Y, (int)ldy);
  if (r != CUBLAS_STATUS_SUCCESS) throw Error(H2_ERR_CUDA, "cublasDgemm failed: " + std::to_string((int)r));
}

}  // namespace h2
