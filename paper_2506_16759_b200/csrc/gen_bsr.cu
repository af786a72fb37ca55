// batchedGen (PAPER.md L212 D blocks, L258 B blocks, L384 batched entry generator) and the
// non-uniform batched block-sparse-row product batchedBSRGemm (L213, L240-243, L385).
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// ------------------------------------------------------------------------------------------
// batchedGen: one CTA per unique block (grid-stride), entries written row-major, coalesced.
// ------------------------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(256) gen_kernel(const double* __restrict__ X, const double* __restrict__ Yc,
                                                  const double* __restrict__ Zc, GenArgs a, double param,
                                                  double inv) {
  __shared__ double cx[256], cy[256], cz[256];
  __shared__ double tab[64];
  fill_exp_table(tab);
  for (int64_t u = blockIdx.x; u < a.nblocks; u += gridDim.x) {
    const int s = a.us[u], b = a.ub[u];
    const int m = a.cnt[s], nc = a.cnt[b];
    const int32_t* ri = a.idx + a.off[s];
    const int32_t* ci = a.idx + a.off[b];
    double* out = a.out + a.out_off[u];
    for (int j0 = 0; j0 < nc; j0 += 256) {
      const int nj = min(256, nc - j0);
      __syncthreads();
      if (threadIdx.x < nj) {
        int p = ci[j0 + threadIdx.x];
        cx[threadIdx.x] = X[p];
        cy[threadIdx.x] = Yc[p];
        cz[threadIdx.x] = Zc[p];
      }
      __syncthreads();
      for (int e = threadIdx.x; e < m * nj; e += blockDim.x) {
        int i = e / nj, j = e - i * nj;
        int p = ri[i];
        double r2 = dist2(X[p], Yc[p], Zc[p], cx[j], cy[j], cz[j]);
        out[(int64_t)i * nc + j0 + j] = kernel_of_r2<KIND>(r2, param, inv, tab);
      }
    }
  }
}

void launch_gen(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, const GenArgs& a,
                cudaStream_t st) {
  if (a.nblocks <= 0) return;
  int grid = (int)std::min<int64_t>(a.nblocks, 148 * 32);
  if (kp.kind == H2_K_EXP)
    gen_kernel<H2_K_EXP><<<grid, 256, 0, st>>>(X, Yc, Zc, a, kp.param, kp.inv);
  else
    gen_kernel<H2_K_HELMHOLTZ><<<grid, 256, 0, st>>>(X, Yc, Zc, a, kp.param, kp.inv);
  H2_CHECK_LAUNCH();
}

__global__ void gen_desc_kernel(GenArgs a, int32_t* m, int32_t* nc, int64_t* roff, int64_t* coff, double** outp,
                                int32_t* ld) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < a.nblocks; u += (int64_t)gridDim.x * blockDim.x) {
    int s = a.us[u], b = a.ub[u];
    m[u] = a.cnt[s];
    nc[u] = a.cnt[b];
    ld[u] = a.cnt[b];
    roff[u] = a.off[s];
    coff[u] = a.off[b];
    outp[u] = a.out + a.out_off[u];
  }
}

void launch_gen_batch_desc(const GenArgs& a, int32_t* m, int32_t* nc, int64_t* roff, int64_t* coff, double** outp,
                           int32_t* ld, cudaStream_t st) {
  if (a.nblocks <= 0) return;
  int grid = (int)std::min<int64_t>((a.nblocks + 255) / 256, 148 * 8);
  gen_desc_kernel<<<grid, 256, 0, st>>>(a, m, nc, roff, coff, outp, ld);
  H2_CHECK_LAUNCH();
}

// ------------------------------------------------------------------------------------------
// BSR product  Y(rows of s) += alpha * sum_{b} Blk(s,b) * Om(rows of b)
// CTA = (row cluster s, 64-row tile, 32-column tile); 256 threads, each 8 accumulators
// (row r = tid/4, columns 8*(tid%4)..+7).  Partners in CSR (ascending) order, k ascending
// inside a block: the accumulation order is fixed -> deterministic, no atomics (L385).
// Blocks are stored once per unordered pair; (s,b) with s != us[u] reads the transpose.
// ------------------------------------------------------------------------------------------
// DMMA tiling: CTA = 4*(CW/32) warps = 64 rows x CW columns; warp (wr, wc) owns rows
// 16wr..16wr+15 (2 m-blocks) x columns 32wc..32wc+31 (4 n-blocks): 16 accumulators / lane.
// Partner blocks stream through shared memory in 32-deep k-slabs (each block entry is read
// once per CW columns); row strides = 4 mod 16 doubles keep the fragment loads conflict free.
constexpr int BT_R = 64, BT_K = 32, BT_LD = 36;

template <int CW>
__global__ void __launch_bounds__(4 * CW) bsr_kernel(BsrArgs a, double alpha) {
  constexpr int NT = 4 * CW;           // threads
  constexpr int LDB = CW + 4;
  constexpr int AE = BT_R * BT_K / NT; // A-slab elements per thread
  constexpr int BE = BT_K * CW / NT;   // B-slab elements per thread
  __shared__ __align__(16) double sA[BT_R * BT_LD];
  __shared__ __align__(16) double sB[BT_K * LDB];
  const int s = blockIdx.x;
  const int ms = a.cnt[s];
  const int r0 = blockIdx.y * BT_R;
  const int cb = a.c0 + blockIdx.z * CW;
  const int nc = min(CW, a.c0 + a.ncols - cb);
  if (r0 >= ms || nc <= 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wr = warp & 3, wc = warp >> 2;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // the (partner, k-slab) sequence, with the next slab prefetched into registers while the
  // current one is multiplied (global loads overlap the DMMAs)
  const int e0 = a.ptr[s], e1 = a.ptr[s + 1];
  if (e0 == e1) return;
  int e = e0, k0 = 0;
  double ra[AE], rb[BE];
  int nk_cur = 0;
  auto load = [&](int ee, int kk0, double* xa, double* xb) -> int {
    const int b = a.idx[ee];
    const int u = a.uidx[ee];
    const int mb = a.cnt[b];
    const bool direct = (a.us[u] == s);
    const double* blk = a.blk + a.blk_off[u];
    const double* om = a.Om + a.ooff[b] * a.ldo + cb;
    const int nk = min(BT_K, mb - kk0);
#pragma unroll
    for (int q = 0; q < AE; ++q) {
      const int t = threadIdx.x + q * NT;
      int r, kk;
      if (direct) {
        r = t >> 5;
        kk = t & 31;
      } else {
        kk = t >> 6;
        r = t & 63;
      }
      xa[q] = (r0 + r < ms && kk < nk)
                  ? (direct ? blk[(int64_t)(r0 + r) * mb + kk0 + kk] : blk[(int64_t)(kk0 + kk) * ms + r0 + r])
                  : 0.0;
    }
#pragma unroll
    for (int q = 0; q < BE; ++q) {
      const int t = threadIdx.x + q * NT;
      const int kk = t / CW, c = t % CW;
      xb[q] = (kk < nk && c < nc) ? om[(int64_t)(kk0 + kk) * a.ldo + c] : 0.0;
    }
    return nk;
  };
  bool cur_direct = (a.us[a.uidx[e]] == s);
  nk_cur = load(e, k0, ra, rb);
  while (true) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < AE; ++q) {
      const int t = threadIdx.x + q * NT;
      const int r = cur_direct ? (t >> 5) : (t & 63);
      const int kk = cur_direct ? (t & 31) : (t >> 6);
      sA[r * BT_LD + kk] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < BE; ++q) {
      const int t = threadIdx.x + q * NT;
      sB[(t / CW) * LDB + (t % CW)] = rb[q];
    }
    __syncthreads();
    const int nk = nk_cur;
    // advance to the next slab and prefetch it
    k0 += BT_K;
    if (k0 >= a.cnt[a.idx[e]]) {
      ++e;
      k0 = 0;
    }
    const bool more = e < e1;
    if (more) {
      cur_direct = (a.us[a.uidx[e]] == s);
      nk_cur = load(e, k0, ra, rb);
    }
    const int ksteps = (nk + 3) >> 2;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = sA[(wr * 16 + i * 8 + (lane >> 2)) * BT_LD + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sB[kk * LDB + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (!more) break;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + wr * 16 + i * 8 + (lane >> 2);
    if (r >= ms) continue;
    double* y = a.Y + (a.yoff[s] + r) * a.ldy + cb;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = wc * 32 + j * 8 + 2 * (lane & 3);
      if (c < nc) y[c] = fma(alpha, acc[i][j][0], y[c]);
      if (c + 1 < nc) y[c + 1] = fma(alpha, acc[i][j][1], y[c + 1]);
    }
  }
}

static void bsr_launch(const BsrArgs& a, double alpha, cudaStream_t st) {
  if (a.nclusters <= 0 || a.ncols <= 0 || a.max_rows <= 0) return;
  if (a.ncols > 32) {
    dim3 grid(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, 64));
    bsr_kernel<64><<<grid, 256, 0, st>>>(a, alpha);
  } else {
    dim3 grid(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, 32));
    bsr_kernel<32><<<grid, 128, 0, st>>>(a, alpha);
  }
  H2_CHECK_LAUNCH();
}

void launch_bsr(const BsrArgs& a, cudaStream_t st) { bsr_launch(a, -1.0, st); }

void launch_spmm(const SpmmArgs& s, cudaStream_t st) {
  BsrArgs a{};
  a.nclusters = s.nclusters;
  a.yoff = s.yoff;
  a.ooff = s.xoff;
  a.cnt = s.cnt;
  a.ptr = s.ptr;
  a.idx = s.idx;
  a.uidx = s.uidx;
  a.us = s.us;
  a.blk_off = s.blk_off;
  a.blk = s.blk;
  a.Y = s.y;
  a.ldy = s.ldy;
  a.Om = s.x;
  a.ldo = s.ldx;
  a.c0 = 0;
  a.ncols = s.q;
  a.max_rows = s.max_rows;
  bsr_launch(a, s.alpha, st);
}

}  // namespace h2
