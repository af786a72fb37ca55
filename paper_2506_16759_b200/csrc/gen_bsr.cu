// batchedGen (PAPER.md L212 D blocks, L258 B blocks, L384 batched entry generator) and the
// non-uniform batched block-sparse-row product batchedBSRGemm (L213, L240-243, L385).
#include <mutex>

#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// ------------------------------------------------------------------------------------------
// batchedGen: one CTA per unique block (grid-stride).  Warp w takes rows i = w, w+8, ...; its
// lanes the columns (coalesced row-major writes).  The coordinates of a 256-row x 256-column
// chunk are staged in shared memory up front (row and column gathers issued together, one
// latency per chunk instead of two dependent global loads per row).
// ------------------------------------------------------------------------------------------
template <int KIND, int CPL, int MINB>
__global__ void __launch_bounds__(256, MINB) gen_kernel(const double* __restrict__ X, const double* __restrict__ Yc,
                                                  const double* __restrict__ Zc, GenArgs a, double param,
                                                  double inv) {
  __shared__ double cx[256], cy[256], cz[256];
  __shared__ double rx[256], ry[256], rz[256];
  __shared__ double tab[64], sk[6];
  fill_exp_table(tab);
  exp_neg_consts_fill(sk);
  __syncthreads();
  const ExpNegC ek = exp_neg_consts_load(sk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t u = a.ulist ? a.ulist[q] : q;
    const int s = a.us[u], b = a.ub[u];
    const int m = a.cnt[s], nc = a.cnt2 ? a.cnt2[b] : a.cnt[b];
    const int32_t* ri = a.idx + a.off[s];
    const int32_t* ci = a.cnt2 ? a.idx2 + a.off2[b] : a.idx + a.off[b];
    double* out = a.out + a.out_off[u];
    for (int i0 = 0; i0 < m; i0 += 256) {
      const int mi = min(256, m - i0);
      for (int j0 = 0; j0 < nc; j0 += 256) {
        const int nj = min(256, nc - j0);
        __syncthreads();
        if (threadIdx.x < nj) {
          const int p = ci[j0 + threadIdx.x];
          cx[threadIdx.x] = X[p];
          cy[threadIdx.x] = Yc[p];
          cz[threadIdx.x] = Zc[p];
        }
        if (j0 == 0 && threadIdx.x < mi) {
          const int p = ri[i0 + threadIdx.x];
          rx[threadIdx.x] = X[p];
          ry[threadIdx.x] = Yc[p];
          rz[threadIdx.x] = Zc[p];
        }
        __syncthreads();
        // a lane owns columns jb + 32 u + lane, u < CPL (coordinates in registers for all the
        // warp's rows; CPL independent entries per row step)
        for (int jb = 0; jb < nj; jb += 32 * CPL) {
          double xj[CPL], yj[CPL], zj[CPL];
          int jj[CPL];
          bool vj[CPL];
#pragma unroll
          for (int u = 0; u < CPL; ++u) {
            jj[u] = jb + 32 * u + lane;
            vj[u] = jj[u] < nj;
            const int js = vj[u] ? jj[u] : 0;
            xj[u] = cx[js];
            yj[u] = cy[js];
            zj[u] = cz[js];
          }
          for (int i = warp; i < mi; i += 8) {
            const double xi = rx[i], yi = ry[i], zi = rz[i];
            double* orow = out + (int64_t)(i0 + i) * nc + j0;
            double e[CPL];
#pragma unroll
            for (int u = 0; u < CPL; ++u) {
              if (KIND == H2_K_RATIONAL)   // exact-order entries (inv carries l^2)
                e[u] = k_rational(r2_exact(xi, yi, zi, xj[u], yj[u], zj[u]), inv);
              else
                e[u] = kernel_of_r2<KIND>(dist2(xi, yi, zi, xj[u], yj[u], zj[u]), param, inv, tab, ek);
            }
#pragma unroll
            for (int u = 0; u < CPL; ++u)
              if (vj[u]) orow[jj[u]] = e[u];
          }
        }
      }
    }
  }
}

// batchedGen from an explicit matrix (H2_E_DENSE_MATRIX): out(i, j) = A[ri[i] * lda + ci[j]]
__global__ void __launch_bounds__(256) gen_dense_kernel(const double* __restrict__ A, int64_t lda, GenArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t u = a.ulist ? a.ulist[q] : q;
    const int s = a.us[u], b = a.ub[u];
    const int m = a.cnt[s], nc = a.cnt2 ? a.cnt2[b] : a.cnt[b];
    const int32_t* ri = a.idx + a.off[s];
    const int32_t* ci = a.cnt2 ? a.idx2 + a.off2[b] : a.idx + a.off[b];
    double* out = a.out + a.out_off[u];
    for (int i = warp; i < m; i += 8) {
      const double* arow = A + (int64_t)ri[i] * lda;
      for (int j = lane; j < nc; j += 32) out[(int64_t)i * nc + j] = arow[ci[j]];
    }
  }
}

void launch_gen_dense(const double* A, int64_t lda, const GenArgs& a, cudaStream_t st) {
  if (a.nblocks <= 0) return;
  gen_dense_kernel<<<(int)std::min<int64_t>(a.nblocks, 148 * 32), 256, 0, st>>>(A, lda, a);
  H2_CHECK_LAUNCH();
}

void launch_gen(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, const GenArgs& a,
                cudaStream_t st) {
  if (a.nblocks <= 0) return;
  int grid = (int)std::min<int64_t>(a.nblocks, 148 * 32);
  // 2 columns per lane, <= 64 registers (4 CTAs / SM): measured 6.2 ms at C2 vs 6.6 (1 column
  // per lane, unbounded registers) -- the phase is bound by its many small per-level launches
  auto go = [&](auto kern, double p2) { kern<<<grid, 256, 0, st>>>(X, Yc, Zc, a, kp.param, p2); };
  if (kp.kind == H2_K_EXP) go(gen_kernel<H2_K_EXP, 2, 4>, kp.inv);
  else if (kp.kind == H2_K_RATIONAL) go(gen_kernel<H2_K_RATIONAL, 1, 1>, kp.l2);
  else go(gen_kernel<H2_K_HELMHOLTZ, 2, 4>, kp.inv);
  H2_CHECK_LAUNCH();
}

__global__ void gen_desc_kernel(GenArgs a, int32_t* m, int32_t* nc, int64_t* roff, int64_t* coff, double** outp,
                                int32_t* ld) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nblocks; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = a.ulist ? a.ulist[q] : q;
    int s = a.us[u], b = a.ub[u];
    m[q] = a.cnt[s];
    nc[q] = a.cnt2 ? a.cnt2[b] : a.cnt[b];
    ld[q] = nc[q];
    roff[q] = a.off[s];
    coff[q] = a.cnt2 ? a.off2[b] : a.off[b];
    outp[q] = a.out + a.out_off[u];
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
// CTA = (row cluster s, 64-row tile, CW-column tile); warp (wr, wc) owns rows 16wr..16wr+15 x
// columns 32wc..32wc+31 (2 x 4 DMMA m8n8k4 tiles, 16 accumulators per lane).  Partners in CSR
// (ascending) order, k ascending inside a block: the accumulation order is fixed ->
// deterministic, no atomics (L385).  Blocks are stored once per unordered pair; (s,b) with
// s != us[u] reads the stored block transposed.
// The (partner, 32-deep k-slab) sequence streams through a BSR_NS-stage cp.async ring in shared
// memory (global -> shared without register staging, zero fill at ragged edges): the loads of
// slab it+NS-1 are in flight while slab it is multiplied.  The block slab is stored in its
// stored orientation (row-major [64][36] for direct, [32][68] for transposed: padded,
// 16-byte rows) and the DMMA A fragments read it accordingly.
// ------------------------------------------------------------------------------------------
constexpr int BT_R = 64, BT_K = 32, BSR_NS = 2;
constexpr int BT_LDD = 36;   // direct slab row stride (doubles)
constexpr int BT_LDT = 68;   // transposed slab row stride
constexpr int BT_ASZ = BT_R * BT_LDD > BT_K * BT_LDT ? BT_R * BT_LDD : BT_K * BT_LDT;

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}

// WM: 8-row DMMA blocks per warp (warp tile 8 WM x 32); warps: NWR along rows x CW/32 along columns
// NS: cp.async ring stages; COLFAST: grid x = column tile (the column tiles of one row tile run
// together and share the block slabs through L2), y = cluster, z = row tile
template <int CW, int WM, int NS = BSR_NS, bool COLFAST = false>
__global__ void __launch_bounds__(32 * (64 / (8 * WM)) * (CW / 32)) bsr_kernel(BsrArgs a, double alpha) {
  constexpr int NWR = 64 / (8 * WM);
  constexpr int NT = 32 * NWR * (CW / 32);   // threads
  constexpr int LDB = CW + 4;
  constexpr int BSZ = BT_K * LDB;
  extern __shared__ __align__(16) double bsm[];   // NS x (A slab + B slab)
  __shared__ int st_nk[NS], st_dir[NS];
  const int s = a.c_begin + (COLFAST ? blockIdx.y : blockIdx.x);
  const int ms = a.cnt[s];
  const int r0 = (COLFAST ? blockIdx.z : blockIdx.y) * BT_R;
  const int cb = a.c0 + (COLFAST ? blockIdx.x : blockIdx.z) * CW;
  const int nc = min(CW, a.c0 + a.ncols - cb);
  if (r0 >= ms || nc <= 0) return;
  const int e0 = a.ptr[s], e1 = a.ptr[s + 1];
  if (e0 == e1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp % NWR, wc = warp / NWR;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bsm);
  // loader state: next (partner, k0) to load
  int le = e0, lk = 0;
  auto load_next = [&](int buf) {
    if (le >= e1) return;
    const int b = a.idx[le];
    const int u = a.uidx ? a.uidx[le] : le;
    const int mb = a.kcnt ? a.kcnt[b] : a.cnt[b];
    const bool direct = a.tmode == 0 ? (a.us[u] == s) : (a.tmode == 1);
    const double* blk = a.blk + a.blk_off[u];
    const double* om = a.Om + a.ooff[b] * a.ldo + cb;
    const int nk = min(BT_K, mb - lk);
    const uint32_t sa = sbase + (uint32_t)(buf * (BT_ASZ + BSZ)) * 8u;
    const uint32_t sb = sa + (uint32_t)BT_ASZ * 8u;
    if (direct) {
      // rows r of s (r0 + r < ms), entries kk of the slab: blk[(r0 + r) * mb + lk + kk]
#pragma unroll 4
      for (int q = tid; q < BT_R * BT_K; q += NT) {
        const int r = q >> 5, kk = q & 31;
        const bool ok = (r0 + r < ms) && (kk < nk);
        cp_async8(sa + (uint32_t)(r * BT_LDD + kk) * 8u, ok ? blk + (int64_t)(r0 + r) * mb + lk + kk : blk, ok);
      }
    } else {
      // stored block is b x s: entry (kk, r) at blk[(lk + kk) * ms + r0 + r]
#pragma unroll 4
      for (int q = tid; q < BT_R * BT_K; q += NT) {
        const int kk = q >> 6, r = q & 63;
        const bool ok = (r0 + r < ms) && (kk < nk);
        cp_async8(sa + (uint32_t)(kk * BT_LDT + r) * 8u, ok ? blk + (int64_t)(lk + kk) * ms + r0 + r : blk, ok);
      }
    }
#pragma unroll 4
    for (int q = tid; q < BT_K * CW; q += NT) {
      const int kk = q / CW, c = q % CW;
      const bool ok = (kk < nk) && (c < nc);
      cp_async8(sb + (uint32_t)(kk * LDB + c) * 8u, ok ? om + (int64_t)(lk + kk) * a.ldo + c : om, ok);
    }
    if (tid == 0) {
      st_nk[buf] = nk;
      st_dir[buf] = direct ? 1 : 0;
    }
    lk += BT_K;
    if (lk >= mb) {
      ++le;
      lk = 0;
    }
  };
  double acc[WM][4][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int nitems = 0;
  for (int e = e0; e < e1; ++e) nitems += ((a.kcnt ? a.kcnt : a.cnt)[a.idx[e]] + BT_K - 1) / BT_K;
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    load_next(q);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int it = 0; it < nitems; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2));
    __syncthreads();
    // the buffer of slab it-1 was consumed before this barrier: refill it with slab it+NS-1
    load_next((it + NS - 1) % NS);
    asm volatile("cp.async.commit_group;\n" ::);
    const int buf = it % NS;
    const double* sA = bsm + buf * (BT_ASZ + BSZ);
    const double* sB = sA + BT_ASZ;
    const int nk = st_nk[buf];
    const bool direct = st_dir[buf] != 0;
    const int ksteps = (nk + 3) >> 2;
    for (int ks = 0; ks < ksteps; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      double af[WM], bf[4];
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        const int r = wr * (8 * WM) + i * 8 + (lane >> 2);
        af[i] = direct ? sA[r * BT_LDD + kk] : sA[kk * BT_LDT + r];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sB[kk * LDB + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    const int r = r0 + wr * (8 * WM) + i * 8 + (lane >> 2);
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

// ------------------------------------------------------------------------------------------
// bsr2_kernel (round 2): the same product, the same DMMA sequence per accumulator (partners in
// CSR order, k ascending, 4-deep DMMA k groups, zero-filled ragged k) -> bitwise the results of
// bsr_kernel, with the instruction overhead per DMMA cut from ~16.6 to a few
// (profiles/r2_bsr2_ncu.md: bsr_kernel was issue-bound at 61 % issue-slot use, 0.6 DMMA per 16
// pipe cycles):
//   * the A slab is stored in ONE layout ([r][kk], row stride 36 doubles) for both orientations:
//     a transposed block is transposed by the loader's scatter (cp.async destinations), so the
//     k loop has no orientation select;
//   * the 8 k steps of a slab are unrolled with compile-time shared-memory offsets (LDS with
//     immediate offsets: no address arithmetic per fragment);
//   * every thread's loader positions are fixed per slab (one row pointer per element row,
//     advanced by a constant), no div/mod per element.
// CTA = (64-row tile, CW columns), 4 row warps x CW/32 column warps, warp tile 16 x 32 (2 x 4
// DMMA m8n8k4 tiles).  NS-stage cp.async ring of (A slab 64 x 32, B slab 32 x CW).
// ------------------------------------------------------------------------------------------
constexpr int B2_LDA = 36;   // A slab row stride (doubles): conflict-free fragment reads
constexpr int B2_MAXP = 256; // partners per row cluster staged in shared memory
// WM: 8-row DMMA blocks per warp (2: warp tile 16 x 32, 4: 32 x 32 -- half the A-fragment loads per
// DMMA); warps NWR = 64 / (8 WM) along rows x CW / 32 along columns
template <int CW, int NS, bool COLFAST, int KD = 32, int WM = 2>
__global__ void __launch_bounds__(32 * (64 / (8 * WM)) * (CW / 32)) bsr2_kernel(BsrArgs a, double alpha) {
  constexpr int NWR = 64 / (8 * WM);
  constexpr int NT = 32 * NWR * (CW / 32);
  constexpr int NW = NT / 32;
  constexpr int LDA = KD + 4;                // A slab row stride: = 4 mod 16 doubles, conflict-free fragments
  constexpr int LDB = CW + 4;
  constexpr int ASZ = BT_R * LDA;            // 2304 doubles at KD = 32
  constexpr int BSZ = KD * LDB;
  constexpr int STG = ASZ + BSZ;
  extern __shared__ __align__(16) double bsm[];
  __shared__ int st_nk[NS];
  const int s = a.c_begin + (COLFAST ? blockIdx.y : blockIdx.x);
  const int ms = a.cnt[s];
  const int r0 = (COLFAST ? blockIdx.z : blockIdx.y) * BT_R;
  const int cb = a.c0 + (COLFAST ? blockIdx.x : blockIdx.z) * CW;
  const int nc = min(CW, a.c0 + a.ncols - cb);
  if (r0 >= ms || nc <= 0) return;
  const int e0 = a.ptr[s], e1 = a.ptr[s + 1];
  if (e0 == e1) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(bsm);
  const int rows_here = min(BT_R, ms - r0);
  // partner metadata of this row cluster staged once in shared memory (one round trip per CTA
  // instead of a dependent global-load chain idx -> uidx -> blk_off / cnt per slab, which was the
  // top stall after the loop rewrite: long scoreboard on the slab addresses)
  __shared__ int64_t p_blk[B2_MAXP], p_om[B2_MAXP];
  __shared__ int p_mb[B2_MAXP];
  __shared__ int s_items;
  const int np = e1 - e0;
  const bool staged = np <= B2_MAXP;
  if (tid == 0) s_items = 0;
  __syncthreads();
  if (staged) {
    int my = 0;
    for (int q = tid; q < np; q += NT) {
      const int e = e0 + q;
      const int b = a.idx[e];
      const int u = a.uidx ? a.uidx[e] : e;
      const int mb = a.kcnt ? a.kcnt[b] : a.cnt[b];
      const bool direct = a.tmode == 0 ? (a.us[u] == s) : (a.tmode == 1);
      p_blk[q] = a.blk_off[u];
      p_om[q] = a.ooff[b];
      p_mb[q] = direct ? mb : -mb;
      my += (mb + KD - 1) / KD;
    }
    if (my) atomicAdd(&s_items, my);
  } else if (tid == 0) {
    int n = 0;
    for (int e = e0; e < e1; ++e) n += ((a.kcnt ? a.kcnt : a.cnt)[a.idx[e]] + KD - 1) / KD;
    s_items = n;
  }
  __syncthreads();
  const int nitems = s_items;
  int le = e0, lk = 0;
  auto load_next = [&](int buf) {
    if (le >= e1) return;
    int mb;
    bool direct;
    int64_t boff, orow;
    if (staged) {
      const int q = le - e0;
      const int sm = p_mb[q];
      mb = sm < 0 ? -sm : sm;
      direct = sm > 0 || (sm == 0 && a.tmode != 2);
      boff = p_blk[q];
      orow = p_om[q];
    } else {
      const int b = a.idx[le];
      const int u = a.uidx ? a.uidx[le] : le;
      mb = a.kcnt ? a.kcnt[b] : a.cnt[b];
      direct = a.tmode == 0 ? (a.us[u] == s) : (a.tmode == 1);
      boff = a.blk_off[u];
      orow = a.ooff[b];
    }
    const double* blk = a.blk + boff;
    const int nk = min(KD, mb - lk);
    const uint32_t sa = sbase + (uint32_t)(buf * STG) * 8u;
    const uint32_t sb = sa + (uint32_t)ASZ * 8u;
    if (direct) {
      // KD consecutive lanes cover one row segment (KD x 8 bytes contiguous), 32 / KD rows per
      // warp instruction, rows r = rl + (32 / KD)(warp + NW q)
      constexpr int RPW = 32 / KD;
      const int kk = lane % KD, rl = lane / KD;
      const bool kok = kk < nk;
      const double* src = blk + (int64_t)(r0 + rl + RPW * warp) * mb + lk + kk;
      const int64_t step = (int64_t)RPW * NW * mb;
#pragma unroll
      for (int q = 0; q < (BT_R + RPW * NW - 1) / (RPW * NW); ++q) {   // NW need not divide 64
        const int r = rl + RPW * (warp + NW * q);
        if (r >= BT_R) break;
        const bool ok = kok && r < rows_here;
        cp_async8(sa + (uint32_t)(r * LDA + kk) * 8u, ok ? src : blk, ok);
        src += step;
      }
    } else {
      // stored block is b x s: entry (kk, r) at blk[(lk + kk) * ms + r0 + r]; a warp covers 8 r x
      // 4 kk (64-byte global runs), scattered transposed into [r][kk]
      const int rl = lane & 7, kl = lane >> 3;
#pragma unroll
      for (int q = 0; q < (2 * KD + NW - 1) / NW; ++q) {
        const int t = warp + NW * q;                      // 2 KD tiles of 8 r x 4 kk
        if (t >= 2 * KD) break;
        const int r = 8 * (t & 7) + rl, kk = 4 * (t >> 3) + kl;
        const bool ok = kk < nk && r < rows_here;
        cp_async8(sa + (uint32_t)(r * LDA + kk) * 8u, ok ? blk + (int64_t)(lk + kk) * ms + r0 + r : blk, ok);
      }
    }
    {
      // B slab element e = tid + NT q: (kk = e / CW, c = e % CW), consecutive lanes along c
      const double* om = a.Om + orow * a.ldo + cb;
#pragma unroll
      for (int q = 0; q < KD * CW / NT; ++q) {
        const int e = tid + NT * q;
        const int kk = e / CW, c = e % CW;
        const bool ok = c < nc && kk < nk;
        cp_async8(sb + (uint32_t)(kk * LDB + c) * 8u, ok ? om + (int64_t)(lk + kk) * a.ldo + c : a.Om, ok);
      }
    }
    if (tid == 0) st_nk[buf] = nk;
    lk += KD;
    if (lk >= mb) {
      ++le;
      lk = 0;
    }
  };
  const int wr = warp % NWR, wc = warp / NWR;
  double acc[WM][4][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) {
    load_next(q);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  // fragment base offsets (doubles) inside a stage
  const int offa = (wr * 8 * WM + (lane >> 2)) * LDA + (lane & 3);
  const int offb = ASZ + (lane & 3) * LDB + wc * 32 + (lane >> 2);
  for (int it = 0; it < nitems; ++it) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NS - 2));
    __syncthreads();
    load_next((it + NS - 1) % NS);
    asm volatile("cp.async.commit_group;\n" ::);
    const double* st = bsm + (it % NS) * STG;
    const double* pa = st + offa;
    const double* pb = st + offb;
    const int ksteps = (st_nk[it % NS] + 3) >> 2;
    auto kstep = [&](int ks) {
      double af[WM], bf[4];
#pragma unroll
      for (int i = 0; i < WM; ++i) af[i] = pa[i * 8 * LDA + ks * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = pb[ks * 4 * LDB + j * 8];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    };
    if (ksteps == KD / 4) {
      // full slab: no per-step guard, so the fragment loads of later k steps can be scheduled
      // ahead of the current step's DMMAs
#pragma unroll
      for (int ks = 0; ks < KD / 4; ++ks) kstep(ks);
    } else {
#pragma unroll
      for (int ks = 0; ks < KD / 4; ++ks)
        if (ks < ksteps) kstep(ks);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    const int r = r0 + wr * 8 * WM + i * 8 + (lane >> 2);
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

template <int CW, int NS, bool COLFAST, int KD = 32, int WM = 2>
static void bsr2_go(const BsrArgs& a, double alpha, cudaStream_t st) {
  const size_t sm = sizeof(double) * NS * (BT_R * (KD + 4) + KD * (CW + 4));
  constexpr int NT = 32 * (64 / (8 * WM)) * (CW / 32);
  H2_CUDA(cudaFuncSetAttribute(bsr2_kernel<CW, NS, COLFAST, KD, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm));
  if (COLFAST)
    bsr2_kernel<CW, NS, COLFAST, KD, WM><<<dim3(div_up(a.ncols, CW), a.nclusters, div_up(a.max_rows, BT_R)), NT, sm,
                                           st>>>(a, alpha);
  else
    bsr2_kernel<CW, NS, COLFAST, KD, WM><<<dim3(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, CW)), NT, sm,
                                           st>>>(a, alpha);
  H2_CHECK_LAUNCH();
}

static void bsr_launch(const BsrArgs& a, double alpha, cudaStream_t st) {
  if (a.nclusters <= 0 || a.ncols <= 0 || a.max_rows <= 0) return;
  // H2_BSR2: 0 = the round-1 kernel family below; 1 = bsr2 32-column tiles (column-fast grid for
  // wide passes); 2 = bsr2 64-column tiles; 3 = bsr2 32-column tiles, 3-stage ring; 4 / 5 = 16-deep
  // slabs (half the shared memory per stage: 7 / 5 CTAs per SM), 2 / 3 stages; 6 / 7 = 160- / 96-column
  // CTAs; 8 / 9 / 10 = 64-column CTAs of four 32 x 32 warp tiles (half the A-fragment loads per DMMA)
  // over the 64-multiple of the columns + 32-column tiles for the rest, 32-deep / 16-deep slabs,
  // 16-deep with 3 stages
  // default 9: 54.9 vs 57.9 ms (variant 1) for the C2 BSR phase (profiles/r2_bsr2_ncu.md)
  static const int v2 = env_int("H2_BSR2", 9);
  if (v2 != 0) {
    const bool wide = a.ncols > 32;
    if (v2 == 2 && a.ncols > 32) bsr2_go<64, 2, true>(a, alpha, st);
    else if (v2 == 3) wide ? bsr2_go<32, 3, true>(a, alpha, st) : bsr2_go<32, 3, false>(a, alpha, st);
    else if (v2 == 4) wide ? bsr2_go<32, 2, true, 16>(a, alpha, st) : bsr2_go<32, 2, false, 16>(a, alpha, st);
    else if (v2 == 5) wide ? bsr2_go<32, 3, true, 16>(a, alpha, st) : bsr2_go<32, 3, false, 16>(a, alpha, st);
    else if (v2 == 6 && a.ncols > 128) bsr2_go<160, 2, true>(a, alpha, st);   // one CTA per 160 columns
    else if (v2 == 7 && a.ncols > 64) bsr2_go<96, 2, true>(a, alpha, st);
    else if (v2 == 11 && a.ncols > 32) bsr2_go<64, 2, true, 16, 4>(a, alpha, st);   // no tail split
    else if ((v2 == 8 || v2 == 9 || v2 == 10 || v2 == 12) && a.ncols > 32) {
      // 64-column CTA tiles with 32 x 32 warp tiles over the first 64-multiple of the columns, the
      // remaining (< 64) columns in 32-column tiles: no half-empty column tile at 160 columns
      const int main = a.ncols / 64 * 64;
      BsrArgs m = a;
      m.ncols = main;
      // the tail columns on a second stream, concurrent with the 64-column launch (disjoint output
      // columns, the same arithmetic: bitwise; the tail's CTAs fill the main launch's last waves):
      // C2 BSR phase 47.6 -> 44.7 ms (tools/ab_phases.py); H2_BSR_TAIL_STREAM=0 serialises
      static const int tail_stream = env_int("H2_BSR_TAIL_STREAM", 1);
      cudaStream_t ts = st;
      cudaEvent_t ev0 = nullptr, ev1 = nullptr;
      if (tail_stream && main > 0 && a.ncols > main) {
        static std::mutex mu;   // builds may run on several host threads / devices
        static cudaStream_t side[64] = {};
        int dev = 0;
        H2_CUDA(cudaGetDevice(&dev));
        {
          std::lock_guard<std::mutex> lk(mu);
          if (!side[dev & 63]) H2_CUDA(cudaStreamCreateWithFlags(&side[dev & 63], cudaStreamNonBlocking));
          ts = side[dev & 63];
        }
        H2_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
        H2_CUDA(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
        H2_CUDA(cudaEventRecord(ev0, st));   // everything before this BSR on st
        H2_CUDA(cudaStreamWaitEvent(ts, ev0, 0));
      }
      if (main == 0) {
      } else if (v2 == 8) bsr2_go<64, 2, true, 32, 4>(m, alpha, st);
      else if (v2 == 9) bsr2_go<64, 2, true, 16, 4>(m, alpha, st);
      else bsr2_go<64, 3, true, 16, 4>(m, alpha, st);
      if (a.ncols > main) {
        BsrArgs t = a;
        t.c0 = a.c0 + main;
        t.ncols = a.ncols - main;
        if (v2 == 12) bsr2_go<32, 2, true, 16, 4>(t, alpha, ts);   // tail in 32 x 32 warp tiles too
        else bsr2_go<32, 2, true>(t, alpha, ts);
        if (ts != st) {
          H2_CUDA(cudaEventRecord(ev1, ts));
          H2_CUDA(cudaStreamWaitEvent(st, ev1, 0));
          H2_CUDA(cudaEventDestroy(ev0));
          H2_CUDA(cudaEventDestroy(ev1));
        }
      }
    }
    else wide ? bsr2_go<32, 2, true>(a, alpha, st) : bsr2_go<32, 2, false>(a, alpha, st);
    return;
  }
  constexpr size_t sm32 = sizeof(double) * BSR_NS * (BT_ASZ + BT_K * (32 + 4));
  constexpr size_t sm64 = sizeof(double) * BSR_NS * (BT_ASZ + BT_K * (64 + 4));
  // per launch: the attribute is per device (a process may drive several GPUs)
  H2_CUDA(cudaFuncSetAttribute(bsr_kernel<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm32));
  H2_CUDA(cudaFuncSetAttribute(bsr_kernel<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64));
  H2_CUDA(cudaFuncSetAttribute(bsr_kernel<64, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64));
  static const int wm64 = env_int("H2_BSR_WM64", 4);   // 32 x 32 warp tiles for 64-column passes (-3 ms at C2)
  // wide passes (the eager sweep): one CTA covers up to 160 columns with 2 x CW/32
  // warps of 32 x 32 tiles, so each block slab is read once per row tile and no column tile runs
  // half empty (160 = 64 + 64 + 32 wasted 17 % of the DMMA work)
  // wide passes (> 64 columns, the eager sweep): 32-column CTA tiles in a column-fast grid (the
  // tiles of one row tile run together and share its block slabs through L2) measured 68.0 vs
  // 72.2 ms at C2; the other variants (160-column CTAs, 3-stage rings, 64-column column-fast)
  // were slower (tools/ab_phases.py)
  static const int var = env_int("H2_BSR_VAR", 3);
  if (a.ncols > 64 && var != 0) {
    auto go = [&](auto kern, int cw, int wm, int ns, bool colfast) {
      const size_t sm = sizeof(double) * ns * (BT_ASZ + BT_K * (cw + 4));
      H2_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      const int nt = 32 * (64 / (8 * wm)) * (cw / 32);
      if (colfast) kern<<<dim3(div_up(a.ncols, cw), a.nclusters, div_up(a.max_rows, BT_R)), nt, sm, st>>>(a, alpha);
      else kern<<<dim3(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, cw)), nt, sm, st>>>(a, alpha);
    };
    const int cwn = std::min(5, div_up(a.ncols, 32));
    if (var == 1) {
      if (cwn == 5) go(bsr_kernel<160, 4>, 160, 4, BSR_NS, false);
      else if (cwn == 4) go(bsr_kernel<128, 4>, 128, 4, BSR_NS, false);
      else go(bsr_kernel<96, 4>, 96, 4, BSR_NS, false);
    } else if (var == 2) {
      if (cwn == 5) go(bsr_kernel<160, 4, 3>, 160, 4, 3, false);
      else if (cwn == 4) go(bsr_kernel<128, 4, 3>, 128, 4, 3, false);
      else go(bsr_kernel<96, 4, 3>, 96, 4, 3, false);
    } else if (var == 3) {
      go(bsr_kernel<32, 2, BSR_NS, true>, 32, 2, BSR_NS, true);
    } else if (var == 4) {
      go(bsr_kernel<64, 4, BSR_NS, true>, 64, 4, BSR_NS, true);
    } else {
      go(bsr_kernel<64, 4, 3>, 64, 4, 3, false);
    }
    H2_CHECK_LAUNCH();
    return;
  }
  if (a.ncols > 32) {
    dim3 grid(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, 64));
    if (wm64 == 4) bsr_kernel<64, 4><<<grid, 128, sm64, st>>>(a, alpha);
    else bsr_kernel<64, 2><<<grid, 256, sm64, st>>>(a, alpha);
  } else {
    dim3 grid(a.nclusters, div_up(a.max_rows, BT_R), div_up(a.ncols, 32));
    bsr_kernel<32, 2><<<grid, 128, sm32, st>>>(a, alpha);
  }
  H2_CHECK_LAUNCH();
}

void launch_bsr(const BsrArgs& a, cudaStream_t st) { bsr_launch(a, -1.0, st); }

void launch_spmm(const SpmmArgs& s, cudaStream_t st) {
  BsrArgs a{};
  a.nclusters = s.nclusters;
  a.c_begin = s.c_begin;
  a.yoff = s.yoff;
  a.ooff = s.xoff;
  a.cnt = s.cnt;
  a.ptr = s.ptr;
  a.idx = s.idx;
  a.uidx = s.uidx;
  a.us = s.us;
  a.blk_off = s.blk_off;
  a.blk = s.blk;
  a.kcnt = s.kcnt;
  a.tmode = s.tmode;
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
