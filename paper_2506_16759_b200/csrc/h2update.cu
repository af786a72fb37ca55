// Black-box operators for the H^2 low-rank update ("the fast H^2-matrix-vector
// product ... (and fast low-rank multiplication) to perform K_blk, and an algorithm that extracts
// entries from the given H^2 and low-rank representations to perform batchedGen"; BASELINE
// configs[4], R24): M = A_H + U U^T with A_H an H^2 matrix on the same tree.
//   sketch  : Y = A_H Omega (h2 matvec) + U (U^T Omega)          (lowrank_* kernels below)
//   entries : D_new(s,b) = D_A(s,b) + U(I_s) U(I_b)^T             (same near pairs)
//             B_new(s,b) = R_s B_A(s,b) R_b^T + U(I~_s) U(I~_b)^T  (same far pairs) with
//             R_s = rows of the expanded basis of A at the new skeletons I~_s (Eq.(2) chain)
#include "common.cuh"
#include "kernels.hpp"

namespace h2 {

// ------------------------------------------------------------------------------------------
// CTA GEMM (256 threads, 64x64 output tiles, 16-deep k slabs; FP64 DMMA m8n8k4, warp tile 16 x 32)
//   C(i,j) = beta C(i,j) + sum_k A(i,k) B(k,j)
//   A(i,k) = tA ? A[k*lda + i] : A[arow(i)*lda + k]     (arow = identity when null)
//   B(k,j) = tB ? B[bcol(j)*ldb + k] : B[k*ldb + j]      (bcol = identity when null)
// ------------------------------------------------------------------------------------------
__device__ void cta_gemm(int M, int N, int K, const double* __restrict__ A, int64_t lda, bool tA,
                         const int32_t* __restrict__ arow, const double* __restrict__ B, int64_t ldb, bool tB,
                         const int32_t* __restrict__ bcol, double* __restrict__ C, int64_t ldc, double beta) {
  // Round 2: (a) the slab loads are coalesced for every operand orientation -- a row-major operand
  // (A not transposed, B transposed: one row of the slab is 16 consecutive k) is read by
  // half-warps along k, a column-major one along i / j -- instead of 8 bytes per 32-byte sector
  // for the strided ones; (b) the next slab is loaded into registers while the current one is
  // multiplied (one slab in flight per thread).  The DMMA sequence per accumulator (k ascending
  // in groups of 4, zero-filled edges) is unchanged: bitwise the previous results.
  __shared__ double sA[16][64 + 1];
  __shared__ double sB[16][64 + 1];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wr = warp & 3, wc = warp >> 2;   // 8 warps: 4 x 16 rows, 2 x 32 columns
  // element q of this thread: A slab entry (ar[q], ak[q]) and B slab entry (bk[q], bc[q])
  int ar[4], ak[4], bk[4], bc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = tid + 256 * q;
    if (tA) { ak[q] = e >> 6; ar[q] = e & 63; } else { ar[q] = e >> 4; ak[q] = e & 15; }
    if (tB) { bc[q] = e >> 4; bk[q] = e & 15; } else { bk[q] = e >> 6; bc[q] = e & 63; }
  }
  for (int i0 = 0; i0 < M; i0 += 64)
    for (int j0 = 0; j0 < N; j0 += 64) {
      double acc[2][4][2] = {};
      double ra[4], rb[4];
      auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = i0 + ar[q], k = k0 + ak[q];
          ra[q] = (i < M && k < K) ? (tA ? A[(int64_t)k * lda + i] : A[(int64_t)(arow ? arow[i] : i) * lda + k]) : 0.0;
          const int j = j0 + bc[q], kb = k0 + bk[q];
          rb[q] = (j < N && kb < K) ? (tB ? B[(int64_t)(bcol ? bcol[j] : j) * ldb + kb] : B[(int64_t)kb * ldb + j]) : 0.0;
        }
      };
      load(0);
      for (int k0 = 0; k0 < K; k0 += 16) {
        __syncthreads();   // the previous slab's fragments have been read
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          sA[ak[q]][ar[q]] = ra[q];
          sB[bk[q]][bc[q]] = rb[q];
        }
        __syncthreads();
        if (k0 + 16 < K) load(k0 + 16);   // in flight during the DMMAs below
        // FP64 tensor cores (DMMA m8n8k4): warp (wr, wc) owns rows 16 wr.. x columns 32 wc..
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int kk = ks * 4 + (lane & 3);
          double af[2], bf[4];
#pragma unroll
          for (int q = 0; q < 2; ++q) af[q] = sA[kk][wr * 16 + q * 8 + (lane >> 2)];
#pragma unroll
          for (int q = 0; q < 4; ++q) bf[q] = sB[kk][wc * 32 + q * 8 + (lane >> 2)];
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) dmma_8x8x4(acc[p][q][0], acc[p][q][1], af[p], bf[q]);
        }
      }
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = i0 + wr * 16 + p * 8 + (lane >> 2), j = j0 + wc * 32 + q * 8 + 2 * (lane & 3) + h;
            if (i < M && j < N) {
              double* c = C + (int64_t)i * ldc + j;
              *c = beta == 0.0 ? acc[p][q][h] : fma(beta, *c, acc[p][q][h]);
            }
          }
      __syncthreads();   // the next tile overwrites sA / sB
    }
}

// ---- sketch: W = U^T Omega (deterministic: fixed 1024-row chunks, chunks summed in order)
__global__ void lowrank_w_partial_kernel(const double* __restrict__ U, int64_t ldu, int r, const double* __restrict__ Om,
                                         int64_t ldo, int nc, int64_t n, double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * 1024;
  const int64_t r1 = (r0 + 1024 < n) ? r0 + 1024 : n;
  for (int e = threadIdx.x; e < r * nc; e += blockDim.x) {
    const int a = e / nc, c = e % nc;
    double s = 0.0;
    for (int64_t i = r0; i < r1; ++i) s = fma(U[i * ldu + a], Om[i * ldo + c], s);
    part[(int64_t)blockIdx.x * r * nc + e] = s;
  }
}
__global__ void lowrank_w_final_kernel(const double* __restrict__ part, int nparts, int rn, double* __restrict__ W) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rn; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * rn + e];
    W[e] = s;
  }
}
// Y(i, c) += sum_a U(i, a) W(a, c)
template <bool SMEM>
__global__ void lowrank_apply_kernel(const double* __restrict__ U, int64_t ldu, int r, const double* __restrict__ W,
                                     int nc, int64_t n, double* __restrict__ Y, int64_t ldy) {
  extern __shared__ double smW[];
  // W = V^T Om (r x nc) staged in shared memory when it fits the default 48 KB, else read
  // through L1 (any rank / column count the build accepts)
  const double* sW = SMEM ? smW : W;
  if (SMEM) {
    for (int e = threadIdx.x; e < r * nc; e += blockDim.x) smW[e] = W[e];
    __syncthreads();
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * nc; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / nc;
    const int c = (int)(t - i * nc);
    double s = 0.0;
    for (int a = 0; a < r; ++a) s = fma(U[i * ldu + a], sW[a * nc + c], s);
    Y[i * ldy + c] += s;
  }
}

void launch_lowrank_sketch(const double* U, int64_t ldu, int r, const double* Om, int64_t ldo, int nc, int64_t n,
                           double* Y, int64_t ldy, double* scratch, cudaStream_t st, const double* V, int64_t ldv) {
  if (r <= 0 || nc <= 0 || n <= 0) return;
  if (!V) {
    V = U;
    ldv = ldu;
  }
  const int np = div_up(n, 1024);
  double* W = scratch + (int64_t)np * r * nc;
  lowrank_w_partial_kernel<<<np, 256, 0, st>>>(V, ldv, r, Om, ldo, nc, n, scratch);   // W = V^T Om
  H2_CHECK_LAUNCH();
  lowrank_w_final_kernel<<<div_up(r * nc, 256), 256, 0, st>>>(scratch, np, r * nc, W);
  H2_CHECK_LAUNCH();
  const int grid = (int)std::min<int64_t>((n * nc + 255) / 256, 148 * 16);
  const size_t wbytes = sizeof(double) * (size_t)r * nc;
  if (wbytes <= 48 * 1024) lowrank_apply_kernel<true><<<grid, 256, wbytes, st>>>(U, ldu, r, W, nc, n, Y, ldy);
  else lowrank_apply_kernel<false><<<grid, 256, 0, st>>>(U, ldu, r, W, nc, n, Y, ldy);
  H2_CHECK_LAUNCH();
}

// ---- entries: D blocks of M over unique near pairs u (stored orientation us <= ub)
__global__ void __launch_bounds__(256) update_D_kernel(UpdateDArgs a) {
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t u = a.ulist ? a.ulist[q] : q;
    const int s = a.us[u], b = a.ub[u];
    const int ms = a.cnt[s], mb = a.cnt[b];
    const double* src = a.Dbase + a.off[u];
    double* out = a.out + a.off[u];
    for (int e = threadIdx.x; e < ms * mb; e += blockDim.x) out[e] = src[e];
    __syncthreads();
    cta_gemm(ms, mb, a.r, a.U + a.begin[s] * a.ldu, a.ldu, false, nullptr, a.U + a.begin[b] * a.ldu, a.ldu, true,
             nullptr, out, mb, 1.0);
    __syncthreads();
  }
}

void launch_update_D(const UpdateDArgs& a, cudaStream_t st) {
  if (a.nblocks <= 0) return;
  update_D_kernel<<<(int)std::min<int64_t>(a.nblocks, 148 * 8), 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

// ---- expanded basis rows of A at the new skeletons of depth t (warp per point):
// v = U^A_leaf(p - begin_leaf, :), then v <- v X^A_tau[rows of the child, :] up to depth t.
__global__ void __launch_bounds__(256) expand_rows_kernel(ExpandArgs a) {
  extern __shared__ double sv[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* v0 = sv + wib * 2 * a.kmax;
  double* v1 = v0 + a.kmax;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib; w < a.npoints; w += warps) {
    const int s = a.pt_cluster[w];
    const int i = (int)(w - a.roff_new[s]);
    const int32_t p = a.skel_new[a.roff_new[s] + i];
    // leaf containing p (binary search in leaf_begin)
    int lo = 0, hi = a.nleaf;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.leaf_begin[mid] <= p) lo = mid;
      else hi = mid;
    }
    int nu = lo;
    int kc = a.kb[a.Dl][nu];
    const double* Ul = a.X[a.Dl] + a.xoff[a.Dl][nu] + (int64_t)(p - a.leaf_begin[nu]) * kc;
    for (int j = lane; j < kc; j += 32) v0[j] = Ul[j];
    __syncwarp();
    for (int u = a.Dl - 1; u >= a.t; --u) {
      const int tau = nu >> 1;
      const int kp = a.kb[u][tau];
      const int off = (nu & 1) ? a.kb[u + 1][nu - 1] : 0;
      const double* Xt = a.X[u] + a.xoff[u][tau] + (int64_t)off * kp;
      for (int j = lane; j < kp; j += 32) {
        double acc = 0.0;
        for (int q = 0; q < kc; ++q) acc = fma(v0[q], Xt[(int64_t)q * kp + j], acc);
        v1[j] = acc;
      }
      __syncwarp();
      double* tmp = v0;
      v0 = v1;
      v1 = tmp;
      kc = kp;
      nu = tau;
    }
    double* R = a.R + a.rowoff[s] + (int64_t)i * kc;
    for (int j = lane; j < kc; j += 32) R[j] = v0[j];
    __syncwarp();
  }
}

void launch_expand_rows(const ExpandArgs& a, cudaStream_t st) {
  if (a.npoints <= 0) return;
  const size_t sm = sizeof(double) * 2 * a.kmax * 8;
  if (sm > 48 * 1024) H2_CUDA(cudaFuncSetAttribute(expand_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int grid = (int)std::min<int64_t>((a.npoints + 7) / 8, 148 * 16);
  expand_rows_kernel<<<grid, 256, sm, st>>>(a);
  H2_CHECK_LAUNCH();
}

// ---- B blocks of M over unique far pairs of depth t: B = R_s (B_A R_b^T) + U(I~_s) U(I~_b)^T
__global__ void __launch_bounds__(256) update_B_kernel(UpdateBArgs a) {
  double* G = a.scratch + (int64_t)blockIdx.x * a.gmax;
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t u = a.ulist ? a.ulist[q] : q;
    const int s = a.us[u], b = a.ub[u];
    const int kns = a.kn[s], knb = a.kn[b], kbs = a.kb[s], kbb = a.kb[b];
    double* out = a.out + a.out_off[u];
    const double* Rs = a.R + a.rowoff[s];
    const double* Rb = a.R + a.rowoff[b];
    // G = B_A(s,b) R_b^T   (kbs x knb)
    cta_gemm(kbs, knb, kbb, a.Bbase + a.Boff[u], kbb, false, nullptr, Rb, kbb, true, nullptr, G, knb, 0.0);
    __syncthreads();
    // out = R_s G
    cta_gemm(kns, knb, kbs, Rs, kbs, false, nullptr, G, knb, false, nullptr, out, knb, 0.0);
    __syncthreads();
    // out += U(I~_s) U(I~_b)^T
    cta_gemm(kns, knb, a.r, a.U, a.ldu, false, a.skel + a.roff_new[s], a.U, a.ldu, true, a.skel + a.roff_new[b], out,
             knb, 1.0);
    __syncthreads();
  }
}

// non-symmetric update M = A_H + U V^T, ordered pairs (h2_build_nonsym):
//   D_{s,b} = D_A(s,b) + U(I_s) V(I_b)^T, D_A(s,b) read from A's unique storage (transposed if s > b)
__global__ void __launch_bounds__(256) update_D_ns_kernel(UpdateNsArgs a) {
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t e = a.ulist ? a.ulist[q] : q;
    const int s = a.os[e], b = a.ob[e];
    const int ms = a.cnt[s], mb = a.cnt[b];
    const int64_t u = a.uidx[e];
    const bool tr = a.us[u] != s;
    const double* src = a.Bbase + a.Boff[u];
    double* out = a.out + a.out_off[e];
    for (int q = threadIdx.x; q < ms * mb; q += blockDim.x) {
      const int i = q / mb, j = q - (q / mb) * mb;
      out[q] = tr ? src[(int64_t)j * ms + i] : src[q];
    }
    __syncthreads();
    cta_gemm(ms, mb, a.r, a.U + a.begin[s] * a.ldu, a.ldu, false, nullptr, a.V + a.begin[b] * a.ldv, a.ldv, true,
             nullptr, out, mb, 1.0);
    __syncthreads();
  }
}

//   B_{s,b} = Rr_s B_A(s,b) Rc_b^T + U(I~_s) V(J~_b)^T: Rr_s / Rc_b = A's expanded basis rows at the
//   new row / column skeletons (launch_expand_rows), B_A(s,b) transposed from storage if s > b
__global__ void __launch_bounds__(256) update_B_ns_kernel(UpdateNsArgs a) {
  double* G = a.scratch + (int64_t)blockIdx.x * a.gmax;
  for (int64_t q = blockIdx.x; q < a.nblocks; q += gridDim.x) {
    const int64_t e = a.ulist ? a.ulist[q] : q;
    const int s = a.os[e], b = a.ob[e];
    const int kns = a.cnt[s], knb = a.cnt2[b], kbs = a.kb[s], kbb = a.kb[b];
    const int64_t u = a.uidx[e];
    const bool tr = a.us[u] != s;
    double* out = a.out + a.out_off[e];
    const double* Rs = a.R + a.rowoff[s];
    const double* Rb = a.R2 + a.rowoff2[b];
    // G = B_A(s,b) Rc_b^T (kbs x knb); stored block is kbs x kbb, or kbb x kbs when transposed
    cta_gemm(kbs, knb, kbb, a.Bbase + a.Boff[u], tr ? kbs : kbb, tr, nullptr, Rb, kbb, true, nullptr, G, knb, 0.0);
    __syncthreads();
    cta_gemm(kns, knb, kbs, Rs, kbs, false, nullptr, G, knb, false, nullptr, out, knb, 0.0);
    __syncthreads();
    cta_gemm(kns, knb, a.r, a.U, a.ldu, false, a.skel + a.roff[s], a.V, a.ldv, true, a.skel2 + a.roff2[b], out, knb,
             1.0);
    __syncthreads();
  }
}

void launch_update_ns(const UpdateNsArgs& a, bool coupling, int grid, cudaStream_t st) {
  if (a.nblocks <= 0) return;
  if (coupling) update_B_ns_kernel<<<grid, 256, 0, st>>>(a);
  else update_D_ns_kernel<<<grid, 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

void launch_update_B(const UpdateBArgs& a, int grid, cudaStream_t st) {
  if (a.nblocks <= 0) return;
  update_B_kernel<<<grid, 256, 0, st>>>(a);
  H2_CHECK_LAUNCH();
}

}  // namespace h2
