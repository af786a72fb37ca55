// Launch wrappers of the sm_100a kernels of libh2 (one line each says which Algorithm-1 step).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

namespace h2 {

// batchedRand: Omega rows [row0,row0+nrows) x cols [col0,col0+ncols)          (L203, L384)
void launch_omega(uint64_t seed, uint32_t sid, int64_t row0, int64_t nrows, int col0, int ncols, double* out,
                  int64_t ld, cudaStream_t st);
// built-in dense sketch Y(rows,:) = K(rows,:) Omega                              (L203 with K_blk = K)
// omega_quarters: every entry is q/4, |q| <= 32 (the h2_omega stream) -> int8 tensor-core path
void launch_dense_sketch(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                         int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Yout,
                         int64_t ldy, bool omega_quarters, cudaStream_t st);
// exp-kernel sketch on the int8 tensor cores (tcgen05 kind::i8, exact slices; sketch_tc.cu)
bool sketch_tc_supported(const KernelParams& kp);
int sketch_tc_pass_cols(int kind);   // Omega columns per tensor-core sketch pass (K evaluated once per pass)
int sketch_tc_slices(int kind);      // byte slices of the fixed-point K (6: 47-bit grid, 7: 52-bit)
int env_int(const char* name, int def);
bool launch_dense_sketch_tc(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                            int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Yout,
                            int64_t ldy, cudaStream_t st);
// the leaf subtraction on the tensor cores (near leaves only; see sketch_tc.cu)
bool launch_near_sketch_tc(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                           int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Y, int64_t ldy,
                           const int32_t* nl_ptr, const int32_t* nl_chunk, const uint8_t* nl_mask, cudaStream_t st);
// explicit dense operator on the int8 tensor cores (Omega = the h2 stream):
// Y(rows) = A(rows, :) Omega, A row-major n x n (lda), 7-slice fixed point of scale 2^E >= amax
double dense_absmax(const double* A, int64_t lda, int64_t n, cudaStream_t st);
void launch_dense_op_tc(const double* A, int64_t lda, int64_t n, int64_t row0, int64_t row1, double amax,
                        const double* Om, int64_t ldo, int ncols, double* Y, int64_t ldy, cudaStream_t st);
// minimum squared distance of distinct points over the near-field leaf pairs (Helmholtz scale)
double min_near_dist2(const double* X, const double* Y, const double* Z, const int64_t* leaf_begin, int nleaf,
                      const int32_t* near_ptr, const int32_t* near_idx, cudaStream_t st);
void launch_sketch_combine(const double* P, int S, int64_t rows, int ncols, double* Y, int64_t ldy, cudaStream_t st);
// accum += ||Y(:, c0:c1)||_F^2 (deterministic)                                   (R10 tolerance scale)
// per-leaf sums of squares of Y(rows of leaf c, c0:c1) for leaves [cb, ce) into part[c] (one CTA
// per leaf), and the fixed-order total over all nleaf partials: accum += sum_c part[c]
void launch_sumsq_leaf(const double* Y, const int64_t* leaf_begin, int cb, int ce, int64_t ld, int c0, int c1,
                       double* part, cudaStream_t st);
void launch_sumsq_total(const double* part, int nleaf, double* accum, int* nonfinite, cudaStream_t st);
// batchedGen over unique pairs u: out[out_off[u] + i*nc + j] = K(idx[off[us]+i], idx[off[ub]+j])
// (L212 for D with idx = iota, off = cluster begin; L258 for B with idx = skeletons)
struct GenArgs {
  int64_t nblocks;
  const int32_t* ulist;   // optional: block q is unique pair ulist[q] (multi-GPU subset), else q
  const int32_t* us;
  const int32_t* ub;
  const int32_t* cnt;     // per cluster rows
  const int64_t* off;     // per cluster offset into idx
  const int32_t* idx;     // tree-order point indices
  const int64_t* out_off; // per unique pair
  double* out;
  // optional column side (non-symmetric B_{s,b} = K(I~_s, J~_b)): columns from cnt2/off2/idx2
  const int32_t* cnt2;
  const int64_t* off2;
  const int32_t* idx2;
};
void launch_gen(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, const GenArgs& a,
                cudaStream_t st);
void launch_gen_dense(const double* A, int64_t lda, const GenArgs& a, cudaStream_t st);
// Y(rows) = A(rows, :) Omega for a dense row-major operator (cuBLAS DGEMM, the plain library GEMM);
// trans: Y(rows) = A(:, rows)^T Omega (the column sketch of the non-symmetric build)
void dense_matrix_sketch(const double* A, int64_t lda, int64_t n, int64_t row0, int64_t row1, const double* Om,
                         int64_t ldo, int ncols, double* Y, int64_t ldy, cudaStream_t st, bool trans = false);
// fill the pointer / size arrays of an h2_block_batch for a user entry callback
void launch_gen_batch_desc(const GenArgs& a, int32_t* m, int32_t* nc, int64_t* roff, int64_t* coff, double** outp,
                           int32_t* ld, cudaStream_t st);

// batchedBSRGemm: Y(rows of s, c0:c0+nc) -= sum_{b in CSR row s} Blk(s,b) Om(rows of b, c0:c0+nc)
// (L213 leaf with D, L240-243 inner with B); partners ascending, no atomics (L385)
struct BsrArgs {
  int32_t nclusters;      // clusters c_begin .. c_begin + nclusters - 1 (multi-GPU: the owned range)
  int32_t c_begin;
  int32_t max_rows;
  const int64_t* yoff;    // per cluster: first row in Y
  const int64_t* ooff;    // per cluster: first row in Om
  const int32_t* cnt;     // per cluster: rows
  const int32_t* ptr;
  const int32_t* idx;
  const int32_t* uidx;    // block of CSR entry e: uidx[e] (NULL: e)
  const int32_t* us;      // stored orientation of unique pair u: rows = cluster us[u]
  const int64_t* blk_off;
  const double* blk;
  const int32_t* kcnt;    // per partner cluster: rows of Om (NULL: cnt; non-symmetric ranks)
  int tmode;              // 0: direct iff us[u] == s; 1: every block direct; 2: every block transposed
  double* Y;
  int64_t ldy;
  const double* Om;
  int64_t ldo;
  int c0, ncols;
};
void launch_bsr(const BsrArgs& a, cudaStream_t st);

// CPQR of every panel A_c = Y(poff[c] : poff[c]+m[c], 0:d)^T (row ID via column ID, L173, L387)
// with threshold eps (R13/R14); W receives the factored panels (packed, ld = d).
struct CpqrArgs {
  int32_t nclusters;      // clusters c_begin .. c_begin + nclusters - 1
  int32_t c_begin;
  int32_t max_m;
  const double* Y;
  int64_t ldy;
  const int64_t* poff;
  const int32_t* m;
  int d;
  double eps;
  int kmax;
  double* W;
  int32_t* k;
  int32_t* perm;          // at poff[c]
  double* cert;           // 2 per cluster (min gap, stop margin)
  int64_t rows;           // total panel rows (poff range) of the depth
  // Adaptive convergence test early exit (exact: the same level decision, no arithmetic change).
  // A level is converged iff every cluster has m <= d or k <= d - 1 - p_os (R12); a cluster with
  // m > d whose residual norm still exceeds eps at step fail_cap = d - p_os - 1 will take >= d - p_os
  // pivots, so the level fails and this round's factorisations are all discarded.  That cluster
  // writes k = fail_k (= d - p_os) and raises *fail_flag; every panel polls the flag once per step
  // (one step late) and stops (k = steps done).  fail_flag NULL: off (fixed-rank builds).
  int32_t fail_cap = -1;
  int32_t fail_k = 0;
  int32_t* fail_flag = nullptr;
};
// returns the variant that ran: H2_CQ_V_WARP (warp per panel, m <= 64), H2_CQ_V_SMEM (CTA per
// panel, panel in shared memory) or H2_CQ_V_GLOBAL (CTA per panel, panel in global W).
// H2_CQ_VARIANT=warp|smem|global forces a variant where it applies (tests of each path).
int launch_cpqr(const CpqrArgs& a, cudaStream_t st);

// ID epilogue: X_c (m x k, U or [E1;E2]) from T = R11^{-1} R12 (R15); skeletons I~ (L224, L253)
struct IdArgs;
struct IdArgs {
  int32_t nclusters;      // clusters c_begin .. c_begin + nclusters - 1
  int32_t c_begin;
  const double* W;
  int d;
  const int64_t* poff;
  const int32_t* m;
  const int32_t* k;
  const int32_t* perm;
  const int64_t* xoff;
  double* X;
  const int32_t* ibar;    // Ibar_c = ibar + poff[c]
  const int64_t* roff;    // rank prefix sum of this depth
  int32_t* skel;
  int32_t max_k, max_red; // max k, max (m - k) over the clusters (grid / shared-memory sizing)
};
void launch_id(const IdArgs& a, cudaStream_t st);

// batchedShrink + batchedGemm upsweep for columns [c0,c1) (L222-223, L251-252):
// Yp(roff[c]+i) = Yl(poff[c] + J[i]);  Op(roff[c]+i) = sum_j X(j,i) Ol(poff[c]+j)
struct ShrinkArgs {
  int32_t nclusters;      // clusters c_begin .. c_begin + nclusters - 1
  int32_t c_begin;
  const int64_t* poff;
  const int32_t* m;
  const int32_t* k;
  const int32_t* perm;
  const int64_t* xoff;
  const double* X;
  const int64_t* roff;
  const double* Yl;
  const double* Ol;
  int64_t ld;
  double* Yp;
  double* Op;
  int64_t ldp;
  int c0, c1;
  int32_t max_k;          // max k over the clusters (grid sizing)
};
void launch_shrink_project(const ShrinkArgs& a, cudaStream_t st);

// ---- H^2 matvec pieces (CS4)
// xh(roff[c]+i, :) = sum_j X_c(j,i) xin(ioff[c]+j, :)       (upward; leaf: xin = x, ioff = begin)
struct UpArgs {
  int32_t nclusters;
  const int64_t* ioff;
  const int32_t* m;
  const int32_t* k;
  const int64_t* xoff;
  const double* X;
  const int64_t* roff;
  const double* xin;
  int64_t ldi;
  double* xh;
  int64_t ldh;
  int q;
  int32_t max_out;        // max k over the clusters (grid sizing; 0: derived per launch as 1024)
};
void launch_upward(const UpArgs& a, cudaStream_t st);
// yout(ioff[c]+j, :) = beta_in*yout + alpha * sum_i X_c(j,i) yh(roff[c]+i, :)     (downward / leaf out)
struct DownArgs {
  int32_t nclusters;
  const int64_t* ioff;
  const int32_t* m;
  const int32_t* k;
  const int64_t* xoff;
  const double* X;
  const int64_t* roff;
  const double* yh;
  int64_t ldh;
  double* yout;
  int64_t ldo;
  int q;
  double alpha;
  int accumulate;          // 1: yout += ..., 0: yout = ...
  int32_t max_out;        // max m over the clusters (grid sizing)
  int32_t c_begin;        // clusters c_begin .. c_begin + nclusters - 1 (a rank's owned range)
};
void launch_downward(const DownArgs& a, cudaStream_t st);
// y(rows of s) += alpha * sum_b Blk(s,b) x(rows of b)   (coupling B / dense D products)
struct SpmmArgs {
  int32_t nclusters;
  int32_t max_rows;
  const int64_t* yoff;
  const int64_t* xoff;
  const int32_t* cnt;
  const int32_t* ptr;
  const int32_t* idx;
  const int32_t* uidx;
  const int32_t* us;
  const int64_t* blk_off;
  const double* blk;
  const int32_t* kcnt;    // see BsrArgs
  int tmode;
  const double* x;
  int64_t ldx;
  double* y;
  int64_t ldy;
  int q;
  double alpha;
  int32_t c_begin;        // row clusters c_begin .. c_begin + nclusters - 1
};
void launch_spmm(const SpmmArgs& a, cudaStream_t st);

// ---- H^2 + low-rank update operators (h2update.cu, BASELINE configs[4])
// Y += U (U^T Omega): scratch >= (ceil(n/1024) + 1) * r * nc doubles
// Y += U (V^T Omega) (V NULL: V = U)
void launch_lowrank_sketch(const double* U, int64_t ldu, int r, const double* Om, int64_t ldo, int nc, int64_t n,
                           double* Y, int64_t ldy, double* scratch, cudaStream_t st, const double* V = nullptr,
                           int64_t ldv = 0);
struct UpdateDArgs {            // D_new = D_A + U(I_s) U(I_b)^T over unique near pairs
  int64_t nblocks;
  const int32_t* ulist;         // unique pairs to produce (a rank's owned pairs); NULL: 0..nblocks-1
  const int32_t *us, *ub, *cnt;
  const int64_t *begin, *off;
  const double* Dbase;
  double* out;
  const double* U;
  int64_t ldu;
  int r;
};
void launch_update_D(const UpdateDArgs& a, cudaStream_t st);
struct ExpandArgs {             // rows of A's expanded basis at the new skeletons of depth t
  int64_t npoints;
  const int32_t* pt_cluster;
  const int64_t* roff_new;
  const int32_t* skel_new;
  int nleaf;
  const int64_t* leaf_begin;
  int Dl, t;
  const int32_t* const* kb;     // per depth: base ranks
  const int64_t* const* xoff;   // per depth: base basis offsets
  const double* const* X;       // per depth: base bases
  int kmax;
  double* R;
  const int64_t* rowoff;        // per cluster of depth t: offset of R_s (kn_s x kb_s)
};
void launch_expand_rows(const ExpandArgs& a, cudaStream_t st);
struct UpdateBArgs {            // B_new = R_s B_A R_b^T + U(I~_s) U(I~_b)^T over unique far pairs
  int64_t nblocks;
  const int32_t* ulist;         // unique pairs to produce (a rank's owned pairs); NULL: 0..nblocks-1
  const int32_t *us, *ub, *kn, *kb;
  double* out;
  const int64_t* out_off;
  const double* R;
  const int64_t* rowoff;
  const double* Bbase;
  const int64_t* Boff;
  const double* U;
  int64_t ldu;
  int r;
  const int32_t* skel;
  const int64_t* roff_new;
  double* scratch;
  int64_t gmax;                 // scratch doubles per CTA (>= max kb_s * kn_b)
};
void launch_update_B(const UpdateBArgs& a, int grid, cudaStream_t st);
// non-symmetric update M = A_H + U V^T over ORDERED pairs e (h2_build_nonsym): D (coupling = false:
// cnt = leaf sizes, begin = leaf begins) or B (coupling = true: row side cnt/roff/skel, column side
// cnt2/roff2/skel2, R / R2 the base's expanded basis rows at the row / column skeletons)
struct UpdateNsArgs {
  int64_t nblocks;
  const int32_t* ulist = nullptr;   // ordered entries to produce (NULL: 0..nblocks-1; sharded builds)
  const int32_t *os, *ob;       // row / column cluster of entry e
  const int32_t* uidx;          // unique (base) pair of entry e
  const int32_t* us;            // stored orientation of the base's unique pair: rows = us[u]
  const double* Bbase;
  const int64_t* Boff;
  double* out;
  const int64_t* out_off;       // per ordered entry
  const int32_t *cnt, *cnt2, *kb;
  const int64_t* begin;
  const double *U, *V;
  int64_t ldu, ldv;
  int r;
  const double *R, *R2;
  const int64_t *rowoff, *rowoff2;
  const int32_t *skel, *skel2;
  const int64_t *roff, *roff2;
  double* scratch;
  int64_t gmax;
};
void launch_update_ns(const UpdateNsArgs& a, bool coupling, int grid, cudaStream_t st);
void launch_scale(double* y, int64_t n, int64_t ld, int q, double beta, cudaStream_t st);
// packed row e <-> panel row rows[e] (ncols columns): dir 0 gathers into buf, dir 1 scatters from it
void launch_rows_move(double* P, int64_t ld, const int32_t* rows, int64_t nrows, int ncols, double* buf, int dir,
                      cudaStream_t st);

// ---- exact-order mode (exact.cu, --fmad=false): the C oracle's operation order
void launch_exact_sketch(const KernelParams& kp, const double* X, const double* Yc, const double* Zc, int64_t n,
                         int64_t row0, int64_t row1, const double* Om, int64_t ldo, int ncols, double* Y, int64_t ldy,
                         cudaStream_t st);
void launch_exact_sumsq_leaf(const double* Y, const int64_t* leaf_begin, int cb, int ce, int64_t ld, int c0, int c1,
                             double* part, cudaStream_t st);
void launch_exact_sumsq_total(const double* part, int nleaf, double* acc, int* nonfinite, cudaStream_t st);
void launch_exact_bsr(const BsrArgs& a, cudaStream_t st);
void launch_exact_cpqr(const CpqrArgs& a, cudaStream_t st);
void launch_exact_id(const IdArgs& a, cudaStream_t st);

}  // namespace h2
