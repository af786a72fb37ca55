/*
 * h2.h -- C ABI of libh2: B200-native (sm_100a) bottom-up adaptive-sketching construction of
 * symmetric H^2 matrices (Boukaram, Liu, Ghysels, Li, "Adaptive Sketching Based Construction of
 * H2 Matrices on GPUs", arXiv 2506.16759; cited below as PAPER.md L<line>).
 *
 * The calls follow the paper's problem statement (Algorithm 1):
 *   Input : sample block size d, a hierarchical partitioning, a relative tolerance eps,
 *           a black-box sketch Y = K_blk(Omega) and a (batched) entry evaluator.
 *   Output: skeleton indices I~_tau, leaf bases U_tau, transfer matrices E, dense blocks D,
 *           coupling blocks B.
 *
 * Conventions (all entry points):
 *   - Every index is a TREE-ORDER index (position after the KD-tree permutation) unless named
 *     "original".  int64 for sizes/offsets, int32 for cluster-local quantities.
 *   - Dense blocks are row-major.  Y and Omega are row-major N x ncols with a leading dimension.
 *   - "dev" pointers are CUDA device memory of the current device, "host" pointers host memory.
 *   - Every call returns h2_status; on failure h2_last_error() gives a thread-local message.
 *     On failure nothing is leaked and any *out handle is set to NULL.
 *   - Handles are owned by the library; free them with the matching *_free call.  A built
 *     h2_matrix is immutable; h2_matvec may be called concurrently on different streams.
 *     An h2_matrix references the h2_tree it was built on: free the tree last.
 *   - stream arguments are cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered; h2_build synchronises the stream internally (it reads ranks
 *     back to size the next level, "prefix sum ... single allocation").
 */
#ifndef H2_H
#define H2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  H2_OK = 0,
  H2_ERR_INVALID_ARG = -1,
  H2_ERR_OOM = -2,
  H2_ERR_CUDA = -3,
  H2_ERR_NCCL = -4,          /* NCCL unavailable or an NCCL call failed (h2_comm_*)         */
  H2_ERR_CALLBACK = -5,      /* a user sketch/entry callback returned non-zero             */
  H2_ERR_NOT_CONVERGED = -6, /* adaptive sampling hit d_max; stats.failed_depth says where */
  H2_ERR_NONFINITE = -7      /* the sketch produced a non-finite sample                    */
} h2_status;

typedef struct h2_tree h2_tree;
typedef struct h2_matrix h2_matrix;

/* ---------------------------------------------------------------------------------------
 * Partition (§II-A; Algorithm 1 input "a hierarchical partitioning", L200)
 * KD-tree: complete binary tree, all leaves at depth Dl = min{D : ceil(n/2^D) <= leaf_size};
 * split the longest bbox axis (ties -> lowest axis) at the median of the stable order
 * (coordinate, original index), lower half ceil(m/2) points (R4).
 * Admissibility Eq.(1): adm(s,t) = s != t and (D(s)+D(t))/2 <= eta * Dist(s,t), D = bbox
 * diagonal, Dist = distance of bbox centres (H2_DIST_CENTER, R1) or minimum box-box
 * distance (H2_DIST_BOX).  Dual traversal from (root, root) (L127).
 * ------------------------------------------------------------------------------------- */
enum { H2_DIST_CENTER = 0, H2_DIST_BOX = 1 };

/* coords_host: n x dim row-major float64 in ORIGINAL order (1 <= dim <= 3, finite).
 * leaf_size >= 2, eta > 0.  The tree keeps a host copy and uploads tree-ordered coordinates
 * to the current device (used by the built-in kernels).  Errors: INVALID_ARG, OOM, CUDA. */
h2_status h2_tree_build(const double* coords_host, int64_t n, int32_t dim, int32_t leaf_size,
                        double eta, int32_t dist_rule, h2_tree** out);

typedef struct {
  int64_t n;
  int32_t dim, leaf_size, leaf_depth; /* depth 0 = root; paper level l = leaf_depth - depth + 1 */
  int32_t top_depth;                  /* coarsest depth with an admissible pair, -1 if none     */
  int64_t near_nnz;                   /* ordered inadmissible leaf pairs (incl. (tau,tau))      */
  int64_t far_nnz_total;              /* ordered admissible pairs over all depths               */
  int32_t csp;                        /* sparsity constant C_sp (max blocks per block row)      */
} h2_tree_info;
h2_status h2_tree_get_info(const h2_tree* tree, h2_tree_info* info);

/* h2_tree_build with the block partition built on a host thread: returns once the KD ordering
 * (R4) and the tree-order coordinates exist.  Every call that reads the partition
 * (h2_tree_get_info, h2_tree_export of near pairs, h2_tree_far_count / export_far, h2_build*)
 * waits for it; h2_build with the built-in exp dense-kernel sketch (symmetric, one GPU, RMS
 * tolerance rule) launches its first sketch pass BEFORE waiting, so the host's dual traversal
 * and CSR construction overlap the O(N^2) pass on the GPU (the end-to-end path of bench.py).
 * Arguments, ownership and errors as h2_tree_build; an error of the partition itself is reported
 * by the first call that waits for it. */
h2_status h2_tree_build_async(const double* coords_host, int64_t n, int32_t dim, int32_t leaf_size, double eta,
                              int32_t dist_rule, h2_tree** out);

/* Host copies of the partition.  perm[n] (tree index -> original index), begin/end of every
 * cluster in heap order (node (depth t, index c) at position 2^t - 1 + c; total 2^(Dl+1)-1
 * entries each), near pairs (near_nnz x 2, sorted), far pairs of one depth (sorted).
 * Any output pointer may be NULL to skip it. */
h2_status h2_tree_export(const h2_tree* tree, int64_t* perm, int64_t* begin, int64_t* end,
                         int32_t* near_pairs);
h2_status h2_tree_far_count(const h2_tree* tree, int32_t depth, int64_t* nnz);

/* A partition built elsewhere (e.g. by the CPU oracle), so that libh2 and another implementation
 * consume the SAME tree (Algorithm 1 takes "a hierarchical partitioning" as input).
 * All arrays are host memory owned by the caller (copied).  Layouts as h2_tree_export:
 *   coords    n x dim row-major, ORIGINAL order;  perm[n]: tree index -> original index
 *   begin/end cluster index ranges (tree order) in heap order, node (t, c) at 2^t - 1 + c,
 *             2^(leaf_depth+1) - 1 entries: a complete binary tree, children split their parent
 *             contiguously, all leaves at leaf_depth
 *   near      near_nnz ordered pairs (s, b) of leaves, symmetric set, including every (s, s)
 *   far[t]    far_nnz[t] ordered admissible pairs of depth t (s != b, symmetric), t = 0..leaf_depth
 * Checked (INVALID_ARG): permutation, nesting, ranges, duplicates, symmetry, and that the block
 * areas sum to n^2.  The admissibility rule is the caller's (eta / dist_rule are not used). */
typedef struct {
  int64_t n;
  int32_t dim, leaf_depth;
  const double* coords;
  const int64_t* perm;
  const int64_t* begin;
  const int64_t* end;
  int64_t near_nnz;
  const int32_t* near_pairs;
  const int64_t* far_nnz;
  const int32_t* const* far_pairs;
} h2_tree_desc;
h2_status h2_tree_import(const h2_tree_desc* desc, h2_tree** out);
h2_status h2_tree_export_far(const h2_tree* tree, int32_t depth, int32_t* far_pairs);
void h2_tree_free(h2_tree* tree);

/* ---------------------------------------------------------------------------------------
 * Operators.  Built-in kernels (§V-A) enable the fused device paths:
 *   H2_K_EXP       K(x,y) = exp(-|x-y|/param)                (Eq. cov, l = 0.2 in L431)
 *   H2_K_HELMHOLTZ K(x,y) = cos(param |x-y|)/|x-y|, 0 at x=y (Eq. ie, k = 3 in L439)
 *   H2_K_RATIONAL  K(x,y) = 1 / (1 + |x-y|^2 / param^2)   (not in the paper: a smooth test kernel
 *                  whose entries are correctly rounded operations only, r^2 = (dx*dx + dy*dy) + dz*dz,
 *                  so CPU and GPU evaluate it bitwise alike -- the exact-order parity mode,
 *                  SURVEY §8(c) contract 2; sketched by the exact-order kernel, any Omega)
 * ------------------------------------------------------------------------------------- */
enum { H2_K_EXP = 0, H2_K_HELMHOLTZ = 1, H2_K_RATIONAL = 2 };
typedef struct {
  int32_t kind;
  double param;
} h2_kernel;

/* Sketch request handed to a callback sampler (Algorithm 1 line 1, "Y = K_blk(Omega)",
 * PAPER.md L203/L216/L246).  Rows [row_begin,row_end) of Y for sample columns
 * [col0, col0+ncols) must be written: y[(i-row_begin)*ld_y + j] = sum_k K(i,k) omega[k*ld_omega+j]
 * for i in the row range (tree order).  omega holds ALL n rows.  Enqueue work on `stream`;
 * do not synchronise it.  Return 0 on success, anything else aborts h2_build with
 * H2_ERR_CALLBACK. */
typedef struct {
  int64_t n, row_begin, row_end;
  int32_t col0, ncols;
  const double* omega; /* dev */
  int64_t ld_omega;
  double* y;           /* dev */
  int64_t ld_y;
  void* stream;
  int32_t transpose;   /* h2_build_nonsym only: 1 = write y = K^T omega (the column sketch), 0 = K omega */
} h2_sketch_req;
typedef int (*h2_sketch_fn)(void* ctx, const h2_sketch_req* req);

/* H^2 + low-rank operator M = A_H + U U^T (BASELINE configs[4]): `base` is an
 * h2_matrix built on the SAME h2_tree, U is dev n x rank row-major (tree-order rows, leading dim
 * ld_U).  As a sketch: Y = A_H Omega (h2_matvec) + U (U^T Omega); rank 0 (U NULL) gives the pure
 * O(N) H^2-matvec sketch Y = A_H Omega (K_blk of an existing H^2, e.g. one of
 * K at a tighter tolerance).  As an entry evaluator (rank >= 1): D / B
 * blocks of M extracted from A_H's D / B and expanded bases plus U U^T. */
enum { H2_S_DENSE_KERNEL = 0, H2_S_CALLBACK = 1, H2_S_H2_LOWRANK = 2, H2_S_DENSE_MATRIX = 3 };
typedef struct {
  int32_t kind;       /* H2_S_DENSE_KERNEL: Y = K Omega with the built-in kernel below (O(N^2)) */
  h2_kernel kern;     /* H2_S_CALLBACK: fn(ctx, req);  H2_S_H2_LOWRANK: base + U                 */
  h2_sketch_fn fn;
  void* ctx;
  const h2_matrix* base;
  const double* U;
  int64_t ld_U;
  int32_t rank;
  /* H2_S_DENSE_MATRIX (an explicit operator such as a frontal matrix,
   * PAPER.md L443/L487): Y = A Omega with A dev n x n row-major in TREE order (leading dim ld_A),
   * on the int8 tensor cores in passes of 128 columns (h2_dense_op_sketch; the Omega stream), or
   * one cuBLAS DGEMM per draw with an external Omega, the non-symmetric build's K^T Psi, or
   * H2_DENSE_TC=0. */
  const double* A;
  int64_t ld_A;
  /* H2_S_H2_LOWRANK with a second factor (h2_build_nonsym only): M = A_H + U V^T, V dev n x rank
   * (leading dim ld_V); NULL = V is U (the symmetric update) */
  const double* V;
  int64_t ld_V;
} h2_sketch;

/* Batched entry evaluator ("batched entry generator ... evaluate all D or B at a
 * given level with a single kernel launch").  Block q: out[q][i*ld[q] + j] = K(row_idx[row_off[q]+i],
 * col_idx[col_off[q]+j]) for i < m[q], j < nc[q] (tree-order indices).  All arrays are device
 * arrays; `out` is a device array of device pointers.  Return 0 on success. */
typedef struct {
  int64_t nblocks;
  const int32_t* m;
  const int32_t* nc;
  const int64_t* row_off;
  const int64_t* col_off;
  const int32_t* row_idx;
  const int32_t* col_idx;
  double* const* out;
  const int32_t* ld;
  void* stream;
} h2_block_batch;
typedef int (*h2_entry_fn)(void* ctx, const h2_block_batch* batch);

enum { H2_E_BUILTIN = 0, H2_E_CALLBACK = 1, H2_E_H2_LOWRANK = 2, H2_E_DENSE_MATRIX = 3 };
typedef struct {
  int32_t kind;       /* H2_E_BUILTIN: entries of `kern` at the tree's coordinates              */
  h2_kernel kern;     /* H2_E_H2_LOWRANK: entries of base + U U^T (see h2_sketch)               */
  h2_entry_fn fn;
  void* ctx;
  const h2_matrix* base;
  const double* U;
  int64_t ld_U;
  int32_t rank;
  const double* A;    /* H2_E_DENSE_MATRIX: entries A[i * ld_A + j] (tree-order, dev)           */
  int64_t ld_A;
  const double* V;    /* H2_E_H2_LOWRANK: entries of A_H + U V^T (h2_build_nonsym); NULL = U    */
  int64_t ld_V;
} h2_entry;

/* ---------------------------------------------------------------------------------------
 * Build options (R9-R13, R26)
 * ------------------------------------------------------------------------------------- */
enum { H2_TOL_RMS = 0, H2_TOL_LITERAL = 1 };
typedef struct {
  int32_t d_init;      /* initial samples (Algorithm 1 line 1)                          [32]  */
  int32_t d_blk;       /* adaptive block: samples added per round (line 216/246)       [32]  */
  int32_t d_max;       /* sample cap; reaching it -> H2_ERR_NOT_CONVERGED              [512] */
  int32_t adaptive;    /* 1: §III-B convergence loop; 0: fixed sample size §III-A      [1]   */
  int32_t tol_rule;    /* H2_TOL_RMS: eps_l = s*tol*||Y||_F/sqrt(N)  (R10/R11)         [RMS] */
                       /* H2_TOL_LITERAL: eps_l = tol*norm (p_os = 0)          */
  double tol_safety;   /* s (at the leaf depth; see eps_decay, R31)          [0.04] */
  int32_t p_os;        /* oversampling margin: converged iff m<=d or k<=d-1-p_os (R12) [10]  */
  double norm;         /* nu for H2_TOL_LITERAL                                        [0]   */
  int32_t max_rank;    /* cap on every rank, <=0: none                                 [0]   */
  uint64_t seed;       /* Omega stream key (Philox4x32-10, R8)               [1]   */
  uint32_t stream_id;  /* Omega stream id (counter word 2)                             [0]   */
  /* A-posteriori check (PAPER.md L447 sampler-based error check; DESIGN.md
   * R30): after the build, e = ||H Om_h - K_blk(Om_h)||_F / ||K_blk(Om_h)||_F over verify_probes
   * held-out columns Om_h of stream stream_id + 2; while e > tol and fewer than verify_retries
   * rebuilds were made, tol_safety /= 3 and the build is redone.  One GPU only (ignored under a
   * communicator). */
  int32_t verify_probes;   /* q, 0 = off, <= 64                                           [0]   */
  int32_t verify_retries;  /* rebuild cap                                                  [2]   */
  /* level schedule of the threshold (R31; a study of S§8(f) NEXT #2, the paper's
   * "simple error compensation scheme" P:L496 being unspecified): eps_l at depth t is multiplied
   * by eps_decay^(leaf_depth - t); 1 = the uniform eps_l of R11                    [1.25] */
  double eps_decay;
  /* Exact-order mode (SURVEY §8(c) parity contract 2): every step runs the
   * exact-order kernels (sequential fma chains in the order the CPU reference states, correctly
   * rounded division / sqrt, no tensor cores, no tree reductions): with H2_K_RATIONAL and the
   * h2_omega stream the result is bitwise the C oracle's.  Slow by design (N <= ~10^4).
   * Symmetric builds with the built-in dense-kernel sketch and built-in entries only.     [0]   */
  int32_t exact_order;
  /* Optional external Omega (SURVEY §8(b) omega_external): dev, n x (>= d_max) row-major with
   * leading dim ld_omega_ext, tree-order rows; sample column c of the build is column c of this
   * array instead of the h2_omega stream (e.g. Gaussian test matrices).  The caller owns it and
   * keeps it alive during h2_build.  The int8 tensor-core sketch needs the stream (quarters), so
   * the dense-kernel sketch runs on the FP64 DMMA path.                                [NULL] */
  const double* omega_ext;
  int64_t ld_omega_ext;
  /* H2_TOL_LITERAL with norm <= 0: nu = ||K||_2 estimated by norm_iters power iterations through
   * the sketch operator ("an approximate norm ... provided via sketching"; the
   * start vector is column 0 of the h2_omega stream (seed, stream_id + 3)); the estimate is
   * reported in h2_build_stats.norm_est.                                                  [10]  */
  int32_t norm_iters;
  /* Work split of an H2_S_CALLBACK sketch under a communicator (BASELINE north
   * star "splitting the sketch's sample columns ... over GPUs"):
   *   H2_SPLIT_ROWS: every rank's callback computes its own leaf rows for all ncols columns
   *                  (row_begin/row_end = the rank's rows): no communication;
   *   H2_SPLIT_COLS: an opaque operator that can only produce whole columns (e.g. a black-box
   *                  matvec): rank g's callback computes ALL n rows of the column slice
   *                  [col0 + c_g, col0 + c_{g+1}), c_g = floor(g ncols / P), into a scratch panel,
   *                  and one all-to-all (comm->alltoallv, or grouped ncclSend/ncclRecv of the
   *                  in-library communicator) turns the column shards into row shards: rank g
   *                  sends rows [row_b(h), row_e(h)) of its slice to rank h and receives its own
   *                  rows of every other slice (n ncols 8 (P-1)/P bytes per draw in total).
   * Ignored on one GPU and for the built-in operators (which shard rows with no exchange). [ROWS] */
  int32_t sketch_split;
} h2_build_opts;
enum { H2_SPLIT_ROWS = 0, H2_SPLIT_COLS = 1 };
void h2_build_opts_default(h2_build_opts* opts);

enum {
  H2_PH_RAND = 0, H2_PH_SKETCH, H2_PH_GEN, H2_PH_BSR, H2_PH_CPQR, H2_PH_ID, H2_PH_MISC, H2_NPHASE
};
typedef struct {
  int32_t samples;            /* d at exit                                                  */
  int32_t failed_depth;       /* depth that hit d_max (H2_ERR_NOT_CONVERGED), else -1       */
  int32_t top_depth, leaf_depth;
  int32_t rounds[64];         /* convergence tests per depth                                */
  int32_t rank_min[64], rank_max[64];
  double rank_mean[64];
  double eps;                 /* final eps_l                                                */
  int64_t entries_D, entries_B; /* unique entries evaluated and stored                       */
  int64_t entries_sketch;     /* kernel entries evaluated by the built-in dense sketch      */
  int64_t sketch_columns;     /* Omega columns pushed through the sketch operator (>= samples:
                                 speculative 64-column tensor-core passes)       */
  int64_t bytes_U, bytes_E, bytes_B, bytes_D;
  int64_t launches;           /* device kernel launches issued by h2_build                  */
  double t_phase_ms[H2_NPHASE];
  double t_total_ms;
  double verify_error;        /* e of the returned matrix (opts.verify_probes > 0), else 0    */
  int32_t verify_rebuilds;    /* rebuilds with s/3 made by the a-posteriori check            */
  double tol_safety_used;     /* s of the returned matrix                                    */
  int32_t cpqr_variants;      /* bitmask of the CPQR kernels that ran (H2_CQ_V_*)             */
  double t_depth_ms[64];      /* device time of each processed depth t (its BSR subtraction,
                                 convergence tests, updateSamples replays, ID, shrink, B)   */
  double norm_est;            /* nu used by H2_TOL_LITERAL (opts.norm, or the power-iteration
                                 estimate when opts.norm <= 0), else 0                       */
  /* ALGORITHMIC work of the symmetric construction per phase (what the method computes / moves,
   * not what the kernels execute; DESIGN.md §6 "whole-build roofline"), this rank's clusters:
   *   bsr   2 nc sum_{ordered pairs} rows_s cols_b flops; 8 B per block entry read + Y/Omega rows
   *   cpqr  sum_c sum_{i<k_c} 4 (d - i)(m_c - i) flops (Householder, no pivot-norm work); panel in/out
   *   id    sum_c k_c^2 (m_c - k_c) flops (T = R11^-1 R12); panel read + X written
   *   shrink (counted under H2_PH_ID) sum_c 2 k_c (m_c - k_c) nc flops; panel rows in/out
   *   gen   8 B written per unique D / B entry (flops 0: the entry chain is counted by the caller)
   *   rand  8 B written per Omega entry
   * The dense sketch's own work (N^2 entries per pass + the contraction) is not included. */
  double work_flops[H2_NPHASE];
  double work_bytes[H2_NPHASE];
} h2_build_stats;
/* CPQR kernel variants (h2_build_stats.cpqr_variants; H2_CQ_VARIANT=warp|smem|global|cluster forces one
 * where it applies): one warp per panel (m <= 64), one CTA per panel with the panel in shared
 * memory, one CTA per panel with the panel in global memory (L1/L2 resident). */
enum { H2_CQ_V_WARP = 1, H2_CQ_V_SMEM = 2, H2_CQ_V_GLOBAL = 4, H2_CQ_V_EXACT = 8 /* exact-order mode */,
       H2_CQ_V_CLUSTER = 16 /* a cluster of 2 or 4 CTAs per panel, rows in distributed shared memory */ };

/* ---------------------------------------------------------------------------------------
 * Multi-GPU (§IV-B: "the batch count becomes roughly the number
 * of nodes per level divided by the number of GPUs").  One process per GPU; every rank calls
 * h2_build_dist collectively with the same tree, operators and options.  Cluster c of depth t
 * (2^t clusters) is owned by rank floor(c * nranks / 2^t): contiguous, subtree-aligned ranges.
 * A rank evaluates the sketch rows of its leaves (Omega is regenerated everywhere), the D / B
 * blocks touching its clusters, and the BSR / CPQR-ID / shrink-upsweep of its clusters; per
 * level it all-gathers ranks, skeleton indices I~ and the next level's Omega rows (the
 * exchange step of the north star).  The result is bitwise the same as a one-GPU build.
 * The communicator is supplied by the caller (torch.distributed / NCCL in the Python binding):
 *   allgatherv(ctx, buf, counts, displs, stream): buf is device memory; on entry the byte
 *   segment [displs[r], displs[r] + counts[r]) holds rank r's data on rank r; on return every
 *   rank holds every segment.  counts/displs are host arrays of nranks entries.  Stream-ordered
 *   on `stream`.  Return 0 on success (else the build fails with H2_ERR_CALLBACK).
 * ------------------------------------------------------------------------------------- */
typedef int (*h2_allgatherv_fn)(void* ctx, void* buf, const int64_t* counts, const int64_t* displs,
                                void* stream);
/* alltoallv(ctx, send, scounts, sdispls, recv, rcounts, rdispls, stream): send and recv are
 * distinct device buffers; byte segment [sdispls[r], sdispls[r] + scounts[r]) of send goes to
 * rank r, which receives it at [rdispls[me], rdispls[me] + rcounts[me]) of its recv (so
 * rcounts[r] on rank me == scounts[me] on rank r).  Host arrays of nranks entries; stream-ordered
 * on `stream`.  Used by sketch_split = H2_SPLIT_COLS only; may be NULL otherwise. */
typedef int (*h2_alltoallv_fn)(void* ctx, const void* send, const int64_t* scounts, const int64_t* sdispls,
                               void* recv, const int64_t* rcounts, const int64_t* rdispls, void* stream);
typedef struct {
  int32_t rank, nranks;
  h2_allgatherv_fn allgatherv;   /* caller's communicator (e.g. torch.distributed), or NULL      */
  void* ctx;
  void* nccl;                    /* library-owned NCCL communicator (h2_comm_init), used when
                                    allgatherv is NULL: grouped ncclBroadcast per segment,
                                    stream-ordered, no host synchronisation                    */
  h2_alltoallv_fn alltoallv;     /* caller's all-to-all (same ctx), or NULL: the NCCL
                                    communicator's grouped ncclSend / ncclRecv                  */
} h2_comm;

/* In-library NCCL communicator (one process per GPU; the NCCL library is loaded at run time,
 * libnccl.so.2 -- the one torch already loaded, if any).  Rank 0 calls h2_comm_get_unique_id
 * and sends the 128 bytes to every rank out of band (torch.distributed in the Python binding);
 * every rank then calls h2_comm_init collectively on its current device.  The returned h2_comm
 * is owned by the library (h2_comm_free).  Errors: H2_ERR_NCCL (library missing / NCCL error),
 * INVALID_ARG. */
h2_status h2_comm_get_unique_id(void* id128);
h2_status h2_comm_init(const void* id128, int32_t rank, int32_t nranks, h2_comm** out);
void h2_comm_free(h2_comm* comm);
/* The collective libh2 runs per level (exposed for tests and users): in-place all-gather of byte
 * segments [displs[r], displs[r] + counts[r]) of the device buffer buf, segment r valid on rank r
 * on entry, on every rank on return; counts/displs host arrays of nranks entries; stream-ordered.
 * Uses comm->allgatherv when set, else the NCCL communicator. */
h2_status h2_comm_allgatherv(const h2_comm* comm, void* buf, const int64_t* counts, const int64_t* displs,
                             void* stream);
/* The exchange of the column-split sketch (sketch_split = H2_SPLIT_COLS; exposed for tests and
 * users): all-to-all of byte segments as h2_alltoallv_fn above.  Uses comm->alltoallv when set,
 * else the NCCL communicator (one group of ncclSend / ncclRecv; the own segment is a device
 * copy).  Errors: INVALID_ARG (no all-to-all available, negative segments), NCCL, CALLBACK. */
h2_status h2_comm_alltoallv(const h2_comm* comm, const void* send, const int64_t* scounts, const int64_t* sdispls,
                            void* recv, const int64_t* rcounts, const int64_t* rdispls, void* stream);

/* Owned cluster range [*begin, *end) of `rank` among `nranks` at a depth with n_clusters
 * clusters (host logic, no device).  Errors: INVALID_ARG. */
h2_status h2_dist_range(int64_t n_clusters, int32_t rank, int32_t nranks, int64_t* begin, int64_t* end);

/* Algorithm 1 on the current device.  tree: from h2_tree_build.  tol >= 0.
 * sketch/entry: operators (see above).  stats may be NULL.  Errors: INVALID_ARG, OOM, CUDA,
 * CALLBACK, NOT_CONVERGED, NONFINITE; *out = NULL on error. */
h2_status h2_build(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                   const h2_build_opts* opts, void* stream, h2_matrix** out, h2_build_stats* stats);

/* h2_build over a communicator (comm NULL or nranks 1: same as h2_build).  The returned matrix
 * holds this rank's bases, the blocks touching its clusters, and every rank / skeleton index;
 * h2_matrix_allgather completes it on every rank (needed before h2_matvec / h2_export of the
 * bases and blocks, which fail with INVALID_ARG on a partial matrix).  nranks must be a power
 * of two <= 2^top_depth (subtree-aligned ownership).  H2 + low-rank operators (H2_S_H2_LOWRANK /
 * H2_E_H2_LOWRANK, SURVEY §8(e) "Config 5's H2 sketch is a distributed h2_matvec") need the base
 * complete on every rank (INVALID_ARG if partial): its matvec is row-sharded (upward pass over
 * all clusters, couplings / downward pass / dense leaves over the owned clusters: no
 * communication, bitwise the one-GPU rows) and its entries are extracted for the owned pairs. */
h2_status h2_build_dist(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                        const h2_build_opts* opts, const h2_comm* comm, void* stream, h2_matrix** out,
                        h2_build_stats* stats);
/* Non-symmetric construction ("the extension to the non-symmetric case is
 * straightforward"; R29): K ~ D + U B V^T with row bases U / E
 * from the sketch Y = K Omega and column bases V / F from Z = K^T Psi, built level by level in
 * lockstep (the two sides meet in the far-field subtraction).  Psi is the h2_omega stream
 * opts->stream_id + 1 (Omega: stream_id).  tol applies to the RMS row norm of Y and Z together;
 * a level converges when every cluster of both sides passes the test.  Operators: sketch
 * H2_S_DENSE_MATRIX (Z via A^T, cuBLAS), H2_S_CALLBACK (called with req->transpose = 0 and 1)
 * or H2_S_DENSE_KERNEL (the built-in kernels are symmetric: Z = K Psi); entry H2_E_BUILTIN,
 * H2_E_CALLBACK or H2_E_DENSE_MATRIX.  One GPU; h2_build_nonsym_dist shards it.  The result works
 * with h2_matvec (upward pass
 * with V, couplings, downward pass with U) and h2_export: H2_X_RANK/SKEL/BASIS/CERT give the row
 * side, H2_X_*_C the column side; D and B are stored for every ORDERED pair (s, b) in (s, b)
 * order, D_{s,b} m_s x m_b, B_{s,b} = K(I~_s, J~_b) k_s x kc_b.  Errors as h2_build. */
h2_status h2_build_nonsym(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                          const h2_build_opts* opts, void* stream, h2_matrix** out, h2_build_stats* stats);
/* The non-symmetric construction over a communicator (SURVEY §8(e) applied to NEXT #3): cluster
 * ownership, sharded sketch rows (Y and Z rows of the owned leaves; Omega and Psi regenerated on
 * every rank), owned-cluster BSR / CPQR-ID / shrink on both sides, the ordered D / B blocks with an
 * owned endpoint, per-level all-gathers of ranks and skeletons of both sides and the halo (or
 * all-gather) exchange of both sides' projected samples.  A callback sketch is called for the
 * rank's rows (row split only).  The result is partial until h2_matrix_allgather (bases,
 * certificates, ordered B and D by the owner of the row cluster); bitwise the one-GPU
 * h2_build_nonsym.  Arguments and errors as h2_build_nonsym and h2_build_dist. */
h2_status h2_build_nonsym_dist(const h2_tree* tree, const h2_sketch* sketch, const h2_entry* entry, double tol,
                               const h2_build_opts* opts, const h2_comm* comm, void* stream, h2_matrix** out,
                               h2_build_stats* stats);

/* Collective: all-gather bases X, certificates, B and D so that every rank holds the full
 * matrix (segments by owner of the cluster / of the stored block's row cluster). */
h2_status h2_matrix_allgather(h2_matrix* H, const h2_comm* comm, void* stream);

/* y = alpha * K_H * x + beta * y for ncols right-hand sides (H^2 matvec: upward pass, couplings,
 * downward pass, dense leaves).  x, y: dev, tree-order rows, row-major with leading dims
 * ldx, ldy >= ncols.  1 <= ncols <= 64. */
h2_status h2_matvec(const h2_matrix* H, const double* x, int64_t ldx, double* y, int64_t ldy,
                    int32_t ncols, double alpha, double beta, void* stream);

/* The paper's error measure ("a few iterations of the power method to approximate
 * the 2-norm of the difference between the constructed hierarchical matrix and the provided
 * sampler"): ||H - K_blk||_2 and ||K_blk||_2, each by `iters` power iterations
 * x <- A x / ||A x|| run independently from nvec unit start vectors (columns 0..nvec-1 of the
 * h2_omega stream (seed, stream_id)) in one block -- the dense sketch costs the same for 1 or 16
 * columns -- estimate = the largest ||A x|| of the last iteration; both operators symmetric
 * (symmetric H, K_blk = `sketch`, any kind: the FP64 DMMA path for the built-in kernels).
 * *err = the ratio; abs_err / knorm (may be NULL) the two estimates (each <= the true 2-norm).
 * 1 <= iters <= 1000, 1 <= nvec <= 64.
 * Errors: INVALID_ARG (partial or non-symmetric matrix, bad sketch), CUDA, CALLBACK, NONFINITE. */
h2_status h2_verify_2norm(const h2_matrix* H, const h2_sketch* sketch, int32_t iters, int32_t nvec, uint64_t seed,
                          uint32_t stream_id, void* stream, double* err, double* abs_err, double* knorm);

/* A-posteriori error estimate: Om_h = ncols columns of the
 * h2_omega stream (seed, stream_id), Y_h = K_blk(Om_h) with `sketch` (any kind; a callback is
 * called once for all n rows with transpose = 0), *err = ||H Om_h - Y_h||_F / ||Y_h||_F.
 * 1 <= ncols <= 64.  Errors: INVALID_ARG (partial matrix, bad sketch), CUDA, CALLBACK. */
h2_status h2_verify(const h2_matrix* H, const h2_sketch* sketch, int32_t ncols, uint64_t seed,
                    uint32_t stream_id, void* stream, double* err);

/* Built-in dense operator product, rows [row_begin,row_end): y = K(rows,:) * omega (the dense
 * sketch of BASELINE configs[1], also the multi-GPU row shard).  omega: dev, all n rows.
 * flags: H2_SKETCH_OMEGA_QUARTERS asserts every omega entry is q/4 with integer |q| <= 32 (true
 * for the h2_omega stream); it enables the int8 tensor-core path: K evaluated in FP64, rounded
 * once to a fixed-point grid (exp: 2^-47, 6 byte slices, 160-column passes; Helmholtz: 2^(E-51),
 * 7 slices; R32) and contracted exactly in integers.  Without it (arbitrary omega) the
 * FP64 DMMA path runs.  Environment: H2_TC_SLICES=7 selects the 52-bit grid for exp too. */
enum { H2_SKETCH_OMEGA_QUARTERS = 1 };
h2_status h2_dense_sketch(const h2_tree* tree, h2_kernel kern, int64_t row_begin, int64_t row_end,
                          const double* omega, int64_t ld_omega, int32_t ncols, double* y,
                          int64_t ld_y, int32_t flags, void* stream);

/* Explicit dense operator product (the H2_S_DENSE_MATRIX sketch), rows
 * [row_begin, row_end): y = A(rows, :) omega, A dev row-major n x n (leading dim lda >= n, tree
 * order), omega dev all n rows.  flags & H2_SKETCH_OMEGA_QUARTERS (omega = the h2_omega stream):
 * int8 tensor cores -- A rounded once to a signed 53-bit fixed point of scale 2^E >= max|A|
 * (<= 2^-52 max|A| per entry, the normwise error level of an FP64 GEMM), 7 byte slices, exact
 * int32 contraction, A read once per 128 columns; otherwise one cuBLAS DGEMM.  Errors:
 * INVALID_ARG, CUDA. */
h2_status h2_dense_op_sketch(const double* A, int64_t lda, int64_t n, int64_t row_begin, int64_t row_end,
                             const double* omega, int64_t ld_omega, int32_t ncols, double* y, int64_t ld_y,
                             int32_t flags, void* stream);

/* Omega stream (Philox4x32-10 -> centred binomial (popcount(64 bits) - 32)/4, R8):
 * rows [row0,row0+nrows) x sample columns [col0,col0+ncols) into out (dev, row-major, ld). */
h2_status h2_omega(uint64_t seed, uint32_t stream_id, int64_t row0, int64_t nrows, int32_t col0,
                   int32_t ncols, double* out, int64_t ld, void* stream);

/* ---------------------------------------------------------------------------------------
 * Inspection (tests, verification).  Sizes first, then copies into caller buffers (host or
 * device: the copy kind is inferred).  Layouts:
 *   rank[t]   : int32 per cluster of depth t, for top_depth <= t <= leaf_depth
 *   skel[t]   : int32, concatenated I~_tau in pivot order (offsets = prefix sum of rank)
 *   basis[t]  : float64, concatenated row-major X_tau (m_tau x k_tau): U_tau at the leaf depth,
 *               [E_nu1; E_nu2] above (m_tau = k_nu1 + k_nu2), offsets = prefix sum m*k
 *   D         : float64, unique near pairs (s <= b) in sorted order, each m_s x m_b row-major
 *   B[t]      : float64, unique far pairs (s < b) of depth t in sorted order, k_s x k_b
 *   cert[t]   : float64 pairs (min pivot gap, stop margin) per cluster (CPQR certification)
 * depth = H2_ALL_DEPTHS (-1) with H2_X_RANK / H2_X_SKEL (or the _C forms): every processed depth
 * top_depth..leaf_depth concatenated in that order, in ONE call (the end-to-end result read).
 * ------------------------------------------------------------------------------------- */
#define H2_ALL_DEPTHS (-1)
enum { H2_X_RANK = 0, H2_X_SKEL, H2_X_BASIS, H2_X_D, H2_X_B, H2_X_CERT,
       /* column side of a non-symmetric matrix (h2_build_nonsym): ranks, J~, V / [F1; F2], cert */
       H2_X_RANK_C, H2_X_SKEL_C, H2_X_BASIS_C, H2_X_CERT_C };
h2_status h2_export_size(const h2_matrix* H, int32_t what, int32_t depth, int64_t* count);
h2_status h2_export(const h2_matrix* H, int32_t what, int32_t depth, void* dst);
h2_status h2_matrix_get_stats(const h2_matrix* H, h2_build_stats* stats);
int64_t h2_matrix_device_bytes(const h2_matrix* H);
/* Device memory held by libh2's block cache (freed workspaces kept for reuse across builds, the
 * "single allocation per operation" of PAPER.md L384) on the current device, and its release
 * (cudaFree of every cached block after a device synchronisation). */
int64_t h2_cache_bytes(void);
void h2_cache_trim(void);
void h2_free(h2_matrix* H);

const char* h2_last_error(void);
const char* h2_version(void);

#ifdef __cplusplus
}
#endif
#endif /* H2_H */
