/*
 * h2oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY) for arXiv 2506.16759, Algorithm 1.
 *
 * A plain C implementation of the bottom-up (adaptive) sketching construction of a symmetric H^2
 * matrix (Algorithm 1; §III-A; adaptive §III-B), written from
 * the paper step by step, with EVERY floating-point operation in a fixed, stated order
 * (DESIGN.md §3 "exact-order specification").  It is the second oracle of this repo, beside the
 * numpy one (oracle/h2.py): same readings, independent code.  Only tests/, __graft_entry__.smoke()
 * and bench.py's reference / cpu_baseline legs may load it (through oracle/c_h2.py).  It shares
 * no code with libh2 (paper_2506_16759_b200/) and includes none of its headers.
 *
 * Uses: (1) parity in exact-order mode -- libh2 with opts.exact_order = 1 on the rational test
 * kernel performs the same operations in the same order, so U/E/B/D/skeletons/ranks agree
 * bitwise; (2) the timed CPU baseline (OpenMP over the rows / clusters / blocks of a level; each
 * output element is computed by one thread in the stated order, so results do not depend on the
 * thread count).
 *
 * Build: gcc -O3 -mavx2 -mfma -ffp-contract=off -fopenmp -shared -fPIC (no contraction: a*b+c stays two
 * roundings; every fused multiply-add below is an explicit fma()).
 *
 * Operation order (the specification both paths follow):
 *   r2(x,y)      = (dx*dx + dy*dy) + dz*dz, d. = x. - y. (coordinates zero-padded to 3D)
 *   K_rational   = 1 / (1 + r2 / l2), l2 = l*l        (all correctly rounded: bitwise portable)
 *   K_exp        = exp(-sqrt(r2) / l)  (PAPER.md Eq. cov; libm: not bitwise portable)
 *   K_helmholtz  = cos(k sqrt(r2)) / sqrt(r2), 0 at r2 = 0 (Eq. ie, R20)
 *   sketch       Y(i,j) = fma-chain over k = 0..n-1 ascending of K(i,k) Omega(k,j), from 0
 *   sum of sq.   per leaf c: p_c = fma-chain over rows i ascending, columns j ascending of y^2;
 *                draw total = ((p_0 + p_1) + ...) over leaves ascending; acc = acc + total
 *   eps_t        = lvl * ((s * tol) * sqrt(acc / n)), lvl = eps_decay^(Dl - t) (pow), RMS rule;
 *                = lvl * (tol * nu) literal rule                        (R10/R11/R31)
 *   BSR          Y(i,j) = Y(i,j) - s_b, partners b ascending, s_b = fma-chain over k ascending of
 *                Blk(i,k) Om(k,j) from 0 (Blk = stored block or its transpose, R18/R19)
 *   CPQR (R12-R14) on A = (Y^loc)^T, column j = panel row j:
 *                norm_j = sqrt(fma-chain over r = i..d-1 of A(r,j)^2); pivot = max, lowest index
 *                on ties; stop if i == kcap or !(max > eps); Householder (dlarfg): x2 = fma-chain
 *                r = i+1..d-1, xnorm = sqrt(x2); xnorm == 0 -> tau = 0, beta = alpha; else
 *                h = sqrt(fma(alpha, alpha, x2)), beta = alpha < 0 ? h : -h,
 *                tau = (beta - alpha) / beta; v(r) = A(r,i) / (alpha - beta) (r > i), v(i) = 1;
 *                trailing column j: w = fma-chain r = i..d-1 of v(r) A(r,j), w = w * tau,
 *                A(r,j) = fma(-w, v(r), A(r,j)), next norm from the updated r > i entries.
 *                Certificates: gap = min (best - second) / best, margin = min |best - eps| / eps.
 *   ID (R15)     T(i,c) = (R(i,k+c) + fma-chain j = i+1..k-1 of -R(i,j) T(j,c)) / R(i,i), i desc.
 *                X(J_i,:) = e_i, X(Rhat_c, i) = T(i,c)  (Eq.(3))
 *   project      Om'(i,j) = Om(J_i,j) then fma-chain c ascending of X(Rhat_c,i) Om(Rhat_c,j)
 *   shrink       Y'(i,j) = Y^loc(J_i,j)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define H2O_MAXD 64

/* ------------------------------------------------------------------------------------------ */
/* interface (mirrored by oracle/c_h2.py)                                                      */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int32_t leaf_depth;                       /* depth of the leaves (root 0); complete tree      */
  const double* pts;                        /* n x 3 tree order, zero padded                    */
  const int64_t* begin;                     /* heap order: node (t,c) at 2^t - 1 + c            */
  const int64_t* end;
  const int64_t* near_ptr;                  /* leaf-depth CSR of N_tau (incl. tau), sorted      */
  const int32_t* near_idx;
  const int64_t* far_ptr[H2O_MAXD];         /* per depth CSR of F_tau (sorted), NULL = none     */
  const int32_t* far_idx[H2O_MAXD];
} h2o_tree;

/* H2O_K_TABLE: K(i, k) = dense[i * ld_dense + k] (tree-order indices) -- an explicit operator for
 * the pins that need a prescribed matrix (known-rank recovery, rank-1, zero) */
enum { H2O_K_EXP = 0, H2O_K_HELMHOLTZ = 1, H2O_K_RATIONAL = 2, H2O_K_TABLE = 3 };

typedef struct {
  int32_t d_init, d_blk, d_max, adaptive, tol_rule; /* tol_rule 0 = RMS, 1 = literal         */
  double tol_safety, norm, eps_decay;
  int32_t p_os, max_rank;
  uint64_t seed;
  uint32_t stream_id;
  int32_t threads;                          /* OpenMP threads, <= 0: runtime default            */
  const double* omega_ext;                  /* optional n x ld_ext row-major Omega (host)       */
  int64_t ld_ext;
  const double* dense;                      /* H2O_K_TABLE operator, n x ld_dense (host)        */
  int64_t ld_dense;
  /* sketch supplied as a table (SURVEY §8(d) "the oracle's construction proper, timed with the
   * sketch supplied as a table"): Y(:, c) = y_table column c for c < table_cols; a draw beyond
   * the table fails (status -2).  The Omega columns are still the oracle's own stream. */
  const double* y_table;
  int64_t ld_table;
  int32_t table_cols;
} h2o_opts;

typedef struct {
  int32_t status;                           /* 0 ok, -6 not converged, -1 bad argument,
                                               -2 sketch table exhausted                        */
  int32_t samples, top, leaf_depth, failed_depth;
  int32_t rounds[H2O_MAXD];
  double eps;
  double t_sketch, t_gen, t_bsr, t_cpqr, t_id, t_total;   /* seconds (wall, omp_get_wtime)    */
  /* export arrays, layouts as include/h2.h "Inspection" (per depth t in [top, leaf_depth]) */
  int32_t* rank[H2O_MAXD];
  int32_t* skel[H2O_MAXD];
  double* basis[H2O_MAXD];
  double* cert[H2O_MAXD];
  double* B[H2O_MAXD];
  int64_t nskel[H2O_MAXD], nbasis[H2O_MAXD], nB[H2O_MAXD];
  double* D;
  int64_t nD;
} h2o_result;

/* ------------------------------------------------------------------------------------------ */
static double wtime(void) {
#ifdef _OPENMP
  return omp_get_wtime();
#else
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
#endif
}

static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s);
  if (!p) {
    fprintf(stderr, "h2oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ---- Philox4x32-10 (Salmon et al. SC'11) and the centred binomial Omega (R8) ------ */
static void philox(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
  }
}

void h2o_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  philox(c, key[0], key[1]);
  memcpy(out, c, sizeof c);
}

/* Omega(i, j) = (popcount(w0) + popcount(w1) - 32)/4 (j even) or (popcount(w2)+popcount(w3)-32)/4
 * (j odd), counter (i, j/2, stream, 0), key (seed lo, seed hi) */
static double omega_entry(uint64_t seed, uint32_t stream, int64_t i, int64_t j) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)(j >> 1), stream, 0u};
  philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const int pc = (j & 1) ? __builtin_popcount(c[2]) + __builtin_popcount(c[3])
                         : __builtin_popcount(c[0]) + __builtin_popcount(c[1]);
  return (double)(pc - 32) / 4.0;
}

void h2o_omega(uint64_t seed, uint32_t stream, int64_t row0, int64_t nrows, int64_t col0, int32_t ncols,
               double* out, int64_t ld) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nrows; ++i)
    for (int32_t j = 0; j < ncols; ++j) out[i * ld + j] = omega_entry(seed, stream, row0 + i, col0 + j);
}

/* ---- kernels ------------------------------------------------------------------------------ */
typedef struct {
  int kind;
  double param, l2;
  const double* pts;
  const double* dense;
  int64_t ld;
} kern_t;

static inline double r2_of(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return (dx * dx + dy * dy) + dz * dz;
}

static inline double kval_pts(const kern_t* K, const double* a, const double* b) {
  const double r2 = r2_of(a, b);
  switch (K->kind) {
    case H2O_K_EXP: return exp(-sqrt(r2) / K->param);
    case H2O_K_HELMHOLTZ: {
      if (r2 == 0.0) return 0.0;
      const double r = sqrt(r2);
      return cos(K->param * r) / r;
    }
    default: return 1.0 / (1.0 + r2 / K->l2);
  }
}

/* K(i, k) for tree-order indices */
static inline double kval(const kern_t* K, int64_t i, int64_t k) {
  if (K->kind == H2O_K_TABLE) return K->dense[i * K->ld + k];
  return kval_pts(K, K->pts + 3 * i, K->pts + 3 * k);
}

void h2o_kernel_block(int kind, double param, const double* pts, const int64_t* rows, int64_t nr,
                      const int64_t* cols, int64_t nc, double* out) {
  kern_t K = {kind, param, param * param, pts, NULL, 0};
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t j = 0; j < nc; ++j) out[i * nc + j] = kval(&K, rows[i], cols[j]);
}

/* dense sketch rows [r0, r1): Y(i, j) = sum_k K(i, k) Om(k, j), k ascending, fma from 0 */
static void sketch_rows(const kern_t* K, int64_t n, int64_t r0, int64_t r1, const double* Om,
                        int64_t ldo, int nc, double* Y, int64_t ldy) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = r0; i < r1; ++i) {
    double* y = Y + (i - r0) * ldy;
    for (int j = 0; j < nc; ++j) y[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double kv = kval(K, i, k);
      const double* o = Om + k * ldo;
      for (int j = 0; j < nc; ++j) y[j] = fma(kv, o[j], y[j]);
    }
  }
}

void h2o_dense_sketch(int kind, double param, const double* pts, int64_t n, int64_t r0, int64_t r1,
                      const double* Om, int64_t ldo, int32_t nc, double* Y, int64_t ldy) {
  kern_t K = {kind, param, param * param, pts, NULL, 0};
  sketch_rows(&K, n, r0, r1, Om, ldo, nc, Y, ldy);
}

/* ---- CPQR + certificates (R12-R14), one panel ---------------------------------------------- */
/* A: m rows (= columns of the CPQR operand) x d, row stride d, factored in place; perm: m */
static int cpqr_panel(double* A, int m, int d, double eps, int kmax, int32_t* perm, double* nrm, double* v,
                      double* cert) {
  for (int j = 0; j < m; ++j) {
    double q = 0.0;
    for (int r = 0; r < d; ++r) q = fma(A[(int64_t)j * d + r], A[(int64_t)j * d + r], q);
    nrm[j] = sqrt(q);
    perm[j] = j;
  }
  const int kfull = d < m ? d : m;
  const int kcap = kmax > 0 ? (kmax < kfull ? kmax : kfull) : kfull;
  double gap = INFINITY, margin = INFINITY;
  int k = 0;
  for (int i = 0;; ++i) {
    if (i >= m) break;
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
    if (eps > 0 && i < kfull) margin = fmin(margin, fabs(bv - eps) / eps);
    if (i == kcap || !(bv > eps)) {
      k = i;
      break;
    }
    if (sv >= 0) gap = fmin(gap, (bv - sv) / bv);
    double* Ai = A + (int64_t)i * d;
    if (bi != i) {
      double* Ap = A + (int64_t)bi * d;
      for (int r = 0; r < d; ++r) {
        const double x = Ai[r];
        Ai[r] = Ap[r];
        Ap[r] = x;
      }
      const int32_t q = perm[i];
      perm[i] = perm[bi];
      perm[bi] = q;
      const double x = nrm[i];
      nrm[i] = nrm[bi];
      nrm[bi] = x;
    }
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
    const double den = alpha - beta;
    v[i] = 1.0;
    for (int r = i + 1; r < d; ++r) {
      v[r] = tau != 0.0 ? Ai[r] / den : 0.0;
      Ai[r] = 0.0;
    }
    Ai[i] = beta;
    for (int j = i + 1; j < m; ++j) {
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
    k = i + 1;
  }
  cert[0] = gap;
  cert[1] = margin;
  return k;
}

/* exported for the LAPACK pin: A given as m x d (row j = column j of the CPQR operand) */
int h2o_cpqr(double* A, int32_t m, int32_t d, double eps, int32_t kmax, int32_t* perm, double* cert) {
  double* nrm = (double*)xcalloc(m + 1, sizeof(double));
  double* v = (double*)xcalloc(d + 1, sizeof(double));
  const int k = cpqr_panel(A, m, d, eps, kmax, perm, nrm, v, cert);
  free(nrm);
  free(v);
  return k;
}

/* ---- per-depth state ------------------------------------------------------------------------ */
typedef struct {
  int nclus;
  int32_t *m, *k;
  int64_t *poff, *roff, *xoff;
  int64_t rows, rtot, xtot;
  int32_t* perm;  /* per panel row: local pivot order */
  double* W;      /* factored panel rows x d (row stride d) */
  double* X;
  int32_t* skel;
  double* cert;
} lvl_t;

typedef struct {
  double *Y, *O;
  int64_t rows, ld;
} panel_t;

typedef struct {
  const h2o_tree* T;
  kern_t K;
  const h2o_opts* o;
  double tol;
  int Dl, top, d;
  int64_t n;
  lvl_t L[H2O_MAXD];
  /* unique pairs and offsets: near (s <= b) and far per depth (s < b) */
  int64_t nu_near, *un_s, *un_b, *D_off;
  int64_t nu_far[H2O_MAXD];
  int64_t *uf_s[H2O_MAXD], *uf_b[H2O_MAXD], *B_off[H2O_MAXD];
  double* D;
  double* B[H2O_MAXD];
  double acc;             /* ||Y||_F^2 over all draws */
  int table_short;        /* a draw went beyond the sketch table */
  h2o_result* res;
} bld_t;

static inline int64_t beg(const bld_t* b, int t, int c) { return b->T->begin[((int64_t)1 << t) - 1 + c]; }
static inline int64_t endd(const bld_t* b, int t, int c) { return b->T->end[((int64_t)1 << t) - 1 + c]; }

static void panel_alloc(panel_t* P, int64_t rows, int64_t ld) {
  P->rows = rows;
  P->ld = ld;
  P->Y = (double*)xcalloc((size_t)(rows > 0 ? rows : 1) * (size_t)ld, sizeof(double));
  P->O = (double*)xcalloc((size_t)(rows > 0 ? rows : 1) * (size_t)ld, sizeof(double));
}
static void panel_free(panel_t* P) {
  free(P->Y);
  free(P->O);
  P->Y = P->O = NULL;
  P->rows = P->ld = 0;
}
/* widen to >= need columns, keeping the first d */
static void panel_grow(panel_t* P, int need, int d) {
  if (need <= P->ld) return;
  panel_t Q;
  panel_alloc(&Q, P->rows, need);
  for (int64_t i = 0; i < P->rows; ++i) {
    memcpy(Q.Y + i * Q.ld, P->Y + i * P->ld, sizeof(double) * d);
    memcpy(Q.O + i * Q.ld, P->O + i * P->ld, sizeof(double) * d);
  }
  panel_free(P);
  *P = Q;
}

/* unique pairs of a symmetric CSR, sorted (s, b), b >= s (strict: b > s) */
static int64_t unique_pairs(const int64_t* ptr, const int32_t* idx, int nrows, int strict, int64_t** us, int64_t** ub) {
  int64_t cnt = 0;
  for (int s = 0; s < nrows; ++s)
    for (int64_t e = ptr[s]; e < ptr[s + 1]; ++e)
      if (strict ? idx[e] > s : idx[e] >= s) ++cnt;
  *us = (int64_t*)xcalloc(cnt, sizeof(int64_t));
  *ub = (int64_t*)xcalloc(cnt, sizeof(int64_t));
  cnt = 0;
  for (int s = 0; s < nrows; ++s)
    for (int64_t e = ptr[s]; e < ptr[s + 1]; ++e)
      if (strict ? idx[e] > s : idx[e] >= s) {
        (*us)[cnt] = s;
        (*ub)[cnt] = idx[e];
        ++cnt;
      }
  return cnt;
}

/* position of the unique pair {min(s,b), max(s,b)} (binary search in the sorted list) */
static int64_t find_pair(const int64_t* us, const int64_t* ub, int64_t nu, int64_t s, int64_t b) {
  const int64_t a = s < b ? s : b, c = s < b ? b : s;
  int64_t lo = 0, hi = nu;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (us[mid] < a || (us[mid] == a && ub[mid] < c)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* ---- steps ------------------------------------------------------------------------------- */
/* line 1 / 216 / 246: Omega columns [c0, c0+nc) -> O, Y = K_blk(Omega) -> Y; ||Y||^2 (R10) */
static void draw(bld_t* b, double* Y, double* O, int64_t ld, int c0, int nc) {
  const int64_t n = b->n;
  if (b->o->omega_ext) {
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < nc; ++j) O[i * ld + j] = b->o->omega_ext[i * b->o->ld_ext + c0 + j];
  } else {
    h2o_omega(b->o->seed, b->o->stream_id, 0, n, c0, nc, O, ld);
  }
  double t0 = wtime();
  if (b->o->y_table) {
    if (c0 + nc > b->o->table_cols) {
      b->table_short = 1;
      nc = b->o->table_cols > c0 ? b->o->table_cols - c0 : 0;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < nc; ++j) Y[i * ld + j] = b->o->y_table[i * b->o->ld_table + c0 + j];
  } else {
    sketch_rows(&b->K, n, 0, n, O, ld, nc, Y, ld);
  }
  b->res->t_sketch += wtime() - t0;
  const int nleaf = 1 << b->Dl;
  double* part = (double*)xcalloc(nleaf, sizeof(double));
#pragma omp parallel for schedule(static)
  for (int c = 0; c < nleaf; ++c) {
    double p = 0.0;
    for (int64_t i = beg(b, b->Dl, c); i < endd(b, b->Dl, c); ++i)
      for (int j = 0; j < nc; ++j) p = fma(Y[i * ld + j], Y[i * ld + j], p);
    part[c] = p;
  }
  double tot = 0.0;
  for (int c = 0; c < nleaf; ++c) tot = tot + part[c];
  free(part);
  b->acc = b->acc + tot;
}

static double eps_now(const bld_t* b, int t) {
  const h2o_opts* o = b->o;
  const double lvl = o->eps_decay == 1.0 ? 1.0 : pow(o->eps_decay, (double)(b->Dl - t));
  if (o->tol_rule == 0) return lvl * (o->tol_safety * b->tol * sqrt(b->acc / (double)b->n));
  return lvl * (b->tol * o->norm);
}

/* BSR subtraction on the panel of depth t, columns [0, nc) of Y / O (pointers at the first
 * column): leaf (t == Dl) with D over N_tau (L213), inner with B of depth t+1 over F_nu of each
 * child nu (L240-243). */
static void bsr(bld_t* b, int t, double* Y, const double* O, int64_t ld, int nc) {
  double t0 = wtime();
  const int leaf = t == b->Dl;
  const int u = leaf ? t : t + 1;                 /* depth of the block rows */
  const int nr = 1 << u;
  const int64_t* ptr = leaf ? b->T->near_ptr : b->T->far_ptr[u];
  const int32_t* idx = leaf ? b->T->near_idx : b->T->far_idx[u];
  if (!ptr) return;
  const int64_t* us = leaf ? b->un_s : b->uf_s[u];
  const int64_t* ub = leaf ? b->un_b : b->uf_b[u];
  const int64_t nu = leaf ? b->nu_near : b->nu_far[u];
  const int64_t* off = leaf ? b->D_off : b->B_off[u];
  const double* blk = leaf ? b->D : b->B[u];
  const lvl_t* C = &b->L[u];
#pragma omp parallel for schedule(dynamic, 4)
  for (int c = 0; c < nr; ++c) {
    const int64_t yo = leaf ? beg(b, u, c) : C->roff[c];
    const int mc = leaf ? (int)(endd(b, u, c) - beg(b, u, c)) : C->k[c];
    double* s = (double*)xcalloc(nc + 1, sizeof(double));
    for (int64_t e = ptr[c]; e < ptr[c + 1]; ++e) {
      const int bb = idx[e];
      const int64_t bo = leaf ? beg(b, u, bb) : C->roff[bb];
      const int mb = leaf ? (int)(endd(b, u, bb) - beg(b, u, bb)) : C->k[bb];
      const int64_t q = find_pair(us, ub, nu, c, bb);
      const double* Bq = blk + off[q];
      const int direct = c <= bb;            /* stored (min, max): rows = min */
      for (int i = 0; i < mc; ++i) {
        for (int j = 0; j < nc; ++j) s[j] = 0.0;
        for (int kk = 0; kk < mb; ++kk) {
          const double a = direct ? Bq[(int64_t)i * mb + kk] : Bq[(int64_t)kk * mc + i];
          const double* o = O + (bo + kk) * ld;
          for (int j = 0; j < nc; ++j) s[j] = fma(a, o[j], s[j]);
        }
        double* y = Y + (yo + i) * ld;
        for (int j = 0; j < nc; ++j) y[j] = y[j] - s[j];
      }
    }
    free(s);
  }
  b->res->t_bsr += wtime() - t0;
}

static void setup_level(bld_t* b, int t) {
  lvl_t* L = &b->L[t];
  L->nclus = 1 << t;
  L->m = (int32_t*)xcalloc(L->nclus, sizeof(int32_t));
  L->k = (int32_t*)xcalloc(L->nclus, sizeof(int32_t));
  L->poff = (int64_t*)xcalloc(L->nclus, sizeof(int64_t));
  L->rows = 0;
  for (int c = 0; c < L->nclus; ++c) {
    if (t == b->Dl) {
      L->m[c] = (int32_t)(endd(b, t, c) - beg(b, t, c));
      L->poff[c] = beg(b, t, c);
    } else {
      const lvl_t* C = &b->L[t + 1];
      L->m[c] = C->k[2 * c] + C->k[2 * c + 1];
      L->poff[c] = C->roff[2 * c];
    }
    L->rows += L->m[c];
  }
  L->perm = (int32_t*)xcalloc(L->rows, sizeof(int32_t));
  L->cert = (double*)xcalloc(2 * (size_t)L->nclus, sizeof(double));
}

/* convergence test / ID factorisation of every panel of depth t (d columns of Y) */
static void cpqr_level(bld_t* b, int t, const double* Y, int64_t ld, double eps) {
  double t0 = wtime();
  lvl_t* L = &b->L[t];
  const int d = b->d;
  free(L->W);
  L->W = (double*)xcalloc((size_t)(L->rows > 0 ? L->rows : 1) * d, sizeof(double));
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < L->nclus; ++c) {
    const int m = L->m[c];
    const int64_t off = L->poff[c];
    double* A = L->W + off * d;
    for (int j = 0; j < m; ++j) memcpy(A + (int64_t)j * d, Y + (off + j) * ld, sizeof(double) * d);
    double* nrm = (double*)xcalloc(m + 1, sizeof(double));
    double* v = (double*)xcalloc(d + 1, sizeof(double));
    L->k[c] = cpqr_panel(A, m, d, eps, b->o->max_rank, L->perm + off, nrm, v, L->cert + 2 * c);
    free(nrm);
    free(v);
  }
  b->res->t_cpqr += wtime() - t0;
}

/* ID epilogue (lines 221-224 / 250-253): X, skeletons */
static void commit(bld_t* b, int t) {
  double t0 = wtime();
  lvl_t* L = &b->L[t];
  const int d = b->d;
  L->roff = (int64_t*)xcalloc(L->nclus, sizeof(int64_t));
  L->xoff = (int64_t*)xcalloc(L->nclus, sizeof(int64_t));
  L->rtot = L->xtot = 0;
  for (int c = 0; c < L->nclus; ++c) {
    L->roff[c] = L->rtot;
    L->xoff[c] = L->xtot;
    L->rtot += L->k[c];
    L->xtot += (int64_t)L->m[c] * L->k[c];
  }
  L->X = (double*)xcalloc(L->xtot, sizeof(double));
  L->skel = (int32_t*)xcalloc(L->rtot, sizeof(int32_t));
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < L->nclus; ++c) {
    const int m = L->m[c], k = L->k[c];
    const int64_t off = L->poff[c];
    const double* A = L->W + off * d;     /* R(i, j) = A[j * d + i] */
    const int32_t* perm = L->perm + off;
    double* X = L->X + L->xoff[c];
    for (int i = 0; i < k; ++i) {
      X[(int64_t)perm[i] * k + i] = 1.0;
      const int64_t pi = off + perm[i];
      L->skel[L->roff[c] + i] = t == b->Dl ? (int32_t)pi : b->L[t + 1].skel[pi];
    }
    double* Tc = (double*)xcalloc(k + 1, sizeof(double));
    for (int cc = 0; cc < m - k; ++cc) {
      for (int i = k - 1; i >= 0; --i) {
        double s = A[(int64_t)(k + cc) * d + i];
        for (int j = i + 1; j < k; ++j) s = fma(-A[(int64_t)j * d + i], Tc[j], s);
        Tc[i] = s / A[(int64_t)i * d + i];
      }
      double* row = X + (int64_t)perm[k + cc] * k;
      for (int i = 0; i < k; ++i) row[i] = Tc[i];
    }
    free(Tc);
  }
  b->res->t_id += wtime() - t0;
}

/* shrink + project of committed depth u, columns [0, nc): source panel (depth u) -> destination
 * (rows = skeleton rows of depth u in roff order) */
static void shrink(bld_t* b, int u, const double* Ys, const double* Os, int64_t lds, double* Yd, double* Od,
                   int64_t ldd, int nc) {
  double t0 = wtime();
  const lvl_t* L = &b->L[u];
#pragma omp parallel for schedule(dynamic, 4)
  for (int c = 0; c < L->nclus; ++c) {
    const int m = L->m[c], k = L->k[c];
    const int64_t off = L->poff[c];
    const int32_t* perm = L->perm + off;
    const double* X = L->X + L->xoff[c];
    for (int i = 0; i < k; ++i) {
      const int64_t src = off + perm[i];
      double* yd = Yd + (L->roff[c] + i) * ldd;
      double* od = Od + (L->roff[c] + i) * ldd;
      for (int j = 0; j < nc; ++j) {
        yd[j] = Ys[src * lds + j];
        double acc = Os[src * lds + j];
        for (int cc = 0; cc < m - k; ++cc)
          acc = fma(X[(int64_t)perm[k + cc] * k + i], Os[(off + perm[k + cc]) * lds + j], acc);
        od[j] = acc;
      }
    }
  }
  b->res->t_id += wtime() - t0;
}

/* line 212 / 258: unique blocks (rows I_s / I~_s, columns I_b / I~_b) */
static void gen_D(bld_t* b) {
  double t0 = wtime();
  const int Dl = b->Dl;
  b->nu_near = unique_pairs(b->T->near_ptr, b->T->near_idx, 1 << Dl, 0, &b->un_s, &b->un_b);
  b->D_off = (int64_t*)xcalloc(b->nu_near + 1, sizeof(int64_t));
  for (int64_t q = 0; q < b->nu_near; ++q)
    b->D_off[q + 1] = b->D_off[q] + (endd(b, Dl, b->un_s[q]) - beg(b, Dl, b->un_s[q])) *
                                        (endd(b, Dl, b->un_b[q]) - beg(b, Dl, b->un_b[q]));
  b->D = (double*)xcalloc(b->D_off[b->nu_near], sizeof(double));
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t q = 0; q < b->nu_near; ++q) {
    const int64_t s0 = beg(b, Dl, b->un_s[q]), s1 = endd(b, Dl, b->un_s[q]);
    const int64_t b0 = beg(b, Dl, b->un_b[q]), b1 = endd(b, Dl, b->un_b[q]);
    double* out = b->D + b->D_off[q];
    for (int64_t i = s0; i < s1; ++i)
      for (int64_t j = b0; j < b1; ++j) out[(i - s0) * (b1 - b0) + (j - b0)] = kval(&b->K, i, j);
  }
  b->res->t_gen += wtime() - t0;
}

static void gen_B(bld_t* b, int t) {
  double t0 = wtime();
  const lvl_t* L = &b->L[t];
  const int64_t nu = b->nu_far[t];
  b->B_off[t] = (int64_t*)xcalloc(nu + 1, sizeof(int64_t));
  for (int64_t q = 0; q < nu; ++q)
    b->B_off[t][q + 1] = b->B_off[t][q] + (int64_t)L->k[b->uf_s[t][q]] * L->k[b->uf_b[t][q]];
  b->B[t] = (double*)xcalloc(b->B_off[t][nu], sizeof(double));
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t q = 0; q < nu; ++q) {
    const int s = (int)b->uf_s[t][q], c = (int)b->uf_b[t][q];
    const int ks = L->k[s], kc = L->k[c];
    double* out = b->B[t] + b->B_off[t][q];
    for (int i = 0; i < ks; ++i)
      for (int j = 0; j < kc; ++j)
        out[(int64_t)i * kc + j] = kval(&b->K, L->skel[L->roff[s] + i], L->skel[L->roff[c] + j]);
  }
  b->res->t_gen += wtime() - t0;
}

/* updateSamples (L216-217, L246-247, L386): b new stream columns swept up through the committed
 * depths Dl..t+1 and appended (columns [d, d+bk)) to the panel of depth t */
static void update_samples(bld_t* b, int t, panel_t* cur, int bk) {
  const int c0 = b->d;
  panel_grow(cur, b->d + bk, b->d);
  if (t == b->Dl) {
    draw(b, cur->Y + c0, cur->O + c0, cur->ld, c0, bk);
    bsr(b, b->Dl, cur->Y + c0, cur->O + c0, cur->ld, bk);
    return;
  }
  panel_t src;
  panel_alloc(&src, b->n, bk);
  draw(b, src.Y, src.O, bk, c0, bk);
  bsr(b, b->Dl, src.Y, src.O, bk, bk);
  for (int u = b->Dl; u > t; --u) {
    if (u - 1 == t) {
      shrink(b, u, src.Y, src.O, src.ld, cur->Y + c0, cur->O + c0, cur->ld, bk);
      bsr(b, t, cur->Y + c0, cur->O + c0, cur->ld, bk);
    } else {
      panel_t dst;
      panel_alloc(&dst, b->L[u].rtot, bk);
      shrink(b, u, src.Y, src.O, src.ld, dst.Y, dst.O, dst.ld, bk);
      bsr(b, u - 1, dst.Y, dst.O, dst.ld, bk);
      panel_free(&src);
      src = dst;
    }
  }
  panel_free(&src);
}

/* Algorithm 1.  Returns the result (caller frees with h2o_free); status < 0 on failure. */
h2o_result* h2o_build(const h2o_tree* T, int32_t kind, double param, double tol, const h2o_opts* o) {
  h2o_result* res = (h2o_result*)xcalloc(1, sizeof(h2o_result));
  res->failed_depth = -1;
  if (!T || !o || T->leaf_depth < 0 || T->leaf_depth >= H2O_MAXD || o->d_init < 1 || o->d_max < o->d_init ||
      o->d_blk < 1) {
    res->status = -1;
    return res;
  }
#ifdef _OPENMP
  if (o->threads > 0) omp_set_num_threads(o->threads);
#endif
  const double t_start = wtime();
  bld_t B;
  memset(&B, 0, sizeof B);
  bld_t* b = &B;
  b->T = T;
  b->K.kind = kind;
  b->K.param = param;
  b->K.l2 = param * param;
  b->K.pts = T->pts;
  b->K.dense = o->dense;
  b->K.ld = o->ld_dense;
  if (kind == H2O_K_TABLE && !o->dense) {
    res->status = -1;
    return res;
  }
  b->o = o;
  b->tol = tol;
  b->n = T->n;
  b->res = res;
  const int Dl = b->Dl = T->leaf_depth;
  int top = Dl;
  for (int t = 0; t <= Dl; ++t)
    if (T->far_ptr[t] && T->far_ptr[t][1 << t] > 0) {
      top = t;
      break;
    }
  b->top = top;
  res->top = top;
  res->leaf_depth = Dl;
  for (int t = top; t <= Dl; ++t) {
    if (T->far_ptr[t]) b->nu_far[t] = unique_pairs(T->far_ptr[t], T->far_idx[t], 1 << t, 1, &b->uf_s[t], &b->uf_b[t]);
    else b->uf_s[t] = b->uf_b[t] = NULL;
  }
  int d = b->d = o->d_init < o->d_max ? o->d_init : o->d_max;
  panel_t cur;
  panel_alloc(&cur, b->n, d);
  draw(b, cur.Y, cur.O, cur.ld, 0, d);                 /* line 1 */
  gen_D(b);                                            /* line 212 */
  setup_level(b, Dl);
  bsr(b, Dl, cur.Y, cur.O, cur.ld, d);                 /* line 213 */
  double eps = 0.0;
  for (int t = Dl; t >= top; --t) {
    if (t < Dl) {
      setup_level(b, t);
      bsr(b, t, cur.Y, cur.O, cur.ld, d);              /* lines 240-243 */
    }
    lvl_t* L = &b->L[t];
    int rounds = 0;
    for (;;) {
      eps = eps_now(b, t);
      cpqr_level(b, t, cur.Y, cur.ld, eps);
      ++rounds;
      if (!o->adaptive) break;
      const int pos = o->tol_rule == 0 ? o->p_os : 0;
      int conv = 1;
      for (int c = 0; c < L->nclus && conv; ++c) conv = (L->m[c] <= d) || (L->k[c] <= d - 1 - pos);
      if (conv) break;
      if (d + o->d_blk > o->d_max) {
        res->status = -6;
        res->failed_depth = t;
        goto out;
      }
      update_samples(b, t, &cur, o->d_blk);
      d = b->d = d + o->d_blk;
      if (b->table_short) {
        res->status = -2;
        res->failed_depth = t;
        goto out;
      }
    }
    res->rounds[t] = rounds;
    commit(b, t);                                      /* lines 221-224 / 250-253 */
    panel_t next;
    memset(&next, 0, sizeof next);
    if (t > top) {
      panel_alloc(&next, L->rtot, d);
      shrink(b, t, cur.Y, cur.O, cur.ld, next.Y, next.O, next.ld, d);
    }
    gen_B(b, t);                                       /* line 258 */
    panel_free(&cur);
    cur = next;
  }
out:
  panel_free(&cur);
  res->samples = b->d;
  res->eps = eps;
  if (res->status == 0) {
    for (int t = top; t <= Dl; ++t) {
      lvl_t* L = &b->L[t];
      res->rank[t] = L->k;
      L->k = NULL;
      res->skel[t] = L->skel;
      res->nskel[t] = L->rtot;
      L->skel = NULL;
      res->basis[t] = L->X;
      res->nbasis[t] = L->xtot;
      L->X = NULL;
      res->cert[t] = L->cert;
      L->cert = NULL;
      res->B[t] = b->B[t];
      res->nB[t] = b->B_off[t] ? b->B_off[t][b->nu_far[t]] : 0;
      b->B[t] = NULL;
    }
    res->D = b->D;
    res->nD = b->D_off[b->nu_near];
    b->D = NULL;
  }
  for (int t = 0; t < H2O_MAXD; ++t) {
    lvl_t* L = &b->L[t];
    free(L->m);
    free(L->k);
    free(L->poff);
    free(L->roff);
    free(L->xoff);
    free(L->perm);
    free(L->W);
    free(L->X);
    free(L->skel);
    free(L->cert);
    free(b->uf_s[t]);
    free(b->uf_b[t]);
    free(b->B_off[t]);
    free(b->B[t]);
  }
  free(b->un_s);
  free(b->un_b);
  free(b->D_off);
  free(b->D);
  res->t_total = wtime() - t_start;
  return res;
}

void h2o_free(h2o_result* r) {
  if (!r) return;
  for (int t = 0; t < H2O_MAXD; ++t) {
    free(r->rank[t]);
    free(r->skel[t]);
    free(r->basis[t]);
    free(r->cert[t]);
    free(r->B[t]);
  }
  free(r->D);
  free(r);
}

int h2o_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
