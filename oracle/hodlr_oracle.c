/*
 * hodlr_oracle.c -- plain single-threaded CPU oracle (TEST INFRASTRUCTURE).
 *
 * See hodlr_oracle.h for the scope statement and the step -> paper map.
 * Every loop here is the definition written out: no blocking, no fusion,
 * no reordering beyond what the paper's algorithm states.  Ambiguities are
 * resolved by the readings listed in DESIGN.md section 3 ("R1".."R15").
 * Compile: gcc -O2 -ffp-contract=off -fPIC -shared (no BLAS, no OpenMP).
 *
 * -DORACLE_TWIN builds the "oracle twin" of SURVEY.md 8(c) Q15 (liboracle_twin.so): the same algorithm with a
 * different backward-stable factorization of every small dense system -- leaf blocks by LU with partial pivoting
 * instead of Cholesky (O5'), coupling systems S_c by Householder QR instead of LU (O7').  Same ACA, same tree,
 * same panel and sweep.  The twin-vs-oracle difference of a solve is the FP64 conditioning floor of that
 * problem (two correct implementations with the same pivots), which sets the parity gate of the badly
 * conditioned config-4 settings: max(1e-9, 10 floor) (R15).
 */
#include "hodlr_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>

static __thread char g_err[512];
static int fail(int code, const char *fmt, ...) {
  va_list ap; va_start(ap, fmt); vsnprintf(g_err, sizeof g_err, fmt, ap); va_end(ap);
  return code;
}
const char *oracle_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* O3: covariance functions, Table I, closed forms  */
/* for nu = 3/2, 5/2 with r -> r/ell and amplitude a^2 (R13). */
/* ------------------------------------------------------------------ */
double oracle_kernel(int kernel, const double *theta, double d) {
  double a = theta[0], ell = theta[1];
  if (kernel == ORACLE_SE) {                      /* a^2 exp(-d^2 / (2 ell^2)) */
    double t = d * d / (2.0 * ell * ell);
    return a * a * exp(-t);
  }
  if (kernel == ORACLE_EXP) return a * a * exp(-fabs(d) / ell);              /* Table I / IV: a^2 e^{-|d|/ell} */
  if (kernel == ORACLE_IMQ) return a * a / sqrt(1.0 + (d / ell) * (d / ell)); /* Table V */
  if (kernel == ORACLE_RQ) return a * a * pow(1.0 + (d / ell) * (d / ell), -theta[2]);   /* Table I */
  /* NEXT-2, not positive definite (R20): multiquadric a^2 sqrt(1 + (d/ell)^2) (sec. 5.2 eq., Table III) and
   * biharmonic / thin-plate a^2 (d/ell)^2 log|d/ell|, 0 at d = 0 (sec. 5.4, Table VI) */
  if (kernel == ORACLE_MQ) return a * a * sqrt(1.0 + (d / ell) * (d / ell));
  if (kernel == ORACLE_BIHARM) {
    double q = fabs(d) / ell;
    return q == 0.0 ? 0.0 : a * a * (q * q) * log(q);
  }
  double r = fabs(d);
  if (kernel == ORACLE_MATERN32) {                /* a^2 (1 + s) e^{-s}, s = sqrt(3) r / ell */
    double s = sqrt(3.0) * r / ell;
    return a * a * (1.0 + s) * exp(-s);
  }
  /* ORACLE_MATERN52: a^2 (1 + s + s^2/3) e^{-s}, s = sqrt(5) r / ell */
  double s = sqrt(5.0) * r / ell;
  return a * a * (1.0 + s + s * s / 3.0) * exp(-s);
}

/* O3 for d >= 2 (NEXT-3): the same Table I functions of the Euclidean distance r = |x_i - x_j|, given its square
 * r2 = sum_k (x_ik - x_jk)^2 (summed over k in order): SE uses r2 directly, the others r = sqrt(r2) in place of |d|.
 * (1-D points use oracle_kernel(d) -- bit for bit the same definition as before.) */
double oracle_kernel_r2(int kernel, const double *theta, double r2) {
  double a = theta[0], ell = theta[1];
  if (kernel == ORACLE_SE) return a * a * exp(-(r2 / (2.0 * ell * ell)));
  return oracle_kernel(kernel, theta, sqrt(r2));
}

/* squared distance of points p, q (dim coordinates each), summed in coordinate order */
static double dist2(const double *p, const double *q, int dim) {
  double r2 = 0.0;
  for (int k = 0; k < dim; k++) { double d = p[k] - q[k]; r2 += d * d; }
  return r2;
}

/* ------------------------------------------------------------------ */
/* O4: adaptive cross approximation (partial-pivoted LU). */
/* Entry source is a callback so the same routine serves kernel blocks and  */
/* explicit dense test blocks.                                               */
/* ------------------------------------------------------------------ */
typedef double (*entry_fn)(const void *ctx, int64_t i, int64_t j);

typedef struct { int64_t m1, m2; int r, capcols; double **U, **V; } lowrank;

static void lowrank_free(lowrank *B) {
  for (int l = 0; l < B->r; l++) { free(B->U[l]); free(B->V[l]); }
  free(B->U); free(B->V); memset(B, 0, sizeof *B);
}

static double dot(const double *a, const double *b, int64_t m) {
  double s = 0.0;
  for (int64_t i = 0; i < m; i++) s += a[i] * b[i];
  return s;
}

/* Returns ORACLE_OK or ORACLE_ERANKCAP/ENOMEM; B->r is the rank. */
/* rowkey (may be NULL): coordinates of the rows (sorted).  Rows with a key equal to a used pivot row
 * have identical residual rows and are treated as used as well (R2). */
/* (d-dimensional points: rowkey holds m1 points of `dim` coordinates; "equal" = every coordinate equal -- the
 * kd ordering keeps identical points adjacent, as the 1-D sort does) */
static int same_point(const double *key, int dim, int64_t a, int64_t b) {
  for (int k = 0; k < dim; k++) if (key[a * dim + k] != key[b * dim + k]) return 0;
  return 1;
}
static void mark_row_run(char *used_r, const double *rowkey, int dim, int64_t m1, int64_t ik) {
  used_r[ik] = 1;
  if (!rowkey) return;
  for (int64_t i = ik - 1; i >= 0 && same_point(rowkey, dim, i, ik); i--) used_r[i] = 1;
  for (int64_t i = ik + 1; i < m1 && same_point(rowkey, dim, i, ik); i++) used_r[i] = 1;
}

#ifdef ORACLE_TRACE_ACA
static int g_trace_aca = 0;     /* diagnostic build only: per-step stop statistics of block ORACLE_TRACE_ACA */
#endif
static int aca(entry_fn f, const void *ctx, int64_t m1, int64_t m2, double eps, int cap, lowrank *B,
               const double *rowkey, int dim) {
  memset(B, 0, sizeof *B);
  B->m1 = m1; B->m2 = m2;
  int64_t mn = m1 < m2 ? m1 : m2;
  if (cap <= 0 || cap > mn) cap = (int)mn;
  char *used_r = calloc((size_t)m1, 1), *used_c = calloc((size_t)m2, 1);
  double *vt = malloc(sizeof(double) * (size_t)m2);
  if (!used_r || !used_c || !vt) { free(used_r); free(used_c); free(vt); return fail(ORACLE_ENOMEM, "aca: out of memory"); }
  int64_t ik = m1 - 1;               /* R2: start at the last row of c1 (nearest c2) */
  double S2 = 0.0;
  int k = 0, status = ORACLE_OK;
  for (;;) {
    /* step 1: residual row v~ = A[ik,:] - sum_{l<k} U[ik,l] V[:,l]  (l ascending) */
    for (int64_t j = 0; j < m2; j++) {
      double v = f(ctx, ik, j);
      for (int l = 0; l < k; l++) v -= B->U[l][ik] * B->V[l][j];
      vt[j] = v;
    }
    mark_row_run(used_r, rowkey, dim, m1, ik);
    /* step 2: jk = smallest unused column maximising |v~_j| */
    int64_t jk = -1; double best = -1.0;
    for (int64_t j = 0; j < m2; j++)
      if (!used_c[j] && fabs(vt[j]) > best) { best = fabs(vt[j]); jk = j; }
    if (jk < 0 || vt[jk] == 0.0) break;                 /* exactly-zero residual row: rank k */
    /* step 3: V[:,k] = v~ / v~_jk ; U[:,k] = A[:,jk] - sum_{l<k} V[jk,l] U[:,l] */
    if (k == B->capcols) {
      int nc = B->capcols ? 2 * B->capcols : 8;
      double **nu = realloc(B->U, sizeof(double *) * nc), **nv;
      if (!nu) { status = fail(ORACLE_ENOMEM, "aca: oom"); break; }
      B->U = nu;
      nv = realloc(B->V, sizeof(double *) * nc);
      if (!nv) { status = fail(ORACLE_ENOMEM, "aca: oom"); break; }
      B->V = nv; B->capcols = nc;
    }
    double *u = malloc(sizeof(double) * (size_t)m1), *v = malloc(sizeof(double) * (size_t)m2);
    if (!u || !v) { free(u); free(v); status = fail(ORACLE_ENOMEM, "aca: oom"); break; }
    double piv = vt[jk];
    for (int64_t j = 0; j < m2; j++) v[j] = vt[j] / piv;
    used_c[jk] = 1;
    for (int64_t i = 0; i < m1; i++) {
      double s = f(ctx, i, jk);
      for (int l = 0; l < k; l++) s -= B->V[l][jk] * B->U[l][i];
      u[i] = s;
    }
    /* step 4: ||S||^2 += 2 sum_{l<k} (u.U_l)(V_l.v) + ||u||^2 ||v||^2 */
    double cross = 0.0;
    for (int l = 0; l < k; l++) cross += dot(u, B->U[l], m1) * dot(B->V[l], v, m2);
    double nu2 = dot(u, u, m1), nv2 = dot(v, v, m2);
    S2 += 2.0 * cross + nu2 * nv2;
    B->U[k] = u; B->V[k] = v; k++; B->r = k;
    /* step 5: stop when ||u_k|| ||v_k|| <= eps ||S_k||_F (term kept, R1/R4) */
#ifdef ORACLE_TRACE_ACA
    if (g_trace_aca) fprintf(stderr, "[oracle aca] k=%d ik=%lld jk=%lld nu2=%.17g nv2=%.17g S2=%.17g ratio=%.17g\n", k,
                             (long long)ik, (long long)jk, nu2, nv2, S2, sqrt(nu2) * sqrt(nv2) / (eps * sqrt(fabs(S2))));
#endif
    if (sqrt(nu2) * sqrt(nv2) <= eps * sqrt(fabs(S2))) break;
    /* step 6 */
    if (k == mn) break;
    if (k == cap) { status = fail(ORACLE_ERANKCAP, "aca: rank cap %d reached without meeting eps", cap); break; }
    /* step 7: next row = smallest unused row maximising |U[:,k-1]| */
    int64_t inext = -1; best = -1.0;
    for (int64_t i = 0; i < m1; i++)
      if (!used_r[i] && fabs(u[i]) > best) { best = fabs(u[i]); inext = i; }
    if (inext < 0 || best == 0.0) break;
    ik = inext;
  }
  free(used_r); free(used_c); free(vt);
  return status;
}

typedef struct { const double *A; int64_t lda; } dense_ctx;
static double dense_entry(const void *c, int64_t i, int64_t j) {
  const dense_ctx *d = c; return d->A[j * d->lda + i];
}

int oracle_aca_dense(const double *A, int64_t m1, int64_t m2, int64_t lda, double eps,
                     int cap, double *U, double *V, int *rank) {
  if (m1 < 1 || m2 < 1 || lda < m1 || !(eps > 0.0 && eps < 1.0) || cap < 1)
    return fail(ORACLE_EINVAL, "aca_dense: bad arguments");
  dense_ctx ctx = { A, lda };
  lowrank B;
  int st = aca(dense_entry, &ctx, m1, m2, eps, cap, &B, NULL, 1);
  *rank = B.r;
  for (int l = 0; l < B.r; l++) {
    memcpy(U + (int64_t)l * m1, B.U[l], sizeof(double) * (size_t)m1);
    memcpy(V + (int64_t)l * m2, B.V[l], sizeof(double) * (size_t)m2);
  }
  lowrank_free(&B);
  return st;
}

/* ------------------------------------------------------------------ */
/* The handle                                                          */
/* ------------------------------------------------------------------ */
struct oracle_hodlr {
  int64_t n; int kern; double theta[3]; double s2; int leaf; double eps; int cap;
  int dim;                          /* coordinates per point (xs: n x dim, point-major, sorted order) */
  int leaf_lu;                      /* leaves by LU with partial pivoting: the twin, or a kernel that is not SPD */
  int nonspd;                       /* kernel not positive definite: det C may be negative (signed log det) */
  int sign;                         /* sign of det C after factor */
  double *dsort;                    /* heteroscedastic: s2 + noise_i in sorted order (NULL: s2 everywhere) */
  int kappa; int64_t nnodes, ninternal, nleaves;
  double *xs; int64_t *perm;
  int64_t *lo, *hi;                 /* heap order: node (d,i) has id 2^d - 1 + i */
  lowrank *blk;                     /* ninternal blocks K[c1,c2] = U V^T */
  int *rdep; int64_t *coff; int64_t K; /* per-depth column width r_e and offset, e = 1..kappa */
  double *X, *Xh;                   /* n x K row-major: processed panel and its unprocessed copy */
  double **Lleaf;                   /* per leaf: m x m lower Cholesky factor (row-major) */
  double **Slu; int **Spiv;         /* per internal node: 2r x 2r LU (row-major) + pivots; twin: Q then R */
  int **Lpiv;                       /* twin: per-leaf LU pivots */
  double *leaf_ld, *node_ld;        /* log det partials */
  double logdet; int state;         /* 1 built, 2 factored, -1 failed */
  int fstatus;
};

typedef struct { const struct oracle_hodlr *h; int64_t r0, c0; } blk_ctx;
/* O3: k(xs_i, xs_j) of sorted points i, j: 1-D as a function of d = x_i - x_j, d-D of r2 = |x_i - x_j|^2 */
static double kval_sorted(const oracle_hodlr *h, int64_t i, int64_t j) {
  if (h->dim == 1) return oracle_kernel(h->kern, h->theta, h->xs[i] - h->xs[j]);
  return oracle_kernel_r2(h->kern, h->theta, dist2(h->xs + i * h->dim, h->xs + j * h->dim, h->dim));
}

static double kernel_entry(const void *c, int64_t i, int64_t j) {
  const blk_ctx *b = c;
  return kval_sorted(b->h, b->r0 + i, b->c0 + j);       /* off-diagonal: no noise term */
}

/* O3: C_ij = k(xs_i, xs_j) + sigma_i^2 [i = j], sorted indices; sigma_i^2 = s2 (+ noise_i). */
static double entry_C(const oracle_hodlr *h, int64_t i, int64_t j) {
  double v = kval_sorted(h, i, j);
  if (i == j) v += h->dsort ? h->dsort[i] : h->s2;
  return v;
}

/* O1: stable ascending argsort (equal keys keep their current relative order), merge sort; the key of index v is
 * key[v * stride] (stride = dim, key = one coordinate of point-major data). */
static void merge_sort_idx(int64_t *idx, int64_t *tmp, int64_t n, const double *key, int stride) {
  if (n < 2) return;
  int64_t h = n / 2;
  merge_sort_idx(idx, tmp, h, key, stride);
  merge_sort_idx(idx + h, tmp, n - h, key, stride);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) {
    if (key[idx[j] * stride] < key[idx[i] * stride]) tmp[k++] = idx[j++];   /* strict: equal keys keep left first */
    else tmp[k++] = idx[i++];
  }
  while (i < h) tmp[k++] = idx[i++];
  while (j < n) tmp[k++] = idx[j++];
  memcpy(idx, tmp, sizeof(int64_t) * (size_t)n);
}

void oracle_free(oracle_hodlr *h) {
  if (!h) return;
  free(h->xs); free(h->perm); free(h->lo); free(h->hi); free(h->dsort);
  if (h->blk) for (int64_t c = 0; c < h->ninternal; c++) lowrank_free(&h->blk[c]);
  free(h->blk); free(h->rdep); free(h->coff); free(h->X); free(h->Xh);
  if (h->Lleaf) for (int64_t l = 0; l < h->nleaves; l++) free(h->Lleaf[l]);
  free(h->Lleaf);
  if (h->Lpiv) for (int64_t l = 0; l < h->nleaves; l++) free(h->Lpiv[l]);
  free(h->Lpiv);
  if (h->Slu) for (int64_t c = 0; c < h->ninternal; c++) { free(h->Slu[c]); free(h->Spiv[c]); }
  free(h->Slu); free(h->Spiv); free(h->leaf_ld); free(h->node_ld);
  free(h);
}

int oracle_build(const double *x, int64_t n, int kernel, const double *theta, double sigma2,
                 int leaf, double eps, int rank_cap, oracle_hodlr **out) {
  return oracle_build_noise(x, n, kernel, theta, sigma2, NULL, leaf, eps, rank_cap, out);
}

int oracle_build_noise(const double *x, int64_t n, int kernel, const double *theta, double sigma2, const double *noise,
                       int leaf, double eps, int rank_cap, oracle_hodlr **out) {
  return oracle_build_nd(x, n, 1, kernel, theta, sigma2, noise, leaf, eps, rank_cap, out);
}

int oracle_build_nd(const double *x, int64_t n, int dim, int kernel, const double *theta, double sigma2,
                    const double *noise, int leaf, double eps, int rank_cap, oracle_hodlr **out) {
  *out = NULL;
  if (n < 1 || dim < 1 || dim > 64 || leaf < 1 || !(eps > 0.0 && eps < 1.0) || !(sigma2 >= 0.0) || !theta ||
      !(theta[1] > 0.0) || !(theta[0] >= 0.0) || kernel < 0 || kernel > 7 || (kernel == ORACLE_RQ && !(theta[2] > 0.0)) ||
      !isfinite(sigma2) ||
      !isfinite(theta[0]) || !isfinite(theta[1]))
    return fail(ORACLE_EINVAL, "build: invalid argument");
  for (int64_t i = 0; i < n * dim; i++)
    if (!isfinite(x[i])) return fail(ORACLE_EINVAL, "build: non-finite x[%lld]", (long long)i);
  if (noise)
    for (int64_t i = 0; i < n; i++)
      if (!isfinite(noise[i]) || noise[i] < 0.0) return fail(ORACLE_EINVAL, "build: bad noise[%lld]", (long long)i);
  oracle_hodlr *h = calloc(1, sizeof *h);
  if (!h) return fail(ORACLE_ENOMEM, "build: oom");
  h->n = n; h->dim = dim; h->kern = kernel; h->theta[0] = theta[0]; h->theta[1] = theta[1];
  h->nonspd = kernel == ORACLE_MQ || kernel == ORACLE_BIHARM;
#ifdef ORACLE_TWIN
  h->leaf_lu = 1;
#else
  h->leaf_lu = h->nonspd;
#endif
  h->theta[2] = kernel == ORACLE_RQ ? theta[2] : 0.0;
  h->s2 = sigma2; h->leaf = leaf; h->eps = eps; h->cap = rank_cap;
  /* O2: kappa = largest integer with leaf * 2^kappa <= n (0 if n <= leaf); count-median split, left = ceil(m/2) */
  int kappa = 0;
  while ((int64_t)leaf << (kappa + 1) <= n && kappa < 62) kappa++;
  h->kappa = kappa;
  h->nnodes = ((int64_t)1 << (kappa + 1)) - 1;
  h->ninternal = ((int64_t)1 << kappa) - 1;
  h->nleaves = (int64_t)1 << kappa;
  h->lo = malloc(sizeof(int64_t) * (size_t)h->nnodes);
  h->hi = malloc(sizeof(int64_t) * (size_t)h->nnodes);
  if (!h->lo || !h->hi) { oracle_free(h); return fail(ORACLE_ENOMEM, "build: oom"); }
  h->lo[0] = 0; h->hi[0] = n;
  for (int64_t c = 0; c < h->ninternal; c++) {       /* split: left gets ceil(m/2) */
    int64_t m = h->hi[c] - h->lo[c], half = (m + 1) / 2;
    h->lo[2 * c + 1] = h->lo[c]; h->hi[2 * c + 1] = h->lo[c] + half;
    h->lo[2 * c + 2] = h->lo[c] + half; h->hi[2 * c + 2] = h->hi[c];
  }
  /* O1: 1-D: one stable ascending sort.  d >= 2: the kd-tree ordering -- each node of depth
   * L < max(kappa, 1), top down, stably sorts its points by coordinate L mod d; the count-median split above then
   * halves it (R19).  For d = 1 this is the same order as the single sort. */
  double *key = malloc(sizeof(double) * (size_t)(n * dim));
  int64_t *tmp = malloc(sizeof(int64_t) * (size_t)n);
  h->perm = malloc(sizeof(int64_t) * (size_t)n);
  h->xs = malloc(sizeof(double) * (size_t)(n * dim));
  if (!key || !tmp || !h->perm || !h->xs) { free(key); free(tmp); oracle_free(h); return fail(ORACLE_ENOMEM, "build: oom"); }
  for (int64_t i = 0; i < n * dim; i++) key[i] = x[i] == 0.0 ? 0.0 : x[i];     /* -0.0 -> +0.0 */
  for (int64_t i = 0; i < n; i++) h->perm[i] = i;
  if (dim == 1) merge_sort_idx(h->perm, tmp, n, key, 1);
  else {
    int levels = kappa > 0 ? kappa : 1;
    for (int L = 0; L < levels; L++)
      for (int64_t c = ((int64_t)1 << L) - 1; c < ((int64_t)2 << L) - 1; c++)
        merge_sort_idx(h->perm + h->lo[c], tmp, h->hi[c] - h->lo[c], key + (L % dim), dim);
  }
  for (int64_t i = 0; i < n; i++)
    for (int k = 0; k < dim; k++) h->xs[i * dim + k] = key[h->perm[i] * dim + k];
  free(key); free(tmp);
  if (noise) {                                       /* sigma_i^2 = s2 + noise_i, carried with its point */
    h->dsort = malloc(sizeof(double) * (size_t)n);
    if (!h->dsort) { oracle_free(h); return fail(ORACLE_ENOMEM, "build: oom"); }
    for (int64_t i = 0; i < n; i++) h->dsort[i] = sigma2 + noise[h->perm[i]];
  }
  /* O4: compress K[c1, c2] of every internal node c */
  h->blk = calloc((size_t)(h->ninternal ? h->ninternal : 1), sizeof(lowrank));
  if (!h->blk) { oracle_free(h); return fail(ORACLE_ENOMEM, "build: oom"); }
  for (int64_t c = 0; c < h->ninternal; c++) {
    int64_t c1 = 2 * c + 1, c2 = 2 * c + 2;
    blk_ctx ctx = { h, h->lo[c1], h->lo[c2] };
#ifdef ORACLE_TRACE_ACA
    g_trace_aca = c == ORACLE_TRACE_ACA;
#endif
    int st = aca(kernel_entry, &ctx, h->hi[c1] - h->lo[c1], h->hi[c2] - h->lo[c2], eps, rank_cap, &h->blk[c],
                 h->xs + h->lo[c1] * dim, dim);
    if (st != ORACLE_OK) {
      int code = st;
      char msg[400]; snprintf(msg, sizeof msg, "%.360s", g_err);
      oracle_free(h);
      return fail(code, "build: node %lld: %s", (long long)c, msg);
    }
  }
  h->state = 1;
  *out = h;
  return ORACLE_OK;
}

static int depth_of(int64_t id) { int d = 0; while (id >= ((int64_t)2 << d) - 1) d++; return d; }

/* O5: unblocked Cholesky (Cholesky-Banachiewicz), A = L L^T, row-major m x m. */
__attribute__((unused)) static int cholesky(double *A, int64_t m) {
  for (int64_t j = 0; j < m; j++) {
    double s = A[j * m + j];
    for (int64_t k = 0; k < j; k++) s -= A[j * m + k] * A[j * m + k];
    if (!(s > 0.0)) return -1;                        /* non-positive pivot before sqrt */
    double ljj = sqrt(s);
    A[j * m + j] = ljj;
    for (int64_t i = j + 1; i < m; i++) {
      double t = A[i * m + j];
      for (int64_t k = 0; k < j; k++) t -= A[i * m + k] * A[j * m + k];
      A[i * m + j] = t / ljj;
    }
    for (int64_t i = 0; i < j; i++) A[i * m + j] = 0.0;
  }
  return 0;
}

/* Solve L L^T w = b in place; b has stride `st`. */
__attribute__((unused)) static void chol_solve(const double *L, int64_t m, double *b, int64_t st) {
  for (int64_t i = 0; i < m; i++) {
    double s = b[i * st];
    for (int64_t k = 0; k < i; k++) s -= L[i * m + k] * b[k * st];
    b[i * st] = s / L[i * m + i];
  }
  for (int64_t i = m - 1; i >= 0; i--) {
    double s = b[i * st];
    for (int64_t k = i + 1; k < m; k++) s -= L[k * m + i] * b[k * st];
    b[i * st] = s / L[i * m + i];
  }
}

/* LU with partial pivoting (row of max |.|, first index on ties), row-major q x q. */
static int lu_factor(double *S, int q, int *piv, double *logabs, int *sign) {
  int sg = 1; double la = 0.0;
  for (int k = 0; k < q; k++) {
    int p = k; double best = fabs(S[k * q + k]);
    for (int i = k + 1; i < q; i++) if (fabs(S[i * q + k]) > best) { best = fabs(S[i * q + k]); p = i; }
    piv[k] = p;
    if (p != k) { for (int j = 0; j < q; j++) { double t = S[k * q + j]; S[k * q + j] = S[p * q + j]; S[p * q + j] = t; } sg = -sg; }
    double ukk = S[k * q + k];
    if (ukk == 0.0) return -1;
    if (ukk < 0.0) sg = -sg;
    la += log(fabs(ukk));
    for (int i = k + 1; i < q; i++) {
      double lik = S[i * q + k] / ukk;
      S[i * q + k] = lik;
      for (int j = k + 1; j < q; j++) S[i * q + j] -= lik * S[k * q + j];
    }
  }
  *logabs = la; *sign = sg;
  return 0;
}

/* Solve (LU) t = b in place for one rhs with stride st. */
static void lu_solve(const double *S, int q, const int *piv, double *b, int64_t st) {
  for (int k = 0; k < q; k++) if (piv[k] != k) { double t = b[k * st]; b[k * st] = b[piv[k] * st]; b[piv[k] * st] = t; }
  for (int i = 0; i < q; i++) { double s = b[i * st]; for (int k = 0; k < i; k++) s -= S[i * q + k] * b[k * st]; b[i * st] = s; }
  for (int i = q - 1; i >= 0; i--) { double s = b[i * st]; for (int k = i + 1; k < q; k++) s -= S[i * q + k] * b[k * st]; b[i * st] = s / S[i * q + i]; }
}

#ifdef ORACLE_TWIN
/* Twin O7': Householder QR of the row-major q x q matrix S (overwritten), Q accumulated explicitly (row-major
 * q x q).  Column k: x = S[k:, k], alpha = -sign(x_0) ||x||, v = x - alpha e_1, H = I - 2 v v^T / v^T v applied
 * to S[k:, k:] from the left and to Q[:, k:] from the right.  det S = (-1)^(reflections) prod R_kk.
 * Returns -1 on a zero R_kk (singular). */
static int qr_factor(double *S, int q, double *Q, double *logabs, int *sign) {
  int sg = 1; double la = 0.0;
  double *v = malloc(sizeof(double) * (size_t)(q > 0 ? q : 1));
  if (!v) return -2;
  for (int i = 0; i < q; i++) for (int j = 0; j < q; j++) Q[i * q + j] = i == j ? 1.0 : 0.0;
  for (int k = 0; k < q; k++) {
    double nx = 0.0;
    for (int i = k; i < q; i++) nx += S[i * q + k] * S[i * q + k];
    nx = sqrt(nx);
    if (nx > 0.0) {
      double alpha = S[k * q + k] >= 0.0 ? -nx : nx;
      double vv = 0.0;
      for (int i = k; i < q; i++) v[i] = S[i * q + k];
      v[k] -= alpha;
      for (int i = k; i < q; i++) vv += v[i] * v[i];
      if (vv > 0.0) {
        for (int j = k; j < q; j++) {                  /* S[k:, j] -= 2 v (v . S[k:, j]) / vv */
          double d = 0.0;
          for (int i = k; i < q; i++) d += v[i] * S[i * q + j];
          d = 2.0 * d / vv;
          for (int i = k; i < q; i++) S[i * q + j] -= d * v[i];
        }
        for (int i = 0; i < q; i++) {                  /* Q[i, k:] -= 2 (Q[i, k:] . v) v / vv */
          double d = 0.0;
          for (int j = k; j < q; j++) d += Q[i * q + j] * v[j];
          d = 2.0 * d / vv;
          for (int j = k; j < q; j++) Q[i * q + j] -= d * v[j];
        }
        sg = -sg;                                     /* det H = -1 */
      }
    }
    double rkk = S[k * q + k];
    if (rkk == 0.0) { free(v); return -1; }
    if (rkk < 0.0) sg = -sg;
    la += log(fabs(rkk));
  }
  free(v);
  *logabs = la; *sign = sg;
  return 0;
}

/* t = R^{-1} Q^T b in place, one rhs with stride st (QR: Q row-major q x q, R upper of the row-major S). */
static void qr_solve(const double *Q, const double *R, int q, double *b, int64_t st) {
  double tmp[2048];
  double *w = q <= 2048 ? tmp : malloc(sizeof(double) * (size_t)q);
  for (int i = 0; i < q; i++) { double s = 0.0; for (int k = 0; k < q; k++) s += Q[k * q + i] * b[k * st]; w[i] = s; }
  for (int i = q - 1; i >= 0; i--) { double s = w[i]; for (int k = i + 1; k < q; k++) s -= R[i * q + k] * w[k]; w[i] = s / R[i * q + i]; }
  for (int i = 0; i < q; i++) b[i * st] = w[i];
  if (w != tmp) free(w);
}
#endif

/* Neumaier-compensated sum (R11). */
typedef struct { double s, c; } nsum;
static void nadd(nsum *a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
  a->s = t;
}

int oracle_factor(oracle_hodlr *h) {
  if (!h || h->state != 1) return fail(ORACLE_ESTATE, "factor: handle not in built state");
  int kappa = h->kappa; int64_t n = h->n;
  /* O6 panel layout: depth e = 1..kappa has width r_e = max rank of depth-(e-1) blocks. */
  h->rdep = calloc((size_t)kappa + 2, sizeof(int));
  h->coff = calloc((size_t)kappa + 2, sizeof(int64_t));
  for (int64_t c = 0; c < h->ninternal; c++) {
    int e = depth_of(c) + 1;
    if (h->blk[c].r > h->rdep[e]) h->rdep[e] = h->blk[c].r;
  }
  int64_t K = 0;
  for (int e = 1; e <= kappa; e++) { h->coff[e] = K; K += h->rdep[e]; }
  h->coff[kappa + 1] = K;
  h->K = K;
  h->X = calloc((size_t)(n * (K ? K : 1)), sizeof(double));
  h->Xh = calloc((size_t)(n * (K ? K : 1)), sizeof(double));
  h->Lleaf = calloc((size_t)h->nleaves, sizeof(double *));
  h->Lpiv = calloc((size_t)h->nleaves, sizeof(int *));
  h->Slu = calloc((size_t)(h->ninternal ? h->ninternal : 1), sizeof(double *));
  h->Spiv = calloc((size_t)(h->ninternal ? h->ninternal : 1), sizeof(int *));
  h->leaf_ld = calloc((size_t)h->nleaves, sizeof(double));
  h->node_ld = calloc((size_t)(h->ninternal ? h->ninternal : 1), sizeof(double));
  if (!h->X || !h->Xh || !h->Lleaf || !h->Lpiv || !h->Slu || !h->Spiv || !h->leaf_ld || !h->node_ld)
    return fail(ORACLE_ENOMEM, "factor: oom");
  /* X[a rows, cols(a)] = L_a for every non-root node a: U for a left child, V for a right child. */
  for (int64_t c = 0; c < h->ninternal; c++) {
    int e = depth_of(c) + 1; const lowrank *B = &h->blk[c];
    int64_t c1 = 2 * c + 1, c2 = 2 * c + 2;
    for (int l = 0; l < B->r; l++) {
      for (int64_t i = 0; i < B->m1; i++) h->X[(h->lo[c1] + i) * K + h->coff[e] + l] = B->U[l][i];
      for (int64_t j = 0; j < B->m2; j++) h->X[(h->lo[c2] + j) * K + h->coff[e] + l] = B->V[l][j];
    }
  }
  memcpy(h->Xh, h->X, sizeof(double) * (size_t)(n * K));
  h->state = -1;   /* until success */
  int sign = 1;    /* sign of det C (R20): product of the leaves' and coupling systems' determinant signs */
  /* O5 + O6: leaves -- Cholesky, log det partial, solve the panel rows (all ancestor columns). */
  for (int64_t l = 0; l < h->nleaves; l++) {
    int64_t id = h->ninternal + l, lo = h->lo[id], m = h->hi[id] - lo;
    double *A = malloc(sizeof(double) * (size_t)(m * m));
    if (!A) return fail(ORACLE_ENOMEM, "factor: oom");
    for (int64_t i = 0; i < m; i++) for (int64_t j = 0; j < m; j++) A[i * m + j] = entry_C(h, lo + i, lo + j);
    if (!h->leaf_lu) {
      if (cholesky(A, m) != 0) {
        free(A); h->logdet = -INFINITY; h->fstatus = ORACLE_ENOTPD;
        return fail(ORACLE_ENOTPD, "factor: leaf %lld not positive definite", (long long)l);
      }
      double s = 0.0;
      for (int64_t i = 0; i < m; i++) s += log(A[i * m + i]);
      h->leaf_ld[l] = 2.0 * s;
      h->Lleaf[l] = A;
      for (int64_t c = 0; c < K; c++) chol_solve(A, m, &h->X[lo * K + c], K);
    } else {
      /* O5' (twin, or a kernel that is not SPD): A = P^T L U with partial pivoting; log|det| = sum log |U_ii|, sign
       * from the pivots and U_ii: must be > 0 for a covariance, may be < 0 otherwise (zero = singular) */
      int *lp = malloc(sizeof(int) * (size_t)m);
      double la = 0.0; int sg = 1;
      if (!lp || lu_factor(A, (int)m, lp, &la, &sg) != 0 || sg == 0 || (sg < 0 && !h->nonspd)) {
        free(A); free(lp); h->logdet = -INFINITY; h->fstatus = ORACLE_ENOTPD;
        return fail(ORACLE_ENOTPD, "factor: leaf %lld singular or det <= 0", (long long)l);
      }
      h->leaf_ld[l] = la;
      if (sg < 0) sign = -sign;
      h->Lleaf[l] = A; h->Lpiv[l] = lp;
      for (int64_t c = 0; c < K; c++) lu_solve(A, (int)m, lp, &h->X[lo * K + c], K);
    }
  }
  /* O7: level sweep d = kappa-1 .. 0 (SMW on [[I, P],[Q, I]], equation_Low_Rank_Update). */
  for (int d = kappa - 1; d >= 0; d--) {
    int e = d + 1; int64_t cs = h->coff[e], Kd = h->coff[e];   /* J = columns of depths 1..d */
    for (int64_t i = 0; i < ((int64_t)1 << d); i++) {
      int64_t c = ((int64_t)1 << d) - 1 + i, c1 = 2 * c + 1, c2 = 2 * c + 2;
      int r = h->blk[c].r, q = 2 * r;
      int64_t lo1 = h->lo[c1], m1 = h->hi[c1] - lo1, lo2 = h->lo[c2], m2 = h->hi[c2] - lo2;
      double *S = calloc((size_t)(q > 0 ? 2 * q * q : 1), sizeof(double));   /* twin: Q in [q*q, 2 q*q) */
      int *piv = calloc((size_t)(q > 0 ? q : 1), sizeof(int));
      if (!S || !piv) return fail(ORACLE_ENOMEM, "factor: oom");
      for (int a = 0; a < q; a++) S[a * q + a] = 1.0;
      for (int a = 0; a < r; a++) for (int b = 0; b < r; b++) {
        double P = 0.0, Q = 0.0;    /* P = Xh[c2,cs]^T X[c2,cs], Q = Xh[c1,cs]^T X[c1,cs] */
        for (int64_t t = 0; t < m2; t++) P += h->Xh[(lo2 + t) * K + cs + a] * h->X[(lo2 + t) * K + cs + b];
        for (int64_t t = 0; t < m1; t++) Q += h->Xh[(lo1 + t) * K + cs + a] * h->X[(lo1 + t) * K + cs + b];
        S[a * q + r + b] = P;
        S[(r + a) * q + b] = Q;
      }
      double la = 0.0; int sg = 1;
#ifndef ORACLE_TWIN
      if (q > 0 && lu_factor(S, q, piv, &la, &sg) != 0) sg = 0;
#else
      if (q > 0 && qr_factor(S, q, S + q * q, &la, &sg) != 0) sg = 0;    /* O7' (twin) */
#endif
      h->Slu[c] = S; h->Spiv[c] = piv;
      if (sg == 0 || (sg < 0 && !h->nonspd)) {
        h->logdet = -INFINITY; h->fstatus = ORACLE_ENOTPD;
        return fail(ORACLE_ENOTPD, "factor: coupling system of node %lld singular or det <= 0", (long long)c);
      }
      if (sg < 0) sign = -sign;
      h->node_ld[c] = la;
      if (Kd == 0 || r == 0) continue;
      /* B = [Xh[c2,cs]^T X[c2,J]; Xh[c1,cs]^T X[c1,J]],  T = S^{-1} B */
      double *T = calloc((size_t)(q * Kd), sizeof(double));
      if (!T) return fail(ORACLE_ENOMEM, "factor: oom");
      for (int a = 0; a < r; a++) for (int64_t j = 0; j < Kd; j++) {
        double s2 = 0.0, s1 = 0.0;
        for (int64_t t = 0; t < m2; t++) s2 += h->Xh[(lo2 + t) * K + cs + a] * h->X[(lo2 + t) * K + j];
        for (int64_t t = 0; t < m1; t++) s1 += h->Xh[(lo1 + t) * K + cs + a] * h->X[(lo1 + t) * K + j];
        T[a * Kd + j] = s2;
        T[(r + a) * Kd + j] = s1;
      }
#ifndef ORACLE_TWIN
      for (int64_t j = 0; j < Kd; j++) lu_solve(S, q, piv, &T[j], Kd);
#else
      for (int64_t j = 0; j < Kd; j++) qr_solve(S + q * q, S, q, &T[j], Kd);
#endif
      /* X[c1,J] -= X[c1,cs] T_top ; X[c2,J] -= X[c2,cs] T_bot */
      for (int64_t t = 0; t < m1; t++) for (int64_t j = 0; j < Kd; j++) {
        double s = 0.0;
        for (int a = 0; a < r; a++) s += h->X[(lo1 + t) * K + cs + a] * T[a * Kd + j];
        h->X[(lo1 + t) * K + j] -= s;
      }
      for (int64_t t = 0; t < m2; t++) for (int64_t j = 0; j < Kd; j++) {
        double s = 0.0;
        for (int a = 0; a < r; a++) s += h->X[(lo2 + t) * K + cs + a] * T[(r + a) * Kd + j];
        h->X[(lo2 + t) * K + j] -= s;
      }
      free(T);
    }
  }
  /* O8: log det = leaves left to right, then nodes by depth kappa-1..0, left to right. */
  nsum acc = { 0.0, 0.0 };
  for (int64_t l = 0; l < h->nleaves; l++) nadd(&acc, h->leaf_ld[l]);
  for (int d = kappa - 1; d >= 0; d--)
    for (int64_t i = 0; i < ((int64_t)1 << d); i++) nadd(&acc, h->node_ld[((int64_t)1 << d) - 1 + i]);
  h->logdet = acc.s + acc.c;
  h->sign = sign;
  h->fstatus = ORACLE_OK;
  h->state = 2;
  return ORACLE_OK;
}

/* O8 for kernels that are not SPD: log |det C| and the sign of det C. */
int oracle_logdet_sign(oracle_hodlr *h, double *logabs, int *sign) {
  if (!h) return fail(ORACLE_EINVAL, "logdet: null handle");
  if (h->state == -1) { *logabs = -INFINITY; *sign = 0; return fail(ORACLE_ENOTPD, "logdet: factorization failed"); }
  if (h->state != 2) return fail(ORACLE_ESTATE, "logdet: not factored");
  *logabs = h->logdet; *sign = h->sign;
  return ORACLE_OK;
}

int oracle_logdet(oracle_hodlr *h, double *logdet) {
  if (!h) return fail(ORACLE_EINVAL, "logdet: null handle");
  if (h->state == -1) { *logdet = -INFINITY; return fail(ORACLE_ENOTPD, "logdet: factorization failed"); }
  if (h->state != 2) return fail(ORACLE_ESTATE, "logdet: not factored");
  *logdet = h->logdet;
  return ORACLE_OK;
}

/* O9: b = y[perm]; leaf solves; sweep with S^{-1}; x[perm[i]] = b[i]  (eq-fac). */
static void solve_sorted(const oracle_hodlr *h, double *b) {
  int64_t K = h->K;
  for (int64_t l = 0; l < h->nleaves; l++) {
    int64_t id = h->ninternal + l, lo = h->lo[id], m = h->hi[id] - lo;
    if (!h->leaf_lu) chol_solve(h->Lleaf[l], m, &b[lo], 1);
    else lu_solve(h->Lleaf[l], (int)m, h->Lpiv[l], &b[lo], 1);
  }
  for (int d = h->kappa - 1; d >= 0; d--) {
    int64_t cs = h->coff[d + 1];
    for (int64_t i = 0; i < ((int64_t)1 << d); i++) {
      int64_t c = ((int64_t)1 << d) - 1 + i, c1 = 2 * c + 1, c2 = 2 * c + 2;
      int r = h->blk[c].r, q = 2 * r;
      if (r == 0) continue;
      int64_t lo1 = h->lo[c1], m1 = h->hi[c1] - lo1, lo2 = h->lo[c2], m2 = h->hi[c2] - lo2;
      double t[2 * 1024];
      double *tt = q <= 2048 ? t : malloc(sizeof(double) * (size_t)q);
      for (int a = 0; a < r; a++) {
        double s2 = 0.0, s1 = 0.0;
        for (int64_t u = 0; u < m2; u++) s2 += h->Xh[(lo2 + u) * K + cs + a] * b[lo2 + u];
        for (int64_t u = 0; u < m1; u++) s1 += h->Xh[(lo1 + u) * K + cs + a] * b[lo1 + u];
        tt[a] = s2; tt[r + a] = s1;
      }
#ifndef ORACLE_TWIN
      lu_solve(h->Slu[c], q, h->Spiv[c], tt, 1);
#else
      qr_solve(h->Slu[c] + q * q, h->Slu[c], q, tt, 1);
#endif
      for (int64_t u = 0; u < m1; u++) { double s = 0.0; for (int a = 0; a < r; a++) s += h->X[(lo1 + u) * K + cs + a] * tt[a]; b[lo1 + u] -= s; }
      for (int64_t u = 0; u < m2; u++) { double s = 0.0; for (int a = 0; a < r; a++) s += h->X[(lo2 + u) * K + cs + a] * tt[r + a]; b[lo2 + u] -= s; }
      if (tt != t) free(tt);
    }
  }
}

int oracle_solve(oracle_hodlr *h, const double *y, double *x, int64_t nrhs, int64_t ld) {
  if (!h) return fail(ORACLE_EINVAL, "solve: null handle");
  if (h->state == -1) return fail(ORACLE_ENOTPD, "solve: factorization failed");
  if (h->state != 2) return fail(ORACLE_ESTATE, "solve: not factored");
  if (nrhs < 1 || ld < h->n) return fail(ORACLE_EINVAL, "solve: bad nrhs/ld");
  int64_t n = h->n;
  for (int64_t j = 0; j < nrhs; j++)
    for (int64_t i = 0; i < n; i++) if (!isfinite(y[j * ld + i])) return fail(ORACLE_EINVAL, "solve: non-finite y");
  double *b = malloc(sizeof(double) * (size_t)n);
  if (!b) return fail(ORACLE_ENOMEM, "solve: oom");
  for (int64_t j = 0; j < nrhs; j++) {
    for (int64_t i = 0; i < n; i++) b[i] = y[j * ld + h->perm[i]];
    solve_sorted(h, b);
    for (int64_t i = 0; i < n; i++) x[j * ld + h->perm[i]] = b[i];
  }
  free(b);
  return ORACLE_OK;
}

int oracle_gp_loglik(oracle_hodlr *h, const double *y, double *out) {
  if (!h) return fail(ORACLE_EINVAL, "loglik: null handle");
  if (h->nonspd) return fail(ORACLE_EINVAL, "loglik: the kernel is not positive definite (not a covariance)");
  if (h->state == -1) { *out = -INFINITY; return fail(ORACLE_ENOTPD, "loglik: factorization failed"); }
  if (h->state != 2) return fail(ORACLE_ESTATE, "loglik: not factored");
  int64_t n = h->n;
  double *x = malloc(sizeof(double) * (size_t)n);
  if (!x) return fail(ORACLE_ENOMEM, "loglik: oom");
  int st = oracle_solve(h, y, x, 1, n);
  if (st != ORACLE_OK) { free(x); return st; }
  nsum acc = { 0.0, 0.0 };
  for (int64_t i = 0; i < n; i++) nadd(&acc, y[i] * x[i]);
  free(x);
  *out = -0.5 * (acc.s + acc.c) - 0.5 * h->logdet - 0.5 * (double)n * log(2.0 * M_PI);
  return ORACLE_OK;
}

int oracle_apply(oracle_hodlr *h, const double *v, double *out) {
  if (!h || h->state == 0) return fail(ORACLE_ESTATE, "apply: not built");
  int64_t n = h->n;
  double *vs = malloc(sizeof(double) * (size_t)n), *ys = calloc((size_t)n, sizeof(double));
  if (!vs || !ys) { free(vs); free(ys); return fail(ORACLE_ENOMEM, "apply: oom"); }
  for (int64_t i = 0; i < n; i++) vs[i] = v[h->perm[i]];
  for (int64_t l = 0; l < h->nleaves; l++) {
    int64_t id = h->ninternal + l, lo = h->lo[id], hi = h->hi[id];
    for (int64_t i = lo; i < hi; i++) { double s = 0.0; for (int64_t j = lo; j < hi; j++) s += entry_C(h, i, j) * vs[j]; ys[i] += s; }
  }
  for (int64_t c = 0; c < h->ninternal; c++) {
    const lowrank *B = &h->blk[c];
    int64_t lo1 = h->lo[2 * c + 1], lo2 = h->lo[2 * c + 2];
    for (int l = 0; l < B->r; l++) {
      double a = 0.0, b = 0.0;
      for (int64_t j = 0; j < B->m2; j++) a += B->V[l][j] * vs[lo2 + j];
      for (int64_t i = 0; i < B->m1; i++) b += B->U[l][i] * vs[lo1 + i];
      for (int64_t i = 0; i < B->m1; i++) ys[lo1 + i] += B->U[l][i] * a;
      for (int64_t j = 0; j < B->m2; j++) ys[lo2 + j] += B->V[l][j] * b;
    }
  }
  for (int64_t i = 0; i < n; i++) out[h->perm[i]] = ys[i];
  free(vs); free(ys);
  return ORACLE_OK;
}

/* Residual rows of a solution: out[k] = sum_j C_{r_k j} x_j - y_{r_k} for original row indices r_k, C assembled
 * entry by entry (O3), original order; plain sequential loops.  Used by tests and the golden-file script. */
int oracle_residual_rows(oracle_hodlr *h, const double *x, const double *y, const int64_t *rows, int64_t nr,
                         double *out) {
  if (!h || h->state == 0) return fail(ORACLE_ESTATE, "residual_rows: not built");
  int64_t n = h->n;
  int64_t *inv = malloc(sizeof(int64_t) * (size_t)n);
  if (!inv) return fail(ORACLE_ENOMEM, "residual_rows: oom");
  for (int64_t i = 0; i < n; i++) inv[h->perm[i]] = i;
  for (int64_t k = 0; k < nr; k++) {
    if (rows[k] < 0 || rows[k] >= n) { free(inv); return fail(ORACLE_EINVAL, "residual_rows: bad row"); }
    int64_t i = inv[rows[k]];
    double s = 0.0;
    for (int64_t j = 0; j < n; j++) s += entry_C(h, i, j) * x[h->perm[j]];
    out[k] = s - y[rows[k]];
  }
  free(inv);
  return ORACLE_OK;
}

int oracle_kappa(oracle_hodlr *h) { return h ? h->kappa : -1; }
int64_t oracle_num_nodes(oracle_hodlr *h) { return h ? h->nnodes : -1; }
int oracle_get_perm(oracle_hodlr *h, int64_t *perm) { memcpy(perm, h->perm, sizeof(int64_t) * (size_t)h->n); return 0; }
int oracle_get_sorted(oracle_hodlr *h, double *xs) { memcpy(xs, h->xs, sizeof(double) * (size_t)(h->n * h->dim)); return 0; }
int oracle_dim(oracle_hodlr *h) { return h ? h->dim : -1; }
int oracle_get_tree(oracle_hodlr *h, int64_t *lo, int64_t *hi) {
  memcpy(lo, h->lo, sizeof(int64_t) * (size_t)h->nnodes); memcpy(hi, h->hi, sizeof(int64_t) * (size_t)h->nnodes); return 0;
}
int oracle_get_ranks(oracle_hodlr *h, int32_t *ranks) {
  for (int64_t c = 0; c < h->ninternal; c++) ranks[c] = h->blk[c].r;
  return 0;
}
int oracle_get_factors(oracle_hodlr *h, int64_t node, double *U, double *V) {
  if (node < 0 || node >= h->ninternal) return fail(ORACLE_EINVAL, "get_factors: bad node");
  const lowrank *B = &h->blk[node];
  for (int l = 0; l < B->r; l++) {
    memcpy(U + (int64_t)l * B->m1, B->U[l], sizeof(double) * (size_t)B->m1);
    memcpy(V + (int64_t)l * B->m2, B->V[l], sizeof(double) * (size_t)B->m2);
  }
  return 0;
}
int oracle_get_logdet_parts(oracle_hodlr *h, double *leaf_parts, double *node_parts) {
  if (h->state != 2) return fail(ORACLE_ESTATE, "logdet parts: not factored");
  memcpy(leaf_parts, h->leaf_ld, sizeof(double) * (size_t)h->nleaves);
  if (h->ninternal) memcpy(node_parts, h->node_ld, sizeof(double) * (size_t)h->ninternal);
  return 0;
}

/* ------------------------------------------------------------------ */
/* O11: dense checker -- an independent code path (own loops).         */
/* ------------------------------------------------------------------ */
int oracle_dense(const double *x, int64_t n, int kernel, const double *theta, double sigma2,
                 const double *y, double *logdet, double *xout) {
  return oracle_dense_noise(x, n, kernel, theta, sigma2, NULL, y, logdet, xout);
}

int oracle_dense_noise(const double *x, int64_t n, int kernel, const double *theta, double sigma2, const double *noise,
                       const double *y, double *logdet, double *xout) {
  return oracle_dense_nd(x, n, 1, kernel, theta, sigma2, noise, y, logdet, xout);
}

int oracle_dense_nd(const double *x, int64_t n, int dim, int kernel, const double *theta, double sigma2,
                    const double *noise, const double *y, double *logdet, double *xout) {
  if (n < 1 || n > 8192 || dim < 1) return fail(ORACLE_EINVAL, "dense: n out of range");
  double *C = malloc(sizeof(double) * (size_t)(n * n));
  if (!C) return fail(ORACLE_ENOMEM, "dense: oom");
  for (int64_t i = 0; i < n; i++)
    for (int64_t j = 0; j < n; j++) {
      double v;
      if (dim == 1) {
        double xi = x[i] == 0.0 ? 0.0 : x[i], xj = x[j] == 0.0 ? 0.0 : x[j];
        v = oracle_kernel(kernel, theta, xi - xj);
      } else {
        double r2 = 0.0;                               /* (x_i - x_j) . (x_i - x_j), coordinates in order */
        for (int k = 0; k < dim; k++) { double d = x[i * dim + k] - x[j * dim + k]; r2 += d * d; }
        v = oracle_kernel_r2(kernel, theta, r2);
      }
      C[i * n + j] = v + (i == j ? (noise ? sigma2 + noise[i] : sigma2) : 0.0);
    }
  /* right-looking (outer-product) Cholesky on the upper triangle, C = U^T U (U = L^T, row k of U = column k of
   * L): after row k is scaled, its rank-1 update is applied to the whole trailing upper triangle at once -- a
   * different operation order from O5's left-looking dot products, so the two agree only to rounding (the
   * independent LAPACK check is numpy's, in the pins) */
  for (int64_t k = 0; k < n; k++) {
    double d = C[k * n + k];
    if (!(d > 0.0)) { free(C); *logdet = -INFINITY; return fail(ORACLE_ENOTPD, "dense: not PD at %lld", (long long)k); }
    double ukk = sqrt(d);
    C[k * n + k] = ukk;
    for (int64_t j = k + 1; j < n; j++) C[k * n + j] /= ukk;
    for (int64_t i = k + 1; i < n; i++) {
      double uki = C[k * n + i];
      for (int64_t j = i; j < n; j++) C[i * n + j] -= uki * C[k * n + j];
    }
  }
  nsum acc = { 0.0, 0.0 };
  for (int64_t i = 0; i < n; i++) nadd(&acc, 2.0 * log(C[i * n + i]));
  *logdet = acc.s + acc.c;
  if (y && xout) {
    for (int64_t i = 0; i < n; i++) xout[i] = y[i];
    /* U^T z = y (L = U^T), then U x = z */
    for (int64_t i = 0; i < n; i++) { double s = xout[i]; for (int64_t k = 0; k < i; k++) s -= C[k * n + i] * xout[k]; xout[i] = s / C[i * n + i]; }
    for (int64_t i = n - 1; i >= 0; i--) { double s = xout[i]; for (int64_t k = i + 1; k < n; k++) s -= C[i * n + k] * xout[k]; xout[i] = s / C[i * n + i]; }
  }
  free(C);
  return ORACLE_OK;
}
