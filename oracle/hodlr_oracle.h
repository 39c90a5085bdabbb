/*
 * hodlr_oracle.h -- plain, slow, single-threaded CPU oracle for the HODLR
 * hot path of Ambikasaran, Foreman-Mackey, Greengard, Hogg, O'Neil,
 * "Fast Direct Methods for Gaussian Processes" (arXiv:1403.6015).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1403_6015_b200/, include/hodlr.h) never links,
 * imports or calls anything under oracle/, and this file shares no code,
 * header or constant with it.
 *
 * The oracle follows the paper's algorithm step by step, in the paper's
 * order:
 *   O1 sort              PAPER.md:666-677 (sec. 3, kd-tree ordering; 1-D = stable sort; d-D: per-level sorts)
 *   O2 tree              PAPER.md:1063 (Fig. 6 line 1, kappa = floor(log2 n/p_max))
 *   O3 entries           PAPER.md:281-308 (Table I), PAPER.md:1251-1256 (C_ij = s2 d_ij + k)
 *   O4 ACA               PAPER.md:837-864 (sec. 3.1, partial-pivoted LU / ACA)
 *   O5 leaves            PAPER.md:1072-1073 (Fig. 6 "form K_kappa"), Cholesky (R6)
 *   O6 leaf panel solve  PAPER.md:1076-1082 (Fig. 6 lines 8-12), eq-two-level-1 PAPER.md:951-962
 *   O7 level sweep       PAPER.md:1021-1048 (equation_Low_Rank_Update + SMW), eq-two-level PAPER.md:970-1014
 *   O8 log det           PAPER.md:1184-1230 (Sylvester theorem, multiplicativity)
 *   O9 solve             PAPER.md:1091-1100 (eq-fac, SMW on every factor)
 *   O10 log-likelihood   PAPER.md:99-103 (eq. 1, log form)
 *   O11 dense checker    plain assembled C, unblocked Cholesky (independent code path)
 *
 * Conventions: host pointers, FP64, column-major multi-RHS (y[j*ld+i]).
 * Every function returns an oracle_status; messages via oracle_last_error().
 * Built with gcc -O2 -ffp-contract=off (no FMA contraction, sequential sums).
 */
#ifndef HODLR_ORACLE_H
#define HODLR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_EINVAL = 1, ORACLE_ENOTPD = 2, ORACLE_ERANKCAP = 3,
       ORACLE_ESTATE = 4, ORACLE_ENOMEM = 5 };
enum { ORACLE_SE = 0, ORACLE_MATERN32 = 1, ORACLE_MATERN52 = 2, ORACLE_EXP = 3, ORACLE_IMQ = 4, ORACLE_RQ = 5,
       ORACLE_MQ = 6, ORACLE_BIHARM = 7 };   /* MQ, BIHARM: not positive definite (NEXT-2) */

typedef struct oracle_hodlr oracle_hodlr;

/* O3: one kernel value k(r) for distance d = x_i - x_j (no noise term). theta = {a, ell} ({a, ell, alpha} for RQ). */
double oracle_kernel(int kernel, const double *theta, double d);
/* O3 for d-dimensional points (NEXT-3): the same function of r = |x_i - x_j| given r2 = r^2 (SE from r2, the others
 * from sqrt(r2)). */
double oracle_kernel_r2(int kernel, const double *theta, double r2);

/* O4 on an explicit dense m1 x m2 column-major block A (lda >= m1).
 * U (m1 x cap) and V (m2 x cap) column-major, caller-allocated.
 * Returns the rank in *rank.  ORACLE_ERANKCAP if cap reached without meeting eps. */
int oracle_aca_dense(const double *A, int64_t m1, int64_t m2, int64_t lda, double eps,
                     int cap, double *U, double *V, int *rank);

/* O1-O4: sort, tree, compress every off-diagonal block ("Assembly").
 * rank_cap <= 0 means min(m1, m2) for every block. */
int oracle_build(const double *x, int64_t n, int kernel, const double *theta, double sigma2,
                 int leaf, double eps, int rank_cap, oracle_hodlr **out);
/* The same with heteroscedastic noise C_ij = k(x_i, x_j) + (sigma2 + noise_i) [i = j]: noise is
 * n finite values >= 0 in the caller's order (NULL = homoscedastic). */
int oracle_build_noise(const double *x, int64_t n, int kernel, const double *theta, double sigma2, const double *noise,
                       int leaf, double eps, int rank_cap, oracle_hodlr **out);
/* d-dimensional points (NEXT-3): x is n x dim, point-major (point i at x[i dim .. i dim + dim)); O1 is the kd-tree
 * ordering of PAPER.md:666-677 (each node of depth L sorts its points stably by coordinate L mod dim, then the
 * count-median split halves it).  dim = 1 is oracle_build_noise. */
int oracle_build_nd(const double *x, int64_t n, int dim, int kernel, const double *theta, double sigma2,
                    const double *noise, int leaf, double eps, int rank_cap, oracle_hodlr **out);
/* O5-O8: leaves, panel, sweep, log det ("Factor"). */
int oracle_factor(oracle_hodlr *h);
/* O8: log det C (after factor).  -INFINITY if the factorization failed.  (log |det C| for MQ / BIHARM.) */
int oracle_logdet(oracle_hodlr *h, double *logdet);
/* O8 with the sign of det C (kernels that are not SPD: leaves by LU, det S_c of either sign; +1 for SPD kernels). */
int oracle_logdet_sign(oracle_hodlr *h, double *logabs, int *sign);
/* O9: x = C^{-1} y in the caller's original point order; nrhs columns, leading dim ld. */
int oracle_solve(oracle_hodlr *h, const double *y, double *x, int64_t nrhs, int64_t ld);
/* O10: -1/2 y^T C^{-1} y - 1/2 log det C - n/2 log(2 pi). */
int oracle_gp_loglik(oracle_hodlr *h, const double *y, double *out);
/* HODLR matvec H v (the assembled hierarchical matrix), original order.  For pins. */
int oracle_apply(oracle_hodlr *h, const double *v, double *out);

/* Residual rows (C x - y)_r for the original row indices rows[0..nr) of a solution x (original order), C
 * assembled entry by entry.  For tests and the golden-file script. */
int oracle_residual_rows(oracle_hodlr *h, const double *x, const double *y, const int64_t *rows, int64_t nr,
                         double *out);

/* Introspection for tests. */
int     oracle_kappa(oracle_hodlr *h);
int64_t oracle_num_nodes(oracle_hodlr *h);
int     oracle_get_perm(oracle_hodlr *h, int64_t *perm);          /* n */
int     oracle_get_sorted(oracle_hodlr *h, double *xs);           /* n x dim, point-major */
int     oracle_dim(oracle_hodlr *h);
int     oracle_get_tree(oracle_hodlr *h, int64_t *lo, int64_t *hi); /* num_nodes each, heap order */
int     oracle_get_ranks(oracle_hodlr *h, int32_t *ranks);        /* 2^kappa - 1 internal nodes */
/* Copy U (m1 x r) and V (m2 x r) of internal node `node` (heap id), column-major. */
int     oracle_get_factors(oracle_hodlr *h, int64_t node, double *U, double *V);
/* Per-node log det partials: leaves (2^kappa, left to right) then internal nodes (heap ids). */
int     oracle_get_logdet_parts(oracle_hodlr *h, double *leaf_parts, double *node_parts);
void    oracle_free(oracle_hodlr *h);
const char *oracle_last_error(void);

/* O11: dense checker, separate code path: assemble C (original order), unblocked
 * Cholesky, log det = 2 sum log L_ii, forward/back solve of one rhs.  n <= 8192. */
int oracle_dense(const double *x, int64_t n, int kernel, const double *theta, double sigma2,
                 const double *y, double *logdet, double *xout);
int oracle_dense_noise(const double *x, int64_t n, int kernel, const double *theta, double sigma2, const double *noise,
                       const double *y, double *logdet, double *xout);
int oracle_dense_nd(const double *x, int64_t n, int dim, int kernel, const double *theta, double sigma2,
                    const double *noise, const double *y, double *logdet, double *xout);

#ifdef __cplusplus
}
#endif
#endif
