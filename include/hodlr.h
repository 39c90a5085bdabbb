/*
 * hodlr.h -- C-ABI of the B200-native HODLR library (libhodlr_b200.so).
 *
 * Hot path of Ambikasaran et al., "Fast Direct Methods for Gaussian Processes"
 * (arXiv:1403.6015): factor the GP covariance C = sigma2 I + K(x; theta) of
 * 1-D points x into the HODLR product K_kappa K_{kappa-1} ... K_0
 * (equation_HODLR_factorization), then log det C
 * (equation_determinant_completely_multiplicative),
 * the solve C^{-1} y (eq-fac) and the GP
 * log-likelihood (eq. 1), all in FP64 on one B200 (sm_100a).
 *
 * Every step runs in hand-written CUDA kernels; there is no CPU fallback.
 * The signatures carry plain pointers and sizes only (no torch types).
 *
 * Pointers: x, y and the solution are DEVICE pointers (contiguous FP64,
 * the caller's original point order), caller-owned, read or written only
 * during the call.  Scalars returned "_host" are host pointers.
 * Ownership: hodlr_build copies x (sorted copy + permutation) into the handle;
 * the handle owns all factors and device memory until hodlr_free.
 * Ordering: all device work is enqueued on `cuda_stream` (NULL = legacy
 * default stream); every call synchronises that stream before it returns its
 * status, so statuses are final.
 * State machine: build -> (factor | factor_solve) -> {logdet, solve, gp_loglik, gp_predict}*; hodlr_apply is legal
 * from build on.  Any other order returns HODLR_ESTATE.  After factor the handle is read-only; one
 * handle must not be used from two threads at once.
 * Errors: every call returns a hodlr_status; hodlr_last_error() gives a
 * thread-local message for the last failing call.
 */
#ifndef HODLR_B200_H
#define HODLR_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct hodlr_s *hodlr_t;   /* opaque handle; owns all device memory */

typedef enum {
  HODLR_OK = 0,
  HODLR_EINVAL = 1,    /* bad argument: n < 1, leaf < 1, eps not in (0,1), sigma2 < 0, ell <= 0, a < 0,
                          unknown kernel, NaN/Inf in x or y, nrhs < 1, ld < n */
  HODLR_ENOTPD = 2,    /* non-positive leaf Cholesky pivot, zero LU pivot or det <= 0 in a coupling
                          system S_c; logdet/loglik return -INFINITY */
  HODLR_ERANKCAP = 3,  /* an ACA block reached the rank cap without meeting eps (R12) */
  HODLR_ESTATE = 4,    /* call out of order */
  HODLR_ENOMEM = 5,    /* device allocation failed */
  HODLR_ECUDA = 6,     /* CUDA runtime error (message has the CUDA error string) */
  HODLR_ENCCL = 7      /* NCCL error (multi-GPU) */
} hodlr_status;

/* Covariance functions (Table I), theta = {a, ell} (RQ: {a, ell, alpha}):
 *   SE:        a^2 exp(-d^2 / (2 ell^2))
 *   MATERN32:  a^2 (1 + s) exp(-s),          s = sqrt(3) |d| / ell
 *   MATERN52:  a^2 (1 + s + s^2/3) exp(-s),  s = sqrt(5) |d| / ell
 *   EXP:       a^2 exp(-|d| / ell)            (Ornstein-Uhlenbeck, Table I; Table IV)
 *   IMQ:       a^2 / sqrt(1 + d^2 / ell^2)    (inverse multiquadric, Table V)
 *   RQ:        a^2 (1 + d^2 / ell^2)^-alpha   (rational quadratic, Table I), alpha = theta[2] > 0
 *   MQ:        a^2 sqrt(1 + d^2 / ell^2)    (multiquadric, sec. 5.2 / Table III)
 *   BIHARM:    a^2 q^2 log q, q = |d| / ell, 0 at d = 0 (biharmonic, sec. 5.4 / Table VI)
 * (NEXT-2 of SURVEY 8(f): the paper's other 1-D kernels.)  MQ and BIHARM are NOT positive definite (R20):
 * their leaves are factored by LU with partial pivoting, coupling systems of either sign are accepted, det C may be
 * negative (hodlr_logdet_sign), gp_loglik and the predictive variance refuse them (HODLR_EINVAL: not a covariance),
 * and they run on one GPU, unbatched (dist / hodlr_build_batch / gp_loglik_sweep: HODLR_EINVAL).
 * C_ij = k(x_i - x_j) + sigma2 [i == j]. */
typedef enum { HODLR_SE = 0, HODLR_MATERN32 = 1, HODLR_MATERN52 = 2, HODLR_EXP = 3, HODLR_IMQ = 4,
               HODLR_RQ = 5, HODLR_MQ = 6, HODLR_BIHARM = 7 } hodlr_kernel;

/* Multi-GPU descriptor (subtree sharding, north_star).  NULL or nranks == 1 => one GPU.
 * nranks = P must be a power of two with P <= 2^kappa.  Rank g owns the depth-log2(P) node g (sorted rows
 * [lo, hi) of that node) and its whole subtree; the points are replicated (every rank passes the same x, y,
 * theta, sigma2, leaf, eps).  The top log2(P) levels (their ACA blocks and coupling systems) are computed
 * redundantly by every rank; the ranks exchange, by allgather: the per-depth ACA ranks (build), the projected
 * Gram matrices of the depth-log2(P) nodes and the log det partials (factor), the solve's projections at
 * depth log2(P) and the sorted solution slices (solve).  Transport: NCCL (nccl_unique_id: the 128-byte
 * ncclUniqueId from hodlr_nccl_unique_id() on rank 0, broadcast by the caller; one GPU per rank), or an
 * in-process group of virtual ranks (group: from hodlr_group_create, one host thread per rank, all on the
 * current device) -- the latter runs the sharded path on one GPU.  Exactly one of the two must be set. */
typedef struct {
  int32_t rank, nranks;
  const void *nccl_unique_id;   /* 128 bytes, or NULL */
  void *group;                  /* hodlr_group_create() handle, or NULL */
} hodlr_dist;

/* Optional build options.  NULL => defaults; zero-initialise unused fields. */
typedef struct {
  int32_t rank_cap;             /* max ACA rank per block, <= 64; 0 => 48 (always clamped to min(m1, m2)) */
  int32_t flags;                /* reserved, must be 0 */
  /* Test hook (parity): HOST array of the 2^kappa - 1 internal nodes' ACA ranks in heap order, or NULL.  When set,
   * the ACA of block b runs exactly forced_ranks[b] cross steps (it still stops early on an exactly-zero residual
   * row) instead of applying the eps stopping test -- so the GPU can be run with the oracle's per-block ranks and
   * a parity difference separated into compression (different ranks) and arithmetic (same ranks).  Read only
   * during hodlr_build. */
  const int32_t *forced_ranks;
  /* Heteroscedastic noise (C_ij = sigma_i^2 delta_ij + k(x_i, x_j); NEXT-2 of SURVEY 8(f)): DEVICE
   * array of n finite values >= 0 in the caller's original point order, or NULL.  The diagonal of C is then
   * sigma2 + noise[i] (pass sigma2 = 0 for a purely per-point noise).  Read only during hodlr_build (copied, sorted,
   * into the handle).  HODLR_EINVAL on a negative or non-finite entry. */
  const double *noise;
  int64_t reserved[5];
} hodlr_opts;

typedef struct {
  int32_t kappa;                /* tree depth, floor(log2(n / leaf)) (Fig. 6 line 1) */
  int32_t leaf_min, leaf_max;   /* leaf block sizes, in [leaf, 2 leaf) */
  int32_t K;                    /* ancestor columns per leaf = sum of per-depth max ranks */
  int32_t max_rank_by_depth[64];   /* depth e = 1..kappa: max rank of the depth-(e-1) blocks */
  double  mean_rank_by_depth[64];
  int64_t factor_bytes;         /* device bytes held by the handle after factor */
  double  t_build, t_factor, t_logdet, t_solve;   /* seconds (CUDA events), last call of each */
  int64_t rank_cap_hits;        /* blocks that hit the rank cap */
  int32_t aca_steps;            /* ACA pivot steps executed (max rank + 1) */
  int32_t gpu_launches_last;    /* kernels launched by the last API call */
  /* Device time (ms, CUDA events on the handle's stream) accumulated since build, and call counts, per
   * kernel family: [0] sort, [1] ACA, [2] leaf factor (Z, Pi), [3] coupling tree, [4] solve (one cooperative
   * kernel), [5], [6] unused, [7] leaf Cholesky + inverse (side stream, overlaps the ACA). */
  double  kernel_ms[16];
  int64_t kernel_calls[16];
  int32_t rank, nranks, split_depth;   /* sharding (split_depth = log2(nranks)); ranks/means above cover the
                                          blocks this rank computed (its subtree and the top levels) */
  int32_t pad_;
} hodlr_info_t;

/* "Assembly": stable sort of x (O(n), K1), balanced count-median
 * tree with kappa = floor(log2(n/leaf)) levels, and ACA compression of every
 * off-diagonal block K[c1,c2] ~ U V^T to relative eps (sec. 3.1).
 * x: device, n doubles.  theta: HOST pointer to {a, ell} ({a, ell, alpha} for HODLR_RQ).  *out receives the
 * handle. */
hodlr_status hodlr_build(const double *x, int64_t n, hodlr_kernel kernel, const double *theta,
                         double sigma2, int32_t leaf, double eps, const hodlr_dist *dist,
                         const hodlr_opts *opts, void *cuda_stream, hodlr_t *out);

/* NEXT-3, d-dimensional points ("points in one, two, or three dimensions", Table II
 * PAPER.md:1302-1351).  Same "Assembly" as hodlr_build with the kd ordering of PAPER.md:666-677 ("sorted
 * recursively, one dimension at a time") as DESIGN.md R19 reads it: every depth-L node (L < max(kappa, 1), top
 * down) sorts its points stably by coordinate L mod dim before the count-median split; kernel entries are the
 * Table I functions of the Euclidean distance |x_i - x_j| (SE from its square).  x: device, n x dim row-major
 * (point i at x[i * dim .. i * dim + dim)).  1 <= dim <= 64 (dim = 1 is hodlr_build, bit for bit).  One GPU,
 * unbatched (no dist); noise, forced_ranks and rank_cap in opts as for hodlr_build.  The rest of the path (factor,
 * logdet, solve, factor_solve, gp_loglik, apply, gp_predict) is unchanged; gp_predict takes xt as m x dim
 * row-major test points.
 * hodlr_get_order returns the sorted points coordinate-major (dim x n: coordinate k of sorted point i at
 * xs[k * n + i]).  Limits: the ranks must meet eps within the rank cap (<= 64, else HODLR_ERANKCAP) and each
 * coupling system's on-chip working set must fit one SM (else HODLR_EINVAL at factor) -- 2-D problems of moderate
 * smoothness do; the paper's Table II 2-D/3-D settings, with ranks in the hundreds, do not. */
hodlr_status hodlr_build_nd(const double *x, int64_t n, int32_t dim, hodlr_kernel kernel, const double *theta,
                            double sigma2, int32_t leaf, double eps, const hodlr_opts *opts, void *cuda_stream,
                            hodlr_t *out);

/* "Factor" (Fig. 6): leaf Cholesky of K_kappa, bottom-up SMW coupling systems
 * S_c = [[I, V^T K_c2^{-1} V], [U^T K_c1^{-1} U, I]] (equation_Low_Rank_Update)
 * and their LU factors; accumulates log det C. */
hodlr_status hodlr_factor(hodlr_t h);

/* Factor with a right-hand side (fused factor + solve): hodlr_factor, with y carried through the
 * factorization as an extra panel column -- leaf Z = L^{-1} [y | E] and Pi = Z^T Z give the solve's leaf
 * projections, the coupling tree's T_c = S_c^{-1} B_c and Pi_c give its tree up pass (eq-fac, PAPER.md:1091-1100;
 * equation_Low_Rank_Update) -- then only the solve's down passes run.
 * y: device, n doubles (original order).  x: n doubles, receives C^{-1} y (original order), or NULL (no down pass):
 * device memory, or page-locked host memory (cudaHostAlloc / cudaMallocHost / cudaHostRegister: the solve kernel
 * writes it through the unified address, so the device-to-host transfer overlaps the leaf phase; pageable host
 * memory is HODLR_EINVAL).  quad_host: host double receiving y^T C^{-1} y (the root's Pi; eq. 1), or NULL.
 * Leaves the handle factored exactly like hodlr_factor (log det, solve / gp_loglik of other right-hand sides).
 * Errors: as hodlr_factor; HODLR_EINVAL if y has NaN/Inf (the handle is still factored). */
hodlr_status hodlr_factor_solve(hodlr_t h, const double *y, double *x, double *quad_host);

/* "Det." (sec. 4): log det C = sum_leaves 2 sum log L_ii + sum_c log det S_c.
 * logdet_host: host double.  -INFINITY with HODLR_ENOTPD if the factorization failed. */
hodlr_status hodlr_logdet(hodlr_t h, double *logdet_host);

/* log |det C| and the sign of det C (O8, R20): the product of the leaves' LU
 * determinant signs and the coupling systems' signs; +1 for every SPD kernel (whose factorization refuses any other
 * sign with HODLR_ENOTPD).  logabs_host: host double (hodlr_logdet's value); sign_host: host int32 in {-1, +1}
 * (0 with HODLR_ENOTPD when the factorization failed: a zero pivot). */
hodlr_status hodlr_logdet_sign(hodlr_t h, double *logabs_host, int32_t *sign_host);

/* Solve C X = Y (eq-fac).  y, x: device, column-major n x nrhs with leading
 * dimension ld >= n, original point order.  x may not alias y. */
hodlr_status hodlr_solve(hodlr_t h, const double *y, double *x, int64_t nrhs, int64_t ld);

/* Forward apply Y = C~ X of the compressed operator (NEXT-1): the leaf diagonal
 * blocks K_ll + sigma^2 I evaluated on the fly (Table I) plus U V^T / V U^T of every ACA block
 * (sec. 3.1) -- the operator hodlr_solve inverts, so apply(solve(y)) = y to rounding.  Legal
 * after hodlr_build (factoring is not needed).  x, y: device, column-major n x nrhs, leading dimension ld >= n,
 * original point order; y may not alias x.  Single-GPU handles only (HODLR_EINVAL when sharded). */
hodlr_status hodlr_apply(hodlr_t h, const double *x, double *y, int64_t nrhs, int64_t ld);

/* GP prediction at m test points (eq_reg1 / eq_reg2; NEXT-1): mean_j = k(xt_j, x) C^{-1} y and,
 * if var != NULL, the latent variance var_j = k(xt_j, xt_j) - k(xt_j, x) C^{-1} k(x, xt_j) (sigma^2 not added).
 * Cross-covariances on the fly, C^{-1} by the HODLR solve.  y: device n (original order); xt: device m (m x dim row-major on a hodlr_build_nd handle); mean, var: device m.
 * Legal after hodlr_factor; single-GPU handles only (HODLR_EINVAL when sharded). */
hodlr_status gp_predict(hodlr_t h, const double *y, const double *xt, int64_t m, double *mean, double *var);

/* GP log-likelihood (eq. 1): -1/2 y^T C^{-1} y - 1/2 log det C - (n/2) log(2 pi).
 * y: device, n doubles.  out_host: host double (-INFINITY with HODLR_ENOTPD on failure). */
hodlr_status gp_loglik(hodlr_t h, const double *y, double *out_host);

/* Batched factorizations (NEXT-4: the marginalisation / hyper-parameter loops of PAPER.md:399-446
 * evaluate many settings on the same points): B = 2^t independent problems C_s = sigma2s[s] I + K(x; thetas[s]) on
 * the same n points x (device, original order), held in ONE handle as the block-diagonal matrix
 * diag(C_0, ..., C_{B-1}) of order B n.  Problem s occupies rows [s n, (s + 1) n) of every vector argument of the
 * handle (y, x of hodlr_solve / hodlr_factor_solve / hodlr_apply: device, B n doubles, problem-major, each problem in
 * the original point order).  The tree is the B-fold tree whose top t levels split exactly between problems (n B
 * halves evenly) -- their off-diagonal blocks are zero and skipped (rank 0) -- and whose subtree s below is problem
 * s's own tree; every kernel launch of the path then covers all B problems (one ACA step loop, one leaf Cholesky
 * launch, one zsyrk, one pass per tree level).  thetas: HOST B x 2 {a, ell} (B x 3 for HODLR_RQ); sigma2s: HOST
 * B.  Requires n >= leaf; no dist, no noise.  The handle then follows the usual state machine; hodlr_logdet /
 * gp_loglik report the whole block-diagonal matrix (the sum over problems), hodlr_batch_results each problem's.
 * gp_predict refuses batched handles (HODLR_EINVAL).  A failure (HODLR_ENOTPD, HODLR_ERANKCAP) in any problem fails
 * the handle. */
hodlr_status hodlr_build_batch(const double *x, int64_t n, hodlr_kernel kernel, const double *thetas,
                               const double *sigma2s, int32_t B, int32_t leaf, double eps, const hodlr_opts *opts,
                               void *cuda_stream, hodlr_t *out);

/* Per-problem results of a factored batched handle (HOST arrays of B doubles): log det C_s (its subtree's leaf and
 * node partials, fixed compensated order) and, if quad_host != NULL, y_s^T C_s^{-1} y_s of the right-hand side fused
 * by hodlr_factor_solve (HODLR_ESTATE if none was).  Synchronizes the handle's stream.  On a B = 1 handle: the
 * handle's own log det and y^T C^{-1} y. */
hodlr_status hodlr_batch_results(hodlr_t h, double *logdet_host, double *quad_host);

/* Config 4 (BASELINE.json): log-likelihoods (eq. 1) of B independent hyper-parameter settings on the same
 * x, y (device, n doubles).  thetas: HOST B x 2 {a, ell}; sigma2s: HOST B; out_host: HOST B doubles (-INFINITY
 * for a setting that failed).  The settings are factored in batches (hodlr_build_batch): the largest powers of two
 * that fit (at most 2^23 / n problems per batch), each one hodlr_factor_solve with y fused into all problems
 * (y^T C_s^{-1} y from the factorization, no solve pass) and hodlr_batch_results.  A batch that fails is redone
 * setting by setting (`workers` host threads, one stream each; <= 0 => 8) so that every setting gets its own status
 * and value.  With dist (nranks > 1) rank g computes settings g, g + P, ... and the values are allgathered, so
 * every rank returns all B (replicas; the settings share nothing).  Returns the first failing setting's status
 * (message names it), HODLR_OK if all succeeded. */
hodlr_status gp_loglik_sweep(const double *x, const double *y, int64_t n, hodlr_kernel kernel, const double *thetas,
                             const double *sigma2s, int32_t B, int32_t leaf, double eps, const hodlr_dist *dist,
                             void *cuda_stream, int32_t workers, double *out_host);

/* Sizes, ranks and phase times.  info: host struct. */
hodlr_status hodlr_info(hodlr_t h, hodlr_info_t *info);

/* Copy the sorted points (n doubles; dim x n coordinate-major for a hodlr_build_nd handle) and the permutation perm[i] = original index of sorted
 * position i (n int64) to DEVICE buffers; either may be NULL.  For parity tests (bit-exact). */
hodlr_status hodlr_get_order(hodlr_t h, double *xs_dev, int64_t *perm_dev);

/* Copy the tree (node ranges [lo, hi) in heap order, 2^(kappa+1)-1 nodes) and the ACA ranks of the
 * 2^kappa - 1 internal nodes to HOST buffers; either may be NULL. */
hodlr_status hodlr_get_tree(hodlr_t h, int64_t *lo_host, int64_t *hi_host, int32_t *ranks_host);

/* Per-leaf (2^kappa) and per-internal-node (heap order) log det partials, HOST buffers. */
hodlr_status hodlr_get_logdet_parts(hodlr_t h, double *leaf_parts_host, double *node_parts_host);

/* Fill out128 with a fresh ncclUniqueId (NCCL is loaded at run time with dlopen("libnccl.so.2")).
 * HODLR_ENCCL if NCCL is unavailable. */
hodlr_status hodlr_nccl_unique_id(void *out128);

/* In-process group of nranks virtual ranks (host threads sharing one process and device).  Destroy only
 * after every handle that uses it has been freed. */
hodlr_status hodlr_group_create(int32_t nranks, void **group);
void         hodlr_group_destroy(void *group);

/* Scaling projection on one GPU: mode 1 records every exchange of the next sharded run (all virtual
 * ranks running, rank 0's gathered buffers kept on the device); mode 2 replays: only rank 0 runs, and each exchange
 * returns the recorded buffer with rank 0's own slot replaced by its live data -- rank 0's critical path without the
 * other ranks' work on the shared GPU (replay must repeat the recorded call sequence; HODLR_EINVAL otherwise);
 * mode 0 = normal.  HODLR_ESTATE for mode 2 with nothing recorded. */
hodlr_status hodlr_group_mode(void *group, int32_t mode);

/* Host-side shard plan (no device work): tree depth kappa, split depth t = log2(nranks), the sorted row range
 * [row_lo, row_hi) and leaf range [leaf_lo, leaf_hi) owned by `rank`.  HODLR_EINVAL for an invalid split. */
hodlr_status hodlr_dist_plan(int64_t n, int32_t leaf, int32_t rank, int32_t nranks, int32_t *kappa, int32_t *t,
                             int64_t *row_lo, int64_t *row_hi, int64_t *leaf_lo, int64_t *leaf_hi);

/* Release everything the handle owns.  NULL is a no-op.  Synchronizes the handle's streams; its device blocks are
 * kept by the library (exact-size reuse by later handles on the same device, at most 16 GB per process) rather
 * than returned to the CUDA pool, so repeated builds of one shape allocate nothing. */
void hodlr_free(hodlr_t h);

/* Return every device block the library keeps for reuse (see hodlr_free) to the CUDA pool.  Safe at any time (cached
 * blocks have no pending work); live handles are unaffected. */
void hodlr_cache_trim(void);

/* Thread-local message of the last failing call (never NULL). */
const char *hodlr_last_error(void);

/* Library self-description, e.g. "hodlr_b200 sm_100a". */
const char *hodlr_version(void);

/* Number of CUDA kernels this library has launched in the process (all handles). */
int64_t hodlr_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
