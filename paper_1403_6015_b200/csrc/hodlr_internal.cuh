// hodlr_internal.cuh -- shared internals of libhodlr_b200 (product path; no oracle code).
//
// Layout in HBM:
//   xs[n], perm[n]            sorted points, permutation (sorted position -> original index)
//   lo[], hi[]                node ranges, heap order: node (d, i) has id 2^d - 1 + i
//   Xh                        ACA factors, column-major per depth "slot": depth e = 1..kappa owns
//                             capd[e] columns of n doubles starting at column colbase[e]; column l
//                             of slot e holds, on the rows of each depth-e node a, the l-th left
//                             factor of a (U' of a left child, V' of a right child)
//   Lf                        leaf Cholesky factors, packed lower row-major, lstride doubles/leaf
//   per depth d:  S LU (q x q), piv, B (q x Kd), T (q x Kd), Pi (Kd x Kd) per node
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "../../include/hodlr.h"
#include <algorithm>

#define HODLR_MAXDEPTH 48
#define HODLR_PIN_BYTES (1 << 20)  // pinned host staging per pooled stream set (flags, ranks, scalars)
#define TREE_TOP_MAXLEV HODLR_MAXDEPTH   // levels of one persistent upper-tree launch
#define ACA_MAXCAP 64      // hard ceiling on the ACA rank cap (records/state are sized by it)
#define ACA_RECW (4 + ACA_MAXCAP)
#ifndef ACA_SUB
#define ACA_SUB 256        // threads per ACA CTA == sub-tile width
#endif
#ifndef ACA_FUSED_MAX
#define ACA_FUSED_MAX 4096 // blocks with both sides <= this run the fused single-CTA ACA
#endif
#ifndef ACA_BIG_CHUNK
#define ACA_BIG_CHUNK 4096 // minimum chunk per CTA for the step-synchronous big blocks (measured: 8192 0.2 ms slower)
#endif
#ifndef ACA_CHUNKS_PER_SIDE
#define ACA_CHUNKS_PER_SIDE 64    // max chunks (CTAs, records) per block side
#endif

// ----------------------------------------------------------------------------------------------
// Covariance functions, Table I; C_ij = k(x_i - x_j) + s2 [i == j]
// (PAPER.md:1251-1256).  kp = {a^2, c} with c = 1/(2 ell^2) for SE, sqrt(3)/ell or sqrt(5)/ell
// for Matern-3/2 and -5/2.
// ----------------------------------------------------------------------------------------------
struct KParams {
  int kern; double a2; double c; double s2; double alpha;
  double ell, c2, sq;       // ell; SE 2 ell^2 as (2 ell) ell; Matern sqrt(3) / sqrt(5) -- for kval_o
  double rc2, rell;         // 1 / c2, 1 / ell when that reciprocal is exact (a power of two: x / c == x * (1 / c)
                            // bit for bit, and a multiply is far cheaper than a division), else 0
  const double *dn;         // heteroscedastic noise: sigma_i^2 = s2 + noise_i in SORTED order (device), or NULL
  int dim;                  // point dimension d (NEXT-3): xs holds coordinate k of sorted point i at xs[k * ldp + i]
  long long ldp;            // coordinate stride of xs (= n; 1-D: the single coordinate row)
};
// the diagonal term sigma_i^2 of sorted point i (C_ij = sigma_i^2 delta_ij + k(x_i, x_j))
__device__ __forceinline__ double sig2(const KParams &kp, long long i) { return kp.dn ? kp.dn[i] : kp.s2; }
// Batched handles (hodlr_build_batch, NEXT-4): B problems on the same points, problem s on the sorted rows
// [s nseg, (s + 1) nseg) with its own covariance parameters kps[s].  Every covariance entry the path evaluates lies
// inside one problem's rows (the blocks of the top log2 B levels are exactly zero and skipped, and leaves never
// straddle problems), so one lookup per block or leaf selects the parameters.
__device__ __forceinline__ const KParams &kp_of(const KParams &kp, const KParams *kps, long long nseg, long long row) {
  return kps ? kps[row / nseg] : kp;
}
// x / b for many x and one b: rb = RN(1 / b), q = RN(x rb), then one FMA correction with the exact remainder
// x - b q (Markstein): the correctly rounded quotient (barring over/underflow) at 3 FP ops instead of a division
__device__ __forceinline__ double div_by(double x, double b, double rb) {
  const double q = x * rb;
  return fma(fma(-q, b, x), rb, q);
}
// x / c with the reciprocal when it is exact (rc != 0), else a correctly rounded division: the same bits either way
__device__ __forceinline__ double div_exact(double x, double c, double rc) { return rc != 0.0 ? x * rc : __ddiv_rn(x, c); }

// Non-SE kernels share one exp: Matern pre (1 + s [+ s^2/3]) e^{-s}; EXP e^{-|d| c}; IMQ / RQ (1 + d^2 c)^{-alpha}
// = e^{-alpha log(1 + d^2 c)} (no pow: u >= 1, alpha > 0), with c = sqrt(3)/ell, sqrt(5)/ell, 1/ell, 1/ell^2.
// MQ a^2 sqrt(1 + d^2 c), BIHARM a^2 s^2 log s with s = |d| c (c = 1/ell^2, 1/ell): DESIGN.md R20.
__device__ __forceinline__ double kval(const KParams &kp, double d) {
  if (kp.kern == HODLR_SE) return kp.a2 * exp(-(d * d) * kp.c);
  if (kp.kern == HODLR_MQ) return kp.a2 * sqrt(fma(d * d, kp.c, 1.0));
  if (kp.kern == HODLR_BIHARM) { const double q = fabs(d) * kp.c; return q == 0.0 ? 0.0 : kp.a2 * (q * q) * log(q); }
  const double s = fabs(d) * kp.c;
  double pre = 1.0, arg = -s;
  if (kp.kern == HODLR_MATERN32) pre = 1.0 + s;
  else if (kp.kern == HODLR_MATERN52) pre = 1.0 + s + s * s * (1.0 / 3.0);
  else if (kp.kern >= HODLR_IMQ) arg = -kp.alpha * log(fma(d * d, kp.c, 1.0));
  return kp.a2 * pre * exp(arg);
}
// KV: the kernel family when the launch knows it (KV_SE: the bench / config 1, 3, 5 path; KV_M52: config 4): exactly
// that code, nothing else inlined; KV_ANY: the run-time switch
constexpr int KV_ANY = -1, KV_SE = HODLR_SE, KV_M52 = HODLR_MATERN52;
static inline int kv_of(int kern) { return kern == HODLR_SE ? KV_SE : (kern == HODLR_MATERN52 ? KV_M52 : KV_ANY); }
template <int KV> __device__ __forceinline__ double kval_t(const KParams &kp, double d) {
  if (KV == KV_SE) return kp.a2 * exp(-(d * d) * kp.c);
  if (KV == KV_M52) { const double s = fabs(d) * kp.c; return kp.a2 * (1.0 + s + s * s * (1.0 / 3.0)) * exp(-s); }
  return kval(kp, d);
}

// ----------------------------------------------------------------------------------------------
// ACA per-block state (device).  Stored factors in the oracle's normalisation (O4, R16): V[:,k] = v~ / v~_jk
// (the row pass writes v~, the next column pass divides it by the pivot), U[:,k] = u unscaled.
// ----------------------------------------------------------------------------------------------
struct AcaState {
  int k;            // number of terms so far
  int done;         // 0 active, 1 finished, 2 hit the rank cap without meeting eps
  int cnt_r, cnt_c; // CTA arrival counters (last-CTA reduction)
  int cap;          // min(rank_cap, m1, m2)
  int raw_last;     // finished in a column pass: V[:, rank-1] still holds the raw residual (k_aca_finish divides it)
  int donly;        // the step after the rank cap: passes form the last column's dots only (lagged stop test)
  long long ipiv;   // current row pivot (local in c1)
  long long jpiv;   // current column pivot (local in c2)
  double pivval;    // v~_jk
  double S2;        // ||S_k||_F^2 estimate
  double nv2;       // ||V'[:,k-1]||^2, formed by the row pass of step k (lagged stop test)
  double dV[ACA_MAXCAP];   // V'_l . V'_{k-1}, l < k - 1, formed by the row pass of step k
};

// One CTA of a big-block pass: a chunk [start, start + len) of one side of `block`, with the block geometry
// precomputed on the host (the kernel prologue then needs no dependent loads of the tree tables).
struct AcaItem {
  int block; int q; long long start; int len; int e;   // e: slot depth (block depth + 1)
  long long lo1, lo2, m1, m2;                         // child ranges: rows c1 = [lo1, lo1+m1), columns c2
  long long slot_off;                                 // colbase[e] * n: first factor column of the slot
};

// Per-depth metadata passed by value.
struct DepthTab {
  long long colbase[HODLR_MAXDEPTH + 2];   // first column of slot e
  int capd[HODLR_MAXDEPTH + 2];            // columns allocated in slot e
  int rdep[HODLR_MAXDEPTH + 2];            // max rank of depth-(e-1) blocks (after build)
  int Kdim[HODLR_MAXDEPTH + 2];            // Kdim[e] = sum_{e'=1..e} rdep[e']
  int Kf[HODLR_MAXDEPTH + 2];              // factor-side widths Kdim[e] + aug: with a right-hand side fused into the
                                           // factorization (hodlr_factor_solve) it is column 0 of every panel / Pi
  long long nodeS[HODLR_MAXDEPTH + 2];     // per depth d: offset of S LU storage (doubles)
  long long nodeBT[HODLR_MAXDEPTH + 2];    // per depth d: offset of B/T storage (doubles)
  long long nodeV[HODLR_MAXDEPTH + 2];     // per depth d: offset of per-node vectors (g, w) (doubles)
  long long nodeT[HODLR_MAXDEPTH + 2];     // per depth d: offset of per-node t (doubles)
  long long piOff[HODLR_MAXDEPTH + 2];     // per depth e: offset of Pi storage (doubles)
};

struct AcaCtx {
  KParams kp;
  long long n;
  long long ldx;            // column stride of Xh (n padded, see hodlr_s::ldx)
  long long zrow;           // first of the 32 padding rows of every Xh column (>= n; zeroed when a chunk needs them)
  double eps;
  const double *xs;
  const long long *lo, *hi;
  double *Xh;
  unsigned char *used;      // kappa x ldx flags: used[(e-1)*ldx + row]
  AcaState *st;
  const AcaItem *items;
  const int *nq;            // chunks per block for this pass
  const long long *recbase; // record base per block for this pass
  double *rec;              // records
  int *active;
  int *rank;
  const int *bdepth;        // depth of each internal block
  DepthTab *dt;             // device copy
  const int *bigidx;        // block -> ordinal among the step-synchronous (big) blocks, -1 otherwise
  int *flags;               // handle flags (rank-cap hits in [5])
  int *step;                // step counter of the device loop
  int maxsteps;
  int nitems;               // items of this pass (the persistent step kernel strides over them)
  const int *forced;        // test hook (hodlr_opts.forced_ranks): stop block b at exactly forced[b] terms, or NULL
  const KParams *kps;       // batched handle: per-problem parameters (kp_of), or NULL
  long long nseg;           // batched handle: rows per problem
};

// ----------------------------------------------------------------------------------------------
// Per-kernel-family device timing (CUDA events on the handle's stream)
// ----------------------------------------------------------------------------------------------
enum { PH_SORT = 0, PH_ACA, PH_LEAF, PH_TREE, PH_SLEAF_UP, PH_STREE, PH_SLEAF_DOWN, PH_CHOL, PH_N };

// ----------------------------------------------------------------------------------------------
// Handle
// ----------------------------------------------------------------------------------------------
struct hodlr_s {
  cudaStream_t st;
  cudaStream_t st2;           // side stream (fused small-block ACA)
  cudaStream_t st2b;          // second fused-ACA stream (the smallest blocks, 64-thread CTAs)
  cudaEvent_t ev_join2;
  cudaStream_t st3;           // side stream (leaf Cholesky, overlapping the ACA)
  cudaStream_t sthi;          // high-priority stream (ACA step loop)
  cudaEvent_t ev_hi;
  cudaEvent_t ev_fork, ev_join, ev_chol;
  int chol_done;              // the leaf Cholesky kernel was issued on st3 (fast path)
  int dev;
  long long n;
  KParams kp;
  // batched handle (hodlr_build_batch): nbatch = 2^tbatch problems of nseg points each (n = nbatch * nseg); the
  // per-problem parameters on the device; nbatch = 1, d_kps = NULL otherwise
  int nbatch, tbatch;
  long long nseg;
  KParams *d_kps;
  double theta[2];
  int leaf;
  double eps;
  int cap;
  int kappa;
  long long nnodes, ninternal, nleaves;
  int leaf_min, leaf_max;
  // subtree sharding (dist.cu): rank g of nranks = 2^tsplit owns the depth-tsplit node g and its subtree
  int grank, nranks, tsplit;
  void *comm;                // ncclComm_t (NCCL transport) or NULL
  void *group;               // HodlrGroup (in-process transport) or NULL
  long long *d_rowlo;        // per rank: first sorted row of its subtree (device, nranks entries)
  long long rows_max;        // max subtree rows over the ranks (allgather slice size of the solution)
  int state;                 // 1 built, 2 factored, -1 factor failed
  int aug;                   // right-hand sides fused into the factorization (0 or 1)
  int coop_ctas;             // cap on the CTAs of the persistent (cooperative) launches, 0 = the whole GPU: concurrent
                             // problems (the config-4 sweep) leave each other room instead of serialising
  const double *y_aug;       // that right-hand side (device, original order) during hodlr_factor_solve
  void *pin;                 // pinned host staging (HODLR_PIN_BYTES, from the per-device pool), or NULL
  int launches;              // kernels launched by the current call
  int aca_steps;
  int x_nonfinite;           // set by the sort: x contains NaN/Inf
  long long rank_cap_hits;
  // host copies
  long long *h_lo, *h_hi;
  int *h_rank;
  DepthTab dt;
  // device
  double *xs;
  long long *perm;
  long long *lo, *hi;
  long long ldx;              // column stride of Xh: n rounded up to 32 plus 32 doubles, so that the columns of a
                              // leaf panel (1 KB each) do not all fall on the same DRAM channels (stride != 2^k)
  double *Xh;
  long long xh_cols;
  unsigned char *used;
  AcaState *ast;
  int *rank;
  int *bdepth;
  int *d_forced;             // hodlr_opts.forced_ranks on the device (test hook), or NULL
  double *d_noise;           // heteroscedastic sigma_i^2 in sorted order (hodlr_opts.noise), or NULL
  struct TreeCtx *d_treectx; // per-level contexts of the persistent upper-tree launch (factor.cu)
  int *d_ready;              // k_tree_top per-node progress flags (factor.cu, tree_node.cuh)
  int *dflags;               // [0] nonfinite x, [1] notpd, [2] notpd node (min), [3] nonfinite y, [4] active big
                             // ACA blocks, [5] rank-cap hits, [6] ACA steps, [7] x not ascending, [10] negative
                             // determinants (LU leaves, coupling systems) of a kernel that is not SPD
  DepthTab *d_dt;
  // factor storage
  double *Lf; long long lstride; int ltiles;   // leaf factor tiles (see storage helpers)
  int dim;                   // point dimension (NEXT-3; xs is coordinate-major, dim x n)
  int nonspd;                // MQ / BIHARM: LU leaves, either sign (R20)
  int det_sign;              // sign of det C after the factorization (+1 for the SPD kernels)
  double *Uf; int *lperm;    // LU leaves: U^{-T} tiles (as Lf) and the row order P (8 ltiles ints per leaf)
  double *Spool;  int *Piv;  double *BTpool; double *Pipool;
  double *leaf_ld, *node_ld, *d_logdet;
  double logdet;
  // solve workspace
  double *Vpool, *Tvec, *hvec;
  int solve_cols;            // right-hand sides the solve pools hold (per column: vcol, tcol, hcol doubles)
  long long vcol, tcol, hcol;
  double *xshard;            // sharded solve: sorted solution rows + allgather send/recv slices
  unsigned long long *stamps;  // HODLR_TRACE phase timestamps
  int bulk_ok, bulk_checked;   // solve leaf staging by bulk copies
  // bookkeeping
  long long bytes;
  double t_build, t_factor, t_logdet, t_solve;
  cudaEvent_t ev0, ev1;
  cudaEvent_t ph_ev[PH_N][2];
  int ph_pending[PH_N];
  double ph_ms[PH_N];        // accumulated device ms per kernel family (since build)
  long long ph_calls[PH_N];
  void *allocs[64]; size_t alloc_bytes[64]; unsigned char alloc_tmp[64]; int nallocs;
  double *apply_ws = nullptr; size_t apply_ws_n = 0;   // hodlr_apply workspace (apply.cu)
  double *pred_ws = nullptr; size_t pred_ws_n = 0;     // gp_predict workspace (predict.cu)
};

static inline void ph_begin(hodlr_s *h, int p, cudaStream_t s = nullptr) { cudaEventRecord(h->ph_ev[p][0], s ? s : h->st); }
static inline void ph_end(hodlr_s *h, int p, cudaStream_t s = nullptr) { cudaEventRecord(h->ph_ev[p][1], s ? s : h->st); h->ph_pending[p] = 1; }

// HODLR_TRACE=1: host timestamps of the orchestration steps on stderr (development aid)
void hodlr_trace(const char *what);
int hodlr_trace_on();

// helpers implemented in api.cu
hodlr_status hodlr_set_error(hodlr_status code, const char *fmt, ...);
hodlr_status hodlr_cuda_check(cudaError_t e, const char *what);
void *hodlr_dalloc(hodlr_s *h, size_t bytes);
// Allow `func` the device's whole opt-in shared memory (minus its static shared memory).  Called before every
// launch that needs more than 48 KB: the value is the same from every thread and handle, so concurrent handles
// needing different sizes cannot race; occupancy follows each launch's own size.
cudaError_t hodlr_allow_smem(const void *func, int dev);
void *hodlr_dalloc_tmp(hodlr_s *h, size_t bytes);   // dead after the build: handed to the block cache when it ends
extern long long hodlr_global_launches;

// phase entry points (one per .cu file)
hodlr_status hodlr_sort_and_tree(hodlr_s *h, const double *x, long long n);   // sorts n <= h->n points
hodlr_status hodlr_kd_sort(hodlr_s *h, const double *x, long long n, int dim);   // NEXT-3: kd ordering, d > 1
hodlr_status hodlr_aca(hodlr_s *h);
hodlr_status hodlr_factor_impl(hodlr_s *h);
hodlr_status hodlr_batch_parts(hodlr_s *h, double *d_out);   // batched: per-problem log det [B] and y^T C^-1 y [B]
hodlr_status hodlr_leaf_factor_mma(hodlr_s *h, int K, double *Pi_leaf, bool *used);
hodlr_status hodlr_apply_impl(hodlr_s *h, const double *x, double *y);
hodlr_status hodlr_predict_impl(hodlr_s *h, const double *y, const double *xt, long long m, double *mean, double *var);
hodlr_status hodlr_leaf_chol_mma(hodlr_s *h, cudaStream_t stream, bool *launched);
hodlr_status hodlr_leaf_alloc(hodlr_s *h);
hodlr_status hodlr_solve_impl(hodlr_s *h, const double *y, double *x, int64_t nrhs, int64_t ld, bool up_only,
                              bool fused = false);

static inline int hodlr_depth_of(long long id) { int d = 0; while (id >= ((2LL << d) - 1)) d++; return d; }

// Nodes of depth d this rank computes: all 2^d above the split depth, its own 2^(d - t) below it.
static inline void hodlr_own_nodes(const hodlr_s *h, int d, long long *i0, long long *cnt) {
  if (d < h->tsplit) { *i0 = 0; *cnt = 1LL << d; }
  else { *cnt = 1LL << (d - h->tsplit); *i0 = (long long)h->grank * *cnt; }
}
// Is internal block b (heap id, depth d) computed by this rank?
static inline bool hodlr_owns_block(const hodlr_s *h, long long b) {
  const int d = hodlr_depth_of(b);
  if (d < h->tsplit) return true;
  return (((b + 1) >> (d - h->tsplit)) - 1) == ((1LL << h->tsplit) - 1 + h->grank);
}

// dist.cu
hodlr_status hodlr_dist_init(hodlr_s *h, const hodlr_dist *d);
void hodlr_dist_fini(hodlr_s *h);
hodlr_status hodlr_allgather(hodlr_s *h, const void *send, void *recv, size_t bytes);   // bytes per rank

#define HCUDA(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) return hodlr_cuda_check(_e, #call); } while (0)
#define HLAUNCH(h, name) do { (h)->launches++; hodlr_global_launches++; cudaError_t _e = cudaGetLastError(); \
    if (_e != cudaSuccess) return hodlr_cuda_check(_e, "launch " name); } while (0)

// ----------------------------------------------------------------------------------------------
// Block-level reduction helpers
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// ----------------------------------------------------------------------------------------------
// Compensated (double-double) arithmetic for the small coupling systems:
// error-free transformations TwoSum / TwoProduct (FMA) and a Dot2-style accumulator.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
  s = a + b; double bb = s - a; e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void two_prod(double a, double b, double &p, double &e) { p = a * b; e = fma(a, b, -p); }
struct Acc2 { double s, c; };
__device__ __forceinline__ Acc2 acc2(double x) { Acc2 A; A.s = x; A.c = 0.0; return A; }
__device__ __forceinline__ void acc_add(Acc2 &A, double x) { double s, e; two_sum(A.s, x, s, e); A.s = s; A.c += e; }
__device__ __forceinline__ void acc_add_dd(Acc2 &A, double xh, double xl) { acc_add(A, xh); A.c += xl; }
__device__ __forceinline__ void acc_fma(Acc2 &A, double a, double b) {          // A += a * b
  double p, e; two_prod(a, b, p, e); acc_add(A, p); A.c += e;
}
__device__ __forceinline__ void acc_fma_dd(Acc2 &A, double a, double bh, double bl) {   // A += a * (bh + bl)
  acc_fma(A, a, bh); A.c = fma(a, bl, A.c);
}
__device__ __forceinline__ double acc_val(const Acc2 &A) { return A.s + A.c; }
__device__ __forceinline__ void acc_dd(const Acc2 &A, double &hi, double &lo) { two_sum(A.s, A.c, hi, lo); }

// exp(x) correctly rounded for x in (-708, 0] (outside: the library exp), for the ACA entries (R17): the
// host libm's exp is correctly rounded in all but ~0.1% of arguments while CUDA's exp differs from it in ~6%; at
// eps = 1e-12 the ACA residuals are rounding noise near the stopping threshold, so entry-level differences flip
// rank decisions.  x = k ln2/512 + r (Cody-Waite in three parts, r as a double-double), exp(r) - 1 by a degree-5
// polynomial (|r| <= ln2/1024, truncation 2^-72 relative), 2^(j/512) from a double-double table, one final rounding.
#include "exp_table.cuh"
__device__ __forceinline__ double exp_cr(double x) {
  if (!(x > -708.0) || x > 0.0) return exp(x);
  const double kd = rint(x * INV_LN2_512);
  const int k = (int)kd;
  const double t = fma(-kd, LN2_512_HI, x);             // exact: k * LN2_512_HI has <= 53 bits
  double p_hi, p_lo; two_prod(kd, LN2_512_LO, p_hi, p_lo);
  double r_hi, r_lo; two_sum(t, -p_hi, r_hi, r_lo);
  r_lo = r_lo - p_lo - kd * LN2_512_LO2;
  const double q = r_hi * r_hi * (0.5 + r_hi * (1.0 / 6.0 + r_hi * (1.0 / 24.0 + r_hi * (1.0 / 120.0))));
  double a_hi, a_lo; two_sum(r_hi, q, a_hi, a_lo);
  a_lo += r_lo + r_lo * r_hi;                          // exp(r) - 1 = a_hi + a_lo
  const int j = k & 511, m = k >> 9;                   // k = 512 m + j
  const double Th = EXP2_HI[j], Tl = EXP2_LO[j];
  double pp_hi, pp_lo, s_hi, s_lo;
  two_prod(Th, a_hi, pp_hi, pp_lo);
  two_sum(Th, pp_hi, s_hi, s_lo);
  const double lo = s_lo + pp_lo + Tl + Th * a_lo + Tl * a_hi;
  return scalbn(s_hi + lo, m);
}

// The same covariance functions in the oracle's operation order (the oracle's covariance function, built without FMA
// contraction): explicitly rounded operations, ell divided rather than multiplied by a reciprocal.  The ACA's pivots
// and ranks are FP-derived (R11); evaluating its entries (and residual updates) in the oracle's order keeps
// its decisions the oracle's up to ulp differences of exp / log / pow between the two math libraries (R17).
__device__ __forceinline__ double kval_o(const KParams &kp, double d) {
  switch (kp.kern) {
    case HODLR_SE: return __dmul_rn(kp.a2, exp_cr(-div_exact(__dmul_rn(d, d), kp.c2, kp.rc2)));
    case HODLR_EXP: return __dmul_rn(kp.a2, exp_cr(-div_exact(fabs(d), kp.ell, kp.rell)));
    case HODLR_IMQ: {
      const double q = div_exact(d, kp.ell, kp.rell);
      return __ddiv_rn(kp.a2, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(q, q))));
    }
    case HODLR_RQ: {
      const double q = div_exact(d, kp.ell, kp.rell);
      return __dmul_rn(kp.a2, pow(__dadd_rn(1.0, __dmul_rn(q, q)), -kp.alpha));
    }
    case HODLR_MQ: {
      const double q = div_exact(d, kp.ell, kp.rell);
      return __dmul_rn(kp.a2, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(q, q))));
    }
    case HODLR_BIHARM: {
      const double q = div_exact(fabs(d), kp.ell, kp.rell);
      return q == 0.0 ? 0.0 : __dmul_rn(__dmul_rn(kp.a2, __dmul_rn(q, q)), log(q));
    }
    case HODLR_MATERN32: {
      const double s = div_exact(__dmul_rn(kp.sq, fabs(d)), kp.ell, kp.rell);
      return __dmul_rn(__dmul_rn(kp.a2, __dadd_rn(1.0, s)), exp_cr(-s));
    }
    default: {                                   // HODLR_MATERN52
      const double s = div_exact(__dmul_rn(kp.sq, fabs(d)), kp.ell, kp.rell);
      const double p = __dadd_rn(__dadd_rn(1.0, s), __ddiv_rn(__dmul_rn(s, s), 3.0));
      return __dmul_rn(__dmul_rn(kp.a2, p), exp_cr(-s));
    }
  }
}
__device__ __forceinline__ double kval_o_se(const KParams &kp, double d) {
  return __dmul_rn(kp.a2, exp_cr(-div_exact(__dmul_rn(d, d), kp.c2, kp.rc2)));
}
__device__ __forceinline__ double kval_o_m52(const KParams &kp, double d) {   // kval_o's Matern-5/2 branch
  const double s = div_exact(__dmul_rn(kp.sq, fabs(d)), kp.ell, kp.rell);
  const double p = __dadd_rn(__dadd_rn(1.0, s), __ddiv_rn(__dmul_rn(s, s), 3.0));
  return __dmul_rn(__dmul_rn(kp.a2, p), exp_cr(-s));
}
template <int KV> __device__ __forceinline__ double kval_ot(const KParams &kp, double d) {
  if (KV == KV_SE) return kval_o_se(kp, d);
  if (KV == KV_M52) return kval_o_m52(kp, d);
  return kval_o(kp, d);
}

// ----------------------------------------------------------------------------------------------
// NEXT-3: d-dimensional points ("points in one, two, or three dimensions", Table II; DESIGN.md
// R19).  Launches on such a handle are the KV_ND instantiations: entries are the Table I functions of the Euclidean
// distance, from the squared distance r2 = sum_k (x_ik - x_jk)^2 summed in coordinate order (SE uses r2 directly,
// the others r = sqrt(r2)), in the oracle's operation order (its oracle_kernel_r2).  Coordinate-major points:
// a warp reading consecutive sorted points reads consecutive addresses of each coordinate row.
// ----------------------------------------------------------------------------------------------
constexpr int KV_ND = -2;
__device__ __forceinline__ double pt_r2(const KParams &kp, const double *xs, long long i, long long j) {
  double r2 = 0.0;
  for (int k = 0; k < kp.dim; k++) {
    const double d = __dsub_rn(xs[k * kp.ldp + i], xs[k * kp.ldp + j]);
    r2 = __dadd_rn(r2, __dmul_rn(d, d));
  }
  return r2;
}
__device__ __forceinline__ double kval_nd(const KParams &kp, const double *xs, long long i, long long j) {
  const double r2 = pt_r2(kp, xs, i, j);
  if (kp.kern == HODLR_SE) return __dmul_rn(kp.a2, exp_cr(-div_exact(r2, kp.c2, kp.rc2)));
  return kval_o(kp, __dsqrt_rn(r2));
}
// the same entry for the leaf blocks and the forward apply (no pivot decision depends on it): kval's fast exp / log
__device__ __forceinline__ double kval_nd_fast(const KParams &kp, const double *xs, long long i, long long j) {
  double r2 = 0.0;
  for (int k = 0; k < kp.dim; k++) { const double d = xs[k * kp.ldp + i] - xs[k * kp.ldp + j]; r2 = fma(d, d, r2); }
  if (kp.kern == HODLR_SE) return kp.a2 * exp(-r2 * kp.c);
  return kval(kp, sqrt(r2));
}
// the launch family of a handle: KV_ND for d > 1, else the kernel family's specialisation
static inline int kv_of_kp(const KParams &kp) { return kp.dim > 1 ? KV_ND : kv_of(kp.kern); }
// sorted points i and j coincide (every coordinate equal; 1-D: xs[i] == xs[j]) -- the duplicate-row rule (R2)
__device__ __forceinline__ bool pt_eq(const KParams &kp, const double *xs, long long i, long long j) {
  for (int k = 0; k < kp.dim; k++)
    if (xs[k * kp.ldp + i] != xs[k * kp.ldp + j]) return false;
  return true;
}

// ----------------------------------------------------------------------------------------------
// Storage helpers shared by the factor and solve kernels.
//   Leaf factors: per leaf, T = ceil(leaf_max / 8) tile rows; lower 8x8 tiles of L in "fragment order"
//   (tile (I,J), I >= J, at tix(I,J)*64; element (r,c) at fo(r,c)), followed by the T inverse diagonal
//   tiles Linv(b) at (NTILE + b)*64.  Padding rows beyond the leaf size are identity.
//   Pi: packed lower triangle, row-major: (a, b), a >= b, at a(a+1)/2 + b.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ int tix(int I, int J) { return I * (I + 1) / 2 + J; }
__device__ __forceinline__ int fo(int r, int c) { return (c >> 2) * 32 + r * 4 + (c & 3); }
__device__ __forceinline__ long long pk(long long a, long long b) { return a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a; }

// argmax with ties -> smallest index; (abs, idx) with idx < 0 meaning "no candidate"
__device__ __forceinline__ bool amax_better(double a1, long long i1, double a2, long long i2) {
  if (i2 < 0) return false;
  if (i1 < 0) return true;
  if (a2 > a1) return true;
  if (a2 == a1 && i2 < i1) return true;
  return false;
}
