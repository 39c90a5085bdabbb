// solve.cu -- G11/G12: x = C^{-1} y by applying the inverse factors (eq-fac)
// in projected form:
//   up   (leaves)  w_l = A_l^{-1} b_l,  g_l = E_l^T w_l,  h_l = b_l . w_l            (k_leaf_up)
//   up   (node c)  t_c = S_c^{-1} [g_c2[s]; g_c1[s]]
//                  g_c = g_c1[a] + g_c2[a] - B_c[r:]^T t_c[:r] - B_c[:r]^T t_c[r:]
//                  h_c = h_c1 + h_c2 - g_c1[s] . t_c[:r] - g_c2[s] . t_c[r:]          (k_tree_up)
//   down (node c)  f = t_c + T_c w_c;  w_c1 = [w_c, -f[:r]],  w_c2 = [w_c, -f[r:]]   (k_tree_down)
//   down (leaves)  x_l = A_l^{-1} (b_l + E_l w_l)                                   (k_leaf_down)
// h_root = y^T C^{-1} y gives the log-likelihood without the down pass (eq. 1).
#include "hodlr_internal.cuh"

namespace {

constexpr int ST = 256;

__device__ __forceinline__ long long P(long long i, long long j) { return i * (i + 1) / 2 + j; }

struct SolveCtx {
  long long n, ninternal, nleaves;
  int kappa, K;
  const long long *lo, *hi, *perm;
  const double *Xh;
  const int *rank;
  const DepthTab *dt;
  const double *Lf; long long lstride;
  const double *Spool, *BTpool;
  double *V;        // per-level node vectors (g on the way up, w on the way down)
  double *Tv;       // per-node t (q doubles, depth-d offset nodeT[d])
  double *hv;       // per-node h = y_c^T K_cc^{-1} y_c as a double-double pair (heap id)
  const double *y;
  double *x;
  int *flags;
  int mmax;
};

// warp 0: solve L L^T w = b in place (packed lower row-major L in shared memory)
__device__ void chol_solve_warp(const double *L, double *b, long long m) {
  const int lane = threadIdx.x & 31;
  for (long long i = 0; i < m; i++) {
    double s = 0.0;
    for (long long j = lane; j < i; j += 32) s += L[P(i, j)] * b[j];
    s = warp_sum(s);
    if (lane == 0) b[i] = (b[i] - s) / L[P(i, i)];
    __syncwarp();
  }
  for (long long i = m - 1; i >= 0; i--) {
    double s = 0.0;
    for (long long k = i + 1 + lane; k < m; k += 32) s += L[P(k, i)] * b[k];
    s = warp_sum(s);
    if (lane == 0) b[i] = (b[i] - s) / L[P(i, i)];
    __syncwarp();
  }
}

__device__ void leaf_colmap(const SolveCtx &c, long long id, long long *colsrc) {
  long long a = id;
  for (int e = c.kappa; e >= 1; e--) {
    long long b = (a - 1) / 2;
    int rb = c.rank[b];
    for (int q = 0; q < c.dt->rdep[e]; q++) colsrc[c.dt->Kdim[e - 1] + q] = q < rb ? c.dt->colbase[e] + q : -1;
    a = b;
  }
}

__global__ void __launch_bounds__(ST) k_leaf_up(SolveCtx c) {
  extern __shared__ double sm[];
  __shared__ long long colsrc[1024];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long leaf = blockIdx.x, id = c.ninternal + leaf, lo = c.lo[id], m = c.hi[id] - lo;
  double *L = sm;                        // packed
  double *b = sm + c.lstride;            // m
  double *w = b + c.mmax;                // m
  const double *Lg = c.Lf + leaf * c.lstride;
  for (long long p = t; p < m * (m + 1) / 2; p += ST) L[p] = Lg[p];
  for (long long i = t; i < m; i += ST) {
    double v = c.y[c.perm[lo + i]];
    if (!isfinite(v)) atomicOr(&c.flags[3], 1);
    b[i] = v; w[i] = v;
  }
  if (t == 0) leaf_colmap(c, id, colsrc);
  __syncthreads();
  if (warp == 0) chol_solve_warp(L, w, m);
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
    for (long long i = lane; i < m; i += 32) s += b[i] * w[i];
    s = warp_sum(s);
    if (lane == 0) { c.hv[2 * id] = s; c.hv[2 * id + 1] = 0.0; }
  }
  double *g = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)c.K;
  for (int col = warp; col < c.K; col += ST / 32) {
    long long src = colsrc[col];
    double s = 0.0;
    if (src >= 0) for (long long i = lane; i < m; i += 32) s += c.Xh[src * c.n + lo + i] * w[i];
    s = warp_sum(s);
    if (lane == 0) g[col] = s;
  }
}

// t = S^{-1} rhs for one short vector: double solve + two refinement steps with a compensated
// residual; result as a double-double pair (th, tl).  Single thread.
__device__ void dd_small_solve(const double *S0, const double *LU, const double *pivd, int q,
                               double *th, double *tl, double *tmp) {
  const double *rhs = th;   // th holds the rhs on entry
  for (int a = 0; a < q; a++) { tmp[a] = rhs[a]; tl[a] = 0.0; }
  // tmp keeps the rhs; th <- LU^{-1} rhs
  for (int k = 0; k < q; k++) { int p = (int)pivd[k]; if (p != k) { double x = th[k]; th[k] = th[p]; th[p] = x; } }
  for (int a = 0; a < q; a++) { double s = th[a]; for (int k = 0; k < a; k++) s -= LU[a * q + k] * th[k]; th[a] = s; }
  for (int a = q - 1; a >= 0; a--) { double s = th[a]; for (int k = a + 1; k < q; k++) s -= LU[a * q + k] * th[k]; th[a] = s / LU[a * q + a]; }
  double res[2 * ACA_MAXCAP];
  for (int it = 0; it < 2; it++) {
    for (int a = 0; a < q; a++) {
      Acc2 A = acc2(tmp[a]);
      for (int k = 0; k < q; k++) acc_fma_dd(A, -S0[a * q + k], th[k], tl[k]);
      res[a] = acc_val(A);
    }
    for (int k = 0; k < q; k++) { int p = (int)pivd[k]; if (p != k) { double x = res[k]; res[k] = res[p]; res[p] = x; } }
    for (int a = 0; a < q; a++) { double s = res[a]; for (int k = 0; k < a; k++) s -= LU[a * q + k] * res[k]; res[a] = s; }
    for (int a = q - 1; a >= 0; a--) { double s = res[a]; for (int k = a + 1; k < q; k++) s -= LU[a * q + k] * res[k]; res[a] = s / LU[a * q + a]; }
    for (int a = 0; a < q; a++) tl[a] += res[a];
  }
}

__global__ void __launch_bounds__(ST) k_tree_up(SolveCtx c, int d) {
  __shared__ double th[2 * ACA_MAXCAP], tl[2 * ACA_MAXCAP], tmp[2 * ACA_MAXCAP];
  const int t = threadIdx.x;
  const long long i = blockIdx.x, node = (1LL << d) - 1 + i;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const double *g1 = c.V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  const double *g2 = g1 + K1;
  const double *S0 = c.Spool + c.dt->nodeS[d] + i * (long long)(2 * q * q + q);
  const double *LU = S0 + q * q;
  const double *pivd = LU + q * q;
  const double *B = c.BTpool + c.dt->nodeBT[d] + i * 3LL * q * Kd;
  if (t == 0) {
    for (int u = 0; u < r; u++) { th[u] = g2[Kd + u]; th[r + u] = g1[Kd + u]; }
    dd_small_solve(S0, LU, pivd, q, th, tl, tmp);
    Acc2 A = acc2(c.hv[2 * (2 * node + 1)]);
    acc_add_dd(A, c.hv[2 * (2 * node + 2)], c.hv[2 * (2 * node + 2) + 1]);
    A.c += c.hv[2 * (2 * node + 1) + 1];
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g1[Kd + u], th[u], tl[u]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g2[Kd + u], th[r + u], tl[r + u]);
    acc_dd(A, c.hv[2 * node], c.hv[2 * node + 1]);
  }
  __syncthreads();
  double *tg = c.Tv + c.dt->nodeT[d] + i * 2LL * q;
  for (int u = t; u < q; u += ST) { tg[u] = th[u]; tg[q + u] = tl[u]; }
  double *gc = c.V + c.dt->nodeV[d] + i * (long long)Kd;
  for (int a = t; a < Kd; a += ST) {
    Acc2 A = acc2(g1[a]);
    acc_add(A, g2[a]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)(r + u) * Kd + a], th[u], tl[u]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)u * Kd + a], th[r + u], tl[r + u]);
    gc[a] = acc_val(A);
  }
}

__global__ void __launch_bounds__(ST) k_tree_down(SolveCtx c, int d) {
  __shared__ double f[2 * ACA_MAXCAP];
  const int t = threadIdx.x;
  const long long i = blockIdx.x;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const double *wc = c.V + c.dt->nodeV[d] + i * (long long)Kd;
  const long long qK = (long long)q * Kd;
  const double *Th = c.BTpool + c.dt->nodeBT[d] + i * 3LL * qK + qK;
  const double *Tl = Th + qK;
  const double *tg = c.Tv + c.dt->nodeT[d] + i * 2LL * q;
  for (int u = t; u < q; u += ST) {
    Acc2 A = acc2(tg[u]);
    A.c += tg[q + u];
    for (int a = 0; a < Kd; a++) acc_fma_dd(A, wc[a], Th[(long long)u * Kd + a], Tl[(long long)u * Kd + a]);
    f[u] = acc_val(A);
  }
  __syncthreads();
  double *w1 = c.V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  double *w2 = w1 + K1;
  for (int a = t; a < Kd; a += ST) { w1[a] = wc[a]; w2[a] = wc[a]; }
  for (int u = t; u < r; u += ST) { w1[Kd + u] = -f[u]; w2[Kd + u] = -f[r + u]; }
}

__global__ void __launch_bounds__(ST) k_leaf_down(SolveCtx c) {
  extern __shared__ double sm[];
  __shared__ long long colsrc[1024];
  const int t = threadIdx.x, warp = t >> 5;
  const long long leaf = blockIdx.x, id = c.ninternal + leaf, lo = c.lo[id], m = c.hi[id] - lo;
  double *L = sm;
  double *v = sm + c.lstride;
  const double *Lg = c.Lf + leaf * c.lstride;
  for (long long p = t; p < m * (m + 1) / 2; p += ST) L[p] = Lg[p];
  if (t == 0) leaf_colmap(c, id, colsrc);
  __syncthreads();
  const double *w = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)c.K;
  for (long long i = t; i < m; i += ST) {
    double s = c.y[c.perm[lo + i]];
    for (int col = 0; col < c.K; col++) {
      long long src = colsrc[col];
      if (src >= 0) s += c.Xh[src * c.n + lo + i] * w[col];
    }
    v[i] = s;
  }
  __syncthreads();
  if (warp == 0) chol_solve_warp(L, v, m);
  __syncthreads();
  for (long long i = t; i < m; i += ST) c.x[c.perm[lo + i]] = v[i];
}

}  // namespace

// y, x: one column each (device).  up_only: stop after the up pass (h_root = y^T C^{-1} y in hvec[0]).
hodlr_status hodlr_solve_impl(hodlr_s *h, const double *y, double *x, bool up_only) {
  const int kappa = h->kappa;
  DepthTab &dt = h->dt;
  if (!h->Vpool) {
    long long vTot = 0, tTot = 0;
    for (int e = 0; e <= kappa; e++) { dt.nodeV[e] = vTot; vTot += (1LL << e) * (long long)dt.Kdim[e]; }
    for (int d = 0; d < kappa; d++) { dt.nodeT[d] = tTot; tTot += (1LL << d) * 4LL * dt.rdep[d + 1]; }
    h->Vpool = (double *)hodlr_dalloc(h, sizeof(double) * (vTot > 0 ? vTot : 1));
    h->Tvec = (double *)hodlr_dalloc(h, sizeof(double) * (tTot > 0 ? tTot : 1));
    h->hvec = (double *)hodlr_dalloc(h, sizeof(double) * 2 * h->nnodes);
    if (!h->Vpool || !h->Tvec || !h->hvec) return hodlr_set_error(HODLR_ENOMEM, "solve: device allocation failed");
    HCUDA(cudaMemcpyAsync(h->d_dt, &dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));
  }
  SolveCtx c;
  c.n = h->n; c.ninternal = h->ninternal; c.nleaves = h->nleaves; c.kappa = kappa; c.K = dt.Kdim[kappa];
  c.lo = h->lo; c.hi = h->hi; c.perm = h->perm; c.Xh = h->Xh; c.rank = h->rank; c.dt = h->d_dt;
  c.Lf = h->Lf; c.lstride = h->lstride; c.Spool = h->Spool; c.BTpool = h->BTpool;
  c.V = h->Vpool; c.Tv = h->Tvec; c.hv = h->hvec; c.y = y; c.x = x; c.flags = h->dflags; c.mmax = h->leaf_max;
  size_t smem_up = sizeof(double) * (h->lstride + 2LL * h->leaf_max);
  size_t smem_dn = sizeof(double) * (h->lstride + h->leaf_max);
  HCUDA(cudaFuncSetAttribute(k_leaf_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_up));
  HCUDA(cudaFuncSetAttribute(k_leaf_down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dn));
  ph_begin(h, PH_SLEAF_UP);
  k_leaf_up<<<(int)h->nleaves, ST, smem_up, h->st>>>(c);
  HLAUNCH(h, "k_leaf_up");
  ph_end(h, PH_SLEAF_UP);
  ph_begin(h, PH_STREE);
  for (int d = kappa - 1; d >= 0; d--) {
    k_tree_up<<<(int)(1LL << d), ST, 0, h->st>>>(c, d);
    HLAUNCH(h, "k_tree_up");
  }
  if (up_only) { ph_end(h, PH_STREE); return HODLR_OK; }
  for (int d = 0; d < kappa; d++) {
    k_tree_down<<<(int)(1LL << d), ST, 0, h->st>>>(c, d);
    HLAUNCH(h, "k_tree_down");
  }
  ph_end(h, PH_STREE);
  ph_begin(h, PH_SLEAF_DOWN);
  k_leaf_down<<<(int)h->nleaves, ST, smem_dn, h->st>>>(c);
  HLAUNCH(h, "k_leaf_down");
  ph_end(h, PH_SLEAF_DOWN);
  return HODLR_OK;
}
