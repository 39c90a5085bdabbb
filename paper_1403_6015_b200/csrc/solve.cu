// solve.cu -- G11/G12: x = C^{-1} y by applying the inverse factors (eq-fac)
// in projected form:
//   up   (leaves)  w_l = A_l^{-1} b_l,  g_l = E_l^T w_l,  h_l = b_l . w_l            (k_leaf_up)
//   up   (node c)  t_c = S_c^{-1} [g_c2[s]; g_c1[s]]
//                  g_c = g_c1[a] + g_c2[a] - B_c[r:]^T t_c[:r] - B_c[:r]^T t_c[r:]
//                  h_c = h_c1 + h_c2 - g_c1[s] . t_c[:r] - g_c2[s] . t_c[r:]          (k_tree_up)
//   down (node c)  f = t_c + T_c w_c;  w_c1 = [w_c, -f[:r]],  w_c2 = [w_c, -f[r:]]   (k_tree_down)
//   down (leaves)  x_l = A_l^{-1} (b_l + E_l w_l)                                   (k_leaf_down)
// h_root = y^T C^{-1} y gives the log-likelihood without the down pass (eq. 1).
// Leaf triangular solves are blocked over 8-row tiles with the stored inverse diagonal tiles; one warp
// per leaf, one warp per tree node (t_c by a double solve + 2 compensated refinement steps).
#include "hodlr_internal.cuh"

namespace {

constexpr int ST = 256;          // threads per CTA (8 warps)
constexpr int NWS = ST / 32;
constexpr int RPL = 8;           // rows per lane: leaves up to 256 rows

struct SolveCtx {
  long long n, ninternal, nleaves;
  int kappa, K, T;
  const long long *lo, *hi, *perm;
  const double *Xh;
  const int *rank;
  const DepthTab *dt;
  const double *Lf; long long lstride;
  const double *Spool, *BTpool;
  double *V;        // per-level node vectors (g on the way up, w on the way down)
  double *Tv;       // per-node t_c (q hi, q lo doubles; depth-d offset nodeT[d])
  double *hv;       // per-node h = y_c^T K_cc^{-1} y_c as a double-double pair (heap id)
  const double *y;
  double *x;
  int *flags;
};

// Rows of the leaf owned by this lane: i = lane + 32 s.  v[s] holds the working vector.
// Forward: v <- L^{-1} v with L in fragment-order tiles (Lg) and the inverse diagonal tiles (Li).
__device__ __forceinline__ void tile_fwd(const double *Lg, const double *Li, int T, double v[RPL], int lane) {
  for (int b = 0; b < T; b++) {
    const int rb = 8 * b;
    double vb[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int row = rb + k, s = row >> 5;
      double val = 0.0;
#pragma unroll
      for (int ss = 0; ss < RPL; ss++) if (ss == s) val = v[ss];
      vb[k] = __shfl_sync(0xffffffffu, val, row & 31);
    }
    double z[8];                       // z_b = Linv(b) v_b
#pragma unroll
    for (int r = 0; r < 8; r++) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k <= r; k++) acc += Li[b * 64 + fo(r, k)] * vb[k];
      z[r] = acc;
    }
#pragma unroll
    for (int s = 0; s < RPL; s++) {
      const int i = lane + 32 * s;
      if (i >= 8 * T) break;
      if (i >= rb && i < rb + 8) {
#pragma unroll
        for (int r = 0; r < 8; r++) if (i == rb + r) v[s] = z[r];
      } else if (i >= rb + 8) {        // v_i -= L(I, b) z
        const double *t = Lg + tix(i >> 3, b) * 64;
        const int r = i & 7;
        double acc = v[s];
#pragma unroll
        for (int k = 0; k < 8; k++) acc -= t[fo(r, k)] * z[k];
        v[s] = acc;
      }
    }
  }
}

// Backward: v <- L^{-T} v.
__device__ __forceinline__ void tile_bwd(const double *Lg, const double *Li, int T, double v[RPL], int lane) {
  for (int b = T - 1; b >= 0; b--) {
    const int rb = 8 * b;
    double vb[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int row = rb + k, s = row >> 5;
      double val = 0.0;
#pragma unroll
      for (int ss = 0; ss < RPL; ss++) if (ss == s) val = v[ss];
      vb[k] = __shfl_sync(0xffffffffu, val, row & 31);
    }
    double z[8];                       // w_b = Linv(b)^T v_b
#pragma unroll
    for (int r = 0; r < 8; r++) {
      double acc = 0.0;
#pragma unroll
      for (int k = r; k < 8; k++) acc += Li[b * 64 + fo(k, r)] * vb[k];
      z[r] = acc;
    }
#pragma unroll
    for (int s = 0; s < RPL; s++) {
      const int j = lane + 32 * s;
      if (j >= 8 * T) break;
      if (j >= rb && j < rb + 8) {
#pragma unroll
        for (int r = 0; r < 8; r++) if (j == rb + r) v[s] = z[r];
      } else if (j < rb) {             // v_j -= sum_r L(b, J)[r][j%8] z_r
        const double *t = Lg + tix(b, j >> 3) * 64;
        const int cj = j & 7;
        double acc = v[s];
#pragma unroll
        for (int r = 0; r < 8; r++) acc -= t[fo(r, cj)] * z[r];
        v[s] = acc;
      }
    }
  }
}

__device__ void leaf_colmap(const SolveCtx &c, long long id, int *colsrc, int lane) {
  if (lane == 0) {
    long long a = id;
    for (int e = c.kappa; e >= 1; e--) {
      long long b = (a - 1) / 2;
      int rb = c.rank[b];
      for (int q = 0; q < c.dt->rdep[e]; q++) colsrc[c.dt->Kdim[e - 1] + q] = q < rb ? (int)(c.dt->colbase[e] + q) : -1;
      a = b;
    }
  }
  __syncwarp();
}

// one warp per leaf
__global__ void __launch_bounds__(ST) k_leaf_up(SolveCtx c) {
  __shared__ int colsrc_s[NWS][1024];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long leaf = (long long)blockIdx.x * NWS + wid;
  if (leaf >= c.nleaves) return;
  int *colsrc = colsrc_s[wid];
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  const double *Lg = c.Lf + leaf * c.lstride;
  const double *Li = Lg + (long long)(c.T * (c.T + 1) / 2) * 64;
  double b[RPL], v[RPL];
  bool bad = false;
#pragma unroll
  for (int s = 0; s < RPL; s++) {
    const int i = lane + 32 * s;
    b[s] = i < m ? c.y[c.perm[lo + i]] : 0.0;
    if (!isfinite(b[s])) bad = true;
    v[s] = b[s];
  }
  if (bad) atomicOr(&c.flags[3], 1);
  leaf_colmap(c, id, colsrc, lane);
  tile_fwd(Lg, Li, c.T, v, lane);
  tile_bwd(Lg, Li, c.T, v, lane);          // v = A^{-1} b
  double hs = 0.0;
#pragma unroll
  for (int s = 0; s < RPL; s++) hs += b[s] * v[s];
  hs = warp_sum(hs);
  if (lane == 0) { c.hv[2 * id] = hs; c.hv[2 * id + 1] = 0.0; }
  double *g = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)c.K;
  for (int col = 0; col < c.K; col++) {    // g = E^T w
    const long long src = colsrc[col];
    double s = 0.0;
    if (src >= 0) {
      const double *e = c.Xh + src * c.n + lo;
#pragma unroll
      for (int ss = 0; ss < RPL; ss++) { const int i = lane + 32 * ss; if (i < m) s += e[i] * v[ss]; }
    }
    s = warp_sum(s);
    if (lane == 0) g[col] = s;
  }
}

__global__ void __launch_bounds__(ST) k_leaf_down(SolveCtx c) {
  __shared__ int colsrc_s[NWS][1024];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long leaf = (long long)blockIdx.x * NWS + wid;
  if (leaf >= c.nleaves) return;
  int *colsrc = colsrc_s[wid];
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  const double *Lg = c.Lf + leaf * c.lstride;
  const double *Li = Lg + (long long)(c.T * (c.T + 1) / 2) * 64;
  leaf_colmap(c, id, colsrc, lane);
  const double *w = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)c.K;
  double v[RPL];
#pragma unroll
  for (int s = 0; s < RPL; s++) {
    const int i = lane + 32 * s;
    v[s] = i < m ? c.y[c.perm[lo + i]] : 0.0;
  }
  for (int col = 0; col < c.K; col++) {    // v = b + E w
    const long long src = colsrc[col];
    if (src < 0) continue;
    const double wc = w[col];
    const double *e = c.Xh + src * c.n + lo;
#pragma unroll
    for (int s = 0; s < RPL; s++) { const int i = lane + 32 * s; if (i < m) v[s] += e[i] * wc; }
  }
  tile_fwd(Lg, Li, c.T, v, lane);
  tile_bwd(Lg, Li, c.T, v, lane);
#pragma unroll
  for (int s = 0; s < RPL; s++) {
    const int i = lane + 32 * s;
    if (i < m) c.x[c.perm[lo + i]] = v[s];
  }
}

// ---------------------------------------------------------------------------------------------
// Tree passes: one warp per node.  Per-warp shared scratch for the short vectors.
// ---------------------------------------------------------------------------------------------
constexpr int QMAX = 2 * ACA_MAXCAP;

// t = S^{-1} rhs as (th, tl): explicit inverse S^{-1} (from the factor phase) + 2 refinement steps with
// compensated residuals.  One warp; all vectors in shared memory.
__device__ void dd_solve_warp(const double *S0, const double *Si, int q, const double *rhs, double *th, double *tl,
                              double *tmp, int lane) {
  for (int a = lane; a < q; a += 32) {
    double s = 0.0;
    for (int j = 0; j < q; j++) s = fma(Si[a * q + j], rhs[j], s);
    th[a] = s; tl[a] = 0.0;
  }
  __syncwarp();
  for (int it = 0; it < 2; it++) {
    for (int a = lane; a < q; a += 32) {
      Acc2 A = acc2(rhs[a]);
      for (int k = 0; k < q; k++) acc_fma_dd(A, -S0[a * q + k], th[k], tl[k]);
      tmp[a] = acc_val(A);
    }
    __syncwarp();
    for (int a = lane; a < q; a += 32) {
      double s = 0.0;
      for (int j = 0; j < q; j++) s = fma(Si[a * q + j], tmp[j], s);
      tl[a] += s;
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(ST) k_tree_up(SolveCtx c, int d) {
  extern __shared__ double dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * NWS + wid;
  if (i >= (1LL << d)) return;
  const long long node = (1LL << d) - 1 + i;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const double *g1 = c.V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  const double *g2 = g1 + K1;
  const double *Sg = c.Spool + c.dt->nodeS[d] + i * (long long)(2 * q * q + q);
  const double *B = c.BTpool + c.dt->nodeBT[d] + i * 3LL * q * Kd;
  // per-warp staging: S0, LU, pivots, rhs, th, tl, tmp (global latency stays out of the sequential solves)
  double *S0 = dsm + (long long)wid * (2 * q * q + 5 * q);
  double *Si = S0 + q * q, *rhs = Si + q * q + q, *th = rhs + q, *tl = th + q, *tmp = tl + q;
  for (int p = lane; p < 2 * q * q + q; p += 32) S0[p] = Sg[p];
  for (int u = lane; u < r; u += 32) { rhs[u] = g2[Kd + u]; rhs[r + u] = g1[Kd + u]; }
  __syncwarp();
  dd_solve_warp(S0, Si, q, rhs, th, tl, tmp, lane);
  double *tg = c.Tv + c.dt->nodeT[d] + i * 2LL * q;
  for (int u = lane; u < q; u += 32) { tg[u] = th[u]; tg[q + u] = tl[u]; }
  if (lane == 0) {
    Acc2 A = acc2(c.hv[2 * (2 * node + 1)]);
    acc_add_dd(A, c.hv[2 * (2 * node + 2)], c.hv[2 * (2 * node + 2) + 1]);
    A.c += c.hv[2 * (2 * node + 1) + 1];
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g1[Kd + u], th[u], tl[u]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g2[Kd + u], th[r + u], tl[r + u]);
    acc_dd(A, c.hv[2 * node], c.hv[2 * node + 1]);
  }
  double *gc = c.V + c.dt->nodeV[d] + i * (long long)Kd;
  for (int a = lane; a < Kd; a += 32) {
    Acc2 A = acc2(g1[a]);
    acc_add(A, g2[a]);
#pragma unroll 4
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)(r + u) * Kd + a], th[u], tl[u]);
#pragma unroll 4
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)u * Kd + a], th[r + u], tl[r + u]);
    gc[a] = acc_val(A);
  }
}

__global__ void __launch_bounds__(ST) k_tree_down(SolveCtx c, int d) {
  __shared__ double sf[NWS][QMAX];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * NWS + wid;
  if (i >= (1LL << d)) return;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const double *wc = c.V + c.dt->nodeV[d] + i * (long long)Kd;
  const long long qK = (long long)q * Kd;
  const double *Th = c.BTpool + c.dt->nodeBT[d] + i * 3LL * qK + qK;
  const double *Tl = Th + qK;
  const double *tg = c.Tv + c.dt->nodeT[d] + i * 2LL * q;
  double *f = sf[wid];
  for (int u = lane; u < q; u += 32) {
    Acc2 A = acc2(tg[u]);
    A.c += tg[q + u];
#pragma unroll 8
    for (int a = 0; a < Kd; a++) acc_fma_dd(A, wc[a], Th[(long long)u * Kd + a], Tl[(long long)u * Kd + a]);
    f[u] = acc_val(A);
  }
  __syncwarp();
  double *w1 = c.V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  double *w2 = w1 + K1;
  for (int a = lane; a < Kd; a += 32) { const double v = wc[a]; w1[a] = v; w2[a] = v; }
  for (int u = lane; u < r; u += 32) { w1[Kd + u] = -f[u]; w2[Kd + u] = -f[r + u]; }
}

}  // namespace

// y, x: one column each (device).  up_only: stop after the up pass (h_root = y^T C^{-1} y in hvec[0]).
hodlr_status hodlr_solve_impl(hodlr_s *h, const double *y, double *x, bool up_only) {
  const int kappa = h->kappa;
  DepthTab &dt = h->dt;
  if (h->leaf_max > 32 * RPL) return hodlr_set_error(HODLR_EINVAL, "solve: leaf size %d > %d", h->leaf_max, 32 * RPL);
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
  c.T = h->ltiles;
  c.lo = h->lo; c.hi = h->hi; c.perm = h->perm; c.Xh = h->Xh; c.rank = h->rank; c.dt = h->d_dt;
  c.Lf = h->Lf; c.lstride = h->lstride; c.Spool = h->Spool; c.BTpool = h->BTpool;
  c.V = h->Vpool; c.Tv = h->Tvec; c.hv = h->hvec; c.y = y; c.x = x; c.flags = h->dflags;
  const int lgrid = (int)((h->nleaves + NWS - 1) / NWS);
  ph_begin(h, PH_SLEAF_UP);
  k_leaf_up<<<lgrid, ST, 0, h->st>>>(c);
  HLAUNCH(h, "k_leaf_up");
  ph_end(h, PH_SLEAF_UP);
  ph_begin(h, PH_STREE);
  size_t up_smem_max = 0;
  for (int d = 0; d < kappa; d++) {
    const size_t q = 2 * (size_t)dt.rdep[d + 1];
    up_smem_max = std::max(up_smem_max, sizeof(double) * NWS * (2 * q * q + 5 * q));
  }
  if (kappa > 0) HCUDA(cudaFuncSetAttribute(k_tree_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)up_smem_max));
  for (int d = kappa - 1; d >= 0; d--) {
    const size_t q = 2 * (size_t)dt.rdep[d + 1];
    k_tree_up<<<(int)(((1LL << d) + NWS - 1) / NWS), ST, sizeof(double) * NWS * (2 * q * q + 5 * q), h->st>>>(c, d);
    HLAUNCH(h, "k_tree_up");
  }
  if (up_only) { ph_end(h, PH_STREE); return HODLR_OK; }
  for (int d = 0; d < kappa; d++) {
    k_tree_down<<<(int)(((1LL << d) + NWS - 1) / NWS), ST, 0, h->st>>>(c, d);
    HLAUNCH(h, "k_tree_down");
  }
  ph_end(h, PH_STREE);
  ph_begin(h, PH_SLEAF_DOWN);
  k_leaf_down<<<lgrid, ST, 0, h->st>>>(c);
  HLAUNCH(h, "k_leaf_down");
  ph_end(h, PH_SLEAF_DOWN);
  return HODLR_OK;
}
