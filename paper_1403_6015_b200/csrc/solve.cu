// solve.cu -- G11/G12: x = C^{-1} y by applying the inverse factors (eq-fac)
// in projected form:
//   up   (leaves)  w_l = A_l^{-1} b_l,  g_l = E_l^T w_l,  h_l = b_l . w_l            (k_leaf_up)
//   up   (node c)  t_c = S_c^{-1} [g_c2[s]; g_c1[s]]
//                  g_c = g_c1[a] + g_c2[a] - B_c[r:]^T t_c[:r] - B_c[:r]^T t_c[r:]
//                  h_c = h_c1 + h_c2 - g_c1[s] . t_c[:r] - g_c2[s] . t_c[r:]          (k_tree_up)
//   down (node c)  f = t_c + T_c w_c;  w_c1 = [w_c, -f[:r]],  w_c2 = [w_c, -f[r:]]   (k_tree_down)
//   down (leaves)  x_l = A_l^{-1} (b_l + E_l w_l)                                   (k_leaf_down)
// h_root = y^T C^{-1} y gives the log-likelihood without the down pass (eq. 1).
// Leaf passes use the stored X = L^{-1} (one CTA per leaf, two triangular matrix-vector products);
// tree passes one warp per node (t_c by S_c^{-1} + 2 compensated refinement steps).
#include "hodlr_internal.cuh"

namespace {

constexpr int ST = 256;          // threads per CTA (8 warps)
constexpr int NWS = ST / 32;


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
  double *xsorted;  // sharded solve: this rank's solution rows in sorted order (NULL on one GPU)
  int *flags;
  long long leaf0;  // first leaf of this rank
};

// ---------------------------------------------------------------------------------------------
// Leaf passes: one CTA (256 threads) per leaf; X = L^{-1} (fragment-order lower tiles) staged in shared
// memory with 16-byte cp.async when it fits (T <= 16), read from global otherwise.
//   u = X b   (row i: sum_{j <= i} X_ij b_j)        v = X^T u   (column j: sum_{i >= j} X_ij u_i)
// so v = A_l^{-1} b with two parallel triangular matrix-vector products.
// ---------------------------------------------------------------------------------------------

// out = X in (lower) for rows < R = 8T; 2 threads per row (interleaved tile columns), partials in red[].
__device__ void tri_mv(const double *X, int T, const double *in, double *out, double *red) {
  const int t = threadIdx.x, R = 8 * T, NT = blockDim.x;
  for (int w = t; w < 2 * R; w += NT) {
    const int i = w % R, h = w / R, I = i >> 3, r = i & 7;
    double s = 0.0;
    for (int k = h; k <= I; k += 2) {
      const double *tl = X + tix(I, k) * 64;
#pragma unroll
      for (int cc = 0; cc < 8; cc++) s = fma(tl[fo(r, cc)], in[8 * k + cc], s);
    }
    red[w] = s;
  }
  __syncthreads();
  for (int i = t; i < R; i += NT) out[i] = red[i] + red[R + i];
  __syncthreads();
}

// out = X^T in for columns < R.
__device__ void tri_mvt(const double *X, int T, const double *in, double *out, double *red) {
  const int t = threadIdx.x, R = 8 * T, NT = blockDim.x;
  for (int w = t; w < 2 * R; w += NT) {
    const int j = w % R, h = w / R, J = j >> 3, cc = j & 7;
    double s = 0.0;
    for (int I = J + h; I < T; I += 2) {
      const double *tl = X + tix(I, J) * 64;
#pragma unroll
      for (int r = 0; r < 8; r++) s = fma(tl[fo(r, cc)], in[8 * I + r], s);
    }
    red[w] = s;
  }
  __syncthreads();
  for (int j = t; j < R; j += NT) out[j] = red[j] + red[R + j];
  __syncthreads();
}

__device__ __forceinline__ int leaf_colsrc(const SolveCtx &c, long long id, int q) {
  if (q >= c.K) return -1;
  int e = 1;
  while (c.dt->Kdim[e] <= q) e++;
  const int qq = q - c.dt->Kdim[e - 1];
  const long long b = ((id + 1) >> (c.kappa - e + 1)) - 1;     // ancestor at depth e - 1 (heap order)
  return qq < c.rank[b] ? (int)(c.dt->colbase[e] + qq) : -1;
}

constexpr int VMAX = 8 * 32;      // leaf rows handled (leaf_max < 2 leaf <= 256)
constexpr int LT = 512;           // threads per leaf CTA

__device__ __forceinline__ void cp16(double *dst, const double *src) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(src));
}
__device__ __forceinline__ void cp8(double *dst, const double *src) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" :: "r"(sa), "l"(src));
}

// Stage X = L^{-1} (tiles) and the ancestor panel E_l (K columns x R rows, column-major, zero beyond each
// block's rank) of one leaf into shared memory with cp.async; all bytes of the leaf in flight at once.
__device__ void stage_leaf(const SolveCtx &c, long long leaf, long long id, long long lo, int m, int R,
                           const int *colsrc, double *sX, double *sE) {
  const int t = threadIdx.x, NT = blockDim.x;
  const double *Xg = c.Lf + leaf * c.lstride;
  const int nx2 = (c.T * (c.T + 1) / 2) * 32;
  for (int p = t; p < nx2; p += NT) cp16(sX + 2 * p, Xg + 2 * p);
  const bool al16 = ((c.n | lo) & 1) == 0;
  if (al16) {
    const int R2 = R / 2;
    for (int p = t; p < c.K * R2; p += NT) {
      const int q = p / R2, i = 2 * (p - q * R2);
      const int src = colsrc[q];
      double *dst = sE + q * R + i;
      if (src >= 0 && i + 1 < m) cp16(dst, c.Xh + (long long)src * c.n + lo + i);
      else { dst[0] = (src >= 0 && i < m) ? c.Xh[(long long)src * c.n + lo + i] : 0.0; dst[1] = 0.0; }
    }
  } else {
    for (int p = t; p < c.K * R; p += NT) {
      const int q = p / R, i = p - q * R;
      const int src = colsrc[q];
      double *dst = sE + q * R + i;
      if (src >= 0 && i < m) cp8(dst, c.Xh + (long long)src * c.n + lo + i); else *dst = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// up: v = A_l^{-1} b, g_l = E_l^T v, h_l = b . v
__global__ void __launch_bounds__(LT, 1) k_leaf_up(SolveCtx c) {
  extern __shared__ double sm[];
  __shared__ double sb[VMAX], su[VMAX], red[2 * VMAX];
  __shared__ int colsrc[1024];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, NW = LT / 32;
  const long long leaf = c.leaf0 + blockIdx.x;
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo), R = 8 * c.T, K = c.K;
  double *sX = sm, *sE = sm + 64 * (c.T * (c.T + 1) / 2);
  for (int q = t; q < K; q += LT) colsrc[q] = leaf_colsrc(c, id, q);
  bool bad = false;
  for (int i = t; i < R; i += LT) {
    const double v = i < m ? c.y[c.perm[lo + i]] : 0.0;
    if (!isfinite(v)) bad = true;
    sb[i] = v;
  }
  if (bad) atomicOr(&c.flags[3], 1);
  __syncthreads();
  stage_leaf(c, leaf, id, lo, m, R, colsrc, sX, sE);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  tri_mv(sX, c.T, sb, su, red);           // u = X b
  tri_mvt(sX, c.T, su, su, red);          // v = X^T u  (in place: tri_mvt reads su fully before its barrier)
  double hs = 0.0;
  for (int i = t; i < m; i += LT) hs += sb[i] * su[i];
  hs = warp_sum(hs);
  if (lane == 0) red[warp] = hs;
  double *g = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)K;
  for (int q = warp; q < K; q += NW) {    // g = E^T v: warp per column, lanes over rows
    const double *e = sE + q * R;
    double s2 = 0.0;
    for (int i = lane; i < R; i += 32) s2 = fma(e[i], su[i], s2);
    s2 = warp_sum(s2);
    if (lane == 0) g[q] = s2;
  }
  __syncthreads();
  if (t == 0) {
    double h = 0.0;
    for (int w = 0; w < NW; w++) h += red[w];
    c.hv[2 * id] = h; c.hv[2 * id + 1] = 0.0;
  }
}

// down: x_l = A_l^{-1} (b_l + E_l w_l)
__global__ void __launch_bounds__(LT, 1) k_leaf_down(SolveCtx c) {
  extern __shared__ double sm[];
  __shared__ double sb[VMAX], su[VMAX], red[2 * VMAX];
  __shared__ int colsrc[1024];
  __shared__ double sw[1024];
  __shared__ double part4[4 * VMAX];
  const int t = threadIdx.x;
  const long long leaf = c.leaf0 + blockIdx.x;
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo), R = 8 * c.T, K = c.K;
  double *sX = sm, *sE = sm + 64 * (c.T * (c.T + 1) / 2);
  const double *w = c.V + c.dt->nodeV[c.kappa] + leaf * (long long)K;
  for (int q = t; q < K; q += LT) { colsrc[q] = leaf_colsrc(c, id, q); sw[q] = w[q]; }
  __syncthreads();
  stage_leaf(c, leaf, id, lo, m, R, colsrc, sX, sE);
  for (int i = t; i < R; i += LT) sb[i] = i < m ? c.y[c.perm[lo + i]] : 0.0;
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // b + E w: 4 threads per row (quarters of the columns), partials combined in a fixed order
  for (int w4 = t; w4 < 4 * R; w4 += LT) {
    const int i = w4 % R, h = w4 / R;
    const int q0 = (K * h) / 4, q1 = (K * (h + 1)) / 4;
    double s2 = 0.0;
    for (int q = q0; q < q1; q++) s2 = fma(sE[q * R + i], sw[q], s2);
    part4[w4] = s2;
  }
  __syncthreads();
  for (int i = t; i < R; i += LT) sb[i] += (part4[i] + part4[R + i]) + (part4[2 * R + i] + part4[3 * R + i]);
  __syncthreads();
  tri_mv(sX, c.T, sb, su, red);
  tri_mvt(sX, c.T, su, sb, red);
  if (c.xsorted) for (int i = t; i < m; i += LT) c.xsorted[lo + i] = sb[i];
  else for (int i = t; i < m; i += LT) c.x[c.perm[lo + i]] = sb[i];
}

// sharded solve: x[perm[row_lo_r + i]] = slice_r[i] for every rank's slice of the gathered solution
__global__ void k_unshard(const double *gathered, const long long *rowlo, int nranks, long long rows_max, long long n,
                          const long long *perm, double *x) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)nranks * rows_max) return;
  const int r = (int)(e / rows_max);
  const long long i = e - (long long)r * rows_max;
  const long long lo = rowlo[r], hi = r + 1 < nranks ? rowlo[r + 1] : n;
  if (lo + i < hi) x[perm[lo + i]] = gathered[e];
}

__global__ void k_pack_rows(const double *xsorted, long long lo, long long m, double *send) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < m) send[i] = xsorted[lo + i];
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

__global__ void __launch_bounds__(ST) k_tree_up(SolveCtx c, int d, long long i0, long long cnt) {
  extern __shared__ double dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((long long)blockIdx.x * NWS + wid >= cnt) return;
  const long long i = i0 + (long long)blockIdx.x * NWS + wid;
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

__global__ void __launch_bounds__(ST) k_tree_down(SolveCtx c, int d, long long i0, long long cnt) {
  __shared__ double sf[NWS][QMAX];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((long long)blockIdx.x * NWS + wid >= cnt) return;
  const long long i = i0 + (long long)blockIdx.x * NWS + wid;
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
  if (h->leaf_max > VMAX || dt.Kdim[kappa] > 1024)
    return hodlr_set_error(HODLR_EINVAL, "solve: leaf size %d > %d or K > 1024", h->leaf_max, VMAX);
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
  long long lcnt;
  hodlr_own_nodes(h, kappa, &c.leaf0, &lcnt);
  c.xsorted = nullptr;
  if (h->nranks > 1 && !up_only) {
    if (!h->xshard) {
      h->xshard = (double *)hodlr_dalloc(h, sizeof(double) * ((size_t)h->n + (size_t)h->rows_max * (h->nranks + 1)));
      if (!h->xshard) return hodlr_set_error(HODLR_ENOMEM, "solve: device allocation failed");
    }
    c.xsorted = h->xshard;
  }
  const int lgrid = (int)lcnt;
  const int R = 8 * h->ltiles;
  // X tiles + E panel in shared memory
  const size_t lsm = sizeof(double) * (64 * (size_t)(h->ltiles * (h->ltiles + 1) / 2) + (size_t)c.K * R);
  int maxsm = 0;
  HCUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  if (lsm + 32 * 1024 > (size_t)maxsm)
    return hodlr_set_error(HODLR_EINVAL, "solve: leaf panel (%d x %d) exceeds shared memory", R, c.K);
  static size_t lattr = 0;
  if (lsm > lattr) {
    HCUDA(cudaFuncSetAttribute(k_leaf_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    HCUDA(cudaFuncSetAttribute(k_leaf_down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    lattr = lsm;
  }
  ph_begin(h, PH_SLEAF_UP);
  k_leaf_up<<<lgrid, LT, lsm, h->st>>>(c);
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
    if (d + 1 == h->tsplit && h->nranks > 1) {   // projections g and h of all depth-t subtree roots
      const long long Kt = dt.Kdim[d + 1];
      double *gb = h->Vpool + dt.nodeV[d + 1];
      hodlr_status xs = hodlr_allgather(h, gb + h->grank * Kt, gb, sizeof(double) * (Kt > 0 ? Kt : 1));
      if (xs != HODLR_OK) return xs;
      double *hb = h->hvec + 2 * ((1LL << (d + 1)) - 1);
      xs = hodlr_allgather(h, hb + 2 * h->grank, hb, sizeof(double) * 2);
      if (xs != HODLR_OK) return xs;
    }
    long long i0, cnt;
    hodlr_own_nodes(h, d, &i0, &cnt);
    const size_t q = 2 * (size_t)dt.rdep[d + 1];
    k_tree_up<<<(int)((cnt + NWS - 1) / NWS), ST, sizeof(double) * NWS * (2 * q * q + 5 * q), h->st>>>(c, d, i0, cnt);
    HLAUNCH(h, "k_tree_up");
  }
  if (up_only) { ph_end(h, PH_STREE); return HODLR_OK; }
  for (int d = 0; d < kappa; d++) {
    long long i0, cnt;
    hodlr_own_nodes(h, d, &i0, &cnt);
    k_tree_down<<<(int)((cnt + NWS - 1) / NWS), ST, 0, h->st>>>(c, d, i0, cnt);
    HLAUNCH(h, "k_tree_down");
  }
  ph_end(h, PH_STREE);
  ph_begin(h, PH_SLEAF_DOWN);
  k_leaf_down<<<lgrid, LT, lsm, h->st>>>(c);
  HLAUNCH(h, "k_leaf_down");
  if (h->nranks > 1) {            // every rank returns the full solution: allgather the sorted row slices
    const long long id = (1LL << h->tsplit) - 1 + h->grank;
    const long long rlo = h->h_lo[id], rm = h->h_hi[id] - rlo;
    double *send = h->xshard + h->n, *recv = send + h->rows_max;
    k_pack_rows<<<(int)((rm + 255) / 256), 256, 0, h->st>>>(h->xshard, rlo, rm, send);
    HLAUNCH(h, "k_pack_rows");
    hodlr_status xs = hodlr_allgather(h, send, recv, sizeof(double) * h->rows_max);
    if (xs != HODLR_OK) return xs;
    const long long tot = (long long)h->nranks * h->rows_max;
    k_unshard<<<(int)((tot + 255) / 256), 256, 0, h->st>>>(recv, h->d_rowlo, h->nranks, h->rows_max, h->n, h->perm, x);
    HLAUNCH(h, "k_unshard");
  }
  ph_end(h, PH_SLEAF_DOWN);
  return HODLR_OK;
}
