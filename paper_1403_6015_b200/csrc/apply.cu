// apply.cu -- forward apply y = C~ x of the compressed operator (NEXT-1 of SURVEY 8(f): GP prediction
// ŷ = K(σ²I + K)⁻¹y and the sec. 5.6 RMSE experiment need the HODLR matvec).
//
// C~ is the operator the factorization inverts: the leaf diagonal blocks K_ll + σ²I (evaluated on the fly,
// Table I) plus, for every internal node c, the ACA factors K[c1,c2] ~ U V^T, K[c2,c1] ~ V U^T
// (sec. 3.1).  With E_l the ancestor panel of leaf l (columns of slot e = the left factor of
// its depth-e ancestor a: U' rows of a left child, V' rows of a right child):
//   leaf up   : ys_l = (K_ll + σ²I) x_l,   P_l = E_l^T x_l
//   tree up   : R_d[a] = R_{d+1}[a1] + R_{d+1}[a2] on the columns of slots <= d (R_kappa = P); t_a is the slot-d
//               part of R_d[a] = F_a^T x_a for a at depth d
//   leaf down : w_l[slot e] = t_{sibling of the depth-e ancestor}, ys_l += E_l w_l, y[perm] = ys
// (y[c1] += U (V^T x[c2]) and y[c2] += V (U^T x[c1]) for every block, as in the oracle's apply).  Fixed-order
// reductions: deterministic.
#include "hodlr_internal.cuh"
#include <algorithm>

namespace {

constexpr int AT = 128;              // threads per leaf CTA
constexpr int AVMAX = 256;           // leaf rows handled (leaf_max < 2 leaf <= 256)
constexpr int AKMAX = 1024;          // ancestor columns per leaf

struct ApplyCtx {
  KParams kp;
  long long n, ninternal, nleaves, ldx;
  int kappa, K;
  const double *xs;
  const long long *lo, *hi, *perm;
  const double *Xh;
  const int *rank;
  const DepthTab *dt;
  const double *x;          // original order
  double *y;                // original order
  double *ys;               // sorted-order accumulator (n)
  double *P;                // nleaves x K
  double *R;                // tree levels: depth d at Roff[d], 2^d x Kdim[d]
  long long Roff[HODLR_MAXDEPTH + 2];
  const KParams *kps; long long nseg;     // batched handle (kp_of), or NULL
};

// Leaf-local panel column q -> global Xh column (slot e = 1..kappa, qq-th factor of the depth-(e-1) ancestor
// block) or -1 beyond that block's rank.
__device__ __forceinline__ long long apply_colsrc(const ApplyCtx &c, long long leaf, int q) {
  if (q >= c.K) return -1;
  int e = 1;
  while (c.dt->Kdim[e] <= q) e++;
  const int qq = q - c.dt->Kdim[e - 1];
  const long long id = c.ninternal + leaf;
  const long long b = ((id + 1) >> (c.kappa - e + 1)) - 1;   // ancestor at depth e - 1 (heap order)
  return qq < c.rank[b] ? c.dt->colbase[e] + qq : -1;
}

__global__ void __launch_bounds__(AT) k_apply_leaf_up(ApplyCtx c) {
  __shared__ double sx[AVMAX], sv[AVMAX];
  const long long leaf = blockIdx.x;
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int i = t; i < m; i += AT) { sx[i] = c.xs[lo + i]; sv[i] = c.x[c.perm[lo + i]]; }
  __syncthreads();
  // dense diagonal block, on the fly (Table I + σ² on the diagonal)
  const KParams kp = kp_of(c.kp, c.kps, c.nseg, lo);
  for (int i = t; i < m; i += AT) {
    const double xi = sx[i];
    double s = 0.0;
    if (kp.dim > 1) for (int j = 0; j < m; j++) s = fma(kval_nd_fast(kp, c.xs, lo + i, lo + j), sv[j], s);   // NEXT-3
    else for (int j = 0; j < m; j++) s = fma(kval(kp, xi - sx[j]), sv[j], s);
    c.ys[lo + i] = fma(sig2(kp, lo + i), sv[i], s);
  }
  // P_l = E_l^T x_l: a warp takes 4 consecutive panel columns at once (lanes over rows, every load of a 128-row
  // chunk issued before the arithmetic), then a transposed butterfly leaves column q0 + j in lanes 8j .. 8j+7
  double *P = c.P + leaf * (long long)c.K;
  const int hi4 = lane & 16, hi3 = lane & 8;
  for (int q0 = 4 * warp; q0 < c.K; q0 += 4 * (AT / 32)) {
    const double *ecol[4];
    bool cv[4];
    double pv[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long src = q0 + j < c.K ? apply_colsrc(c, leaf, q0 + j) : -1;
      cv[j] = src >= 0;
      ecol[j] = c.Xh + (src >= 0 ? src : 0) * c.ldx + lo;
      pv[j] = 0.0;
    }
    for (int r0 = 0; r0 < m; r0 += 128) {
      double ev[4][4];
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = r0 + lane + 32 * u;
          ev[j][u] = (cv[j] && i < m) ? __ldg(ecol[j] + i) : 0.0;
        }
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = r0 + lane + 32 * u;
          pv[j] = fma(ev[j][u], i < m ? sv[i] : 0.0, pv[j]);
        }
    }
    double s0v = hi4 ? pv[0] : pv[2], s1v = hi4 ? pv[1] : pv[3];
    double k0 = hi4 ? pv[2] : pv[0], k1 = hi4 ? pv[3] : pv[1];
    k0 += __shfl_xor_sync(0xffffffffu, s0v, 16);
    k1 += __shfl_xor_sync(0xffffffffu, s1v, 16);
    const double svv = hi3 ? k0 : k1;
    double kk = hi3 ? k1 : k0;
    kk += __shfl_xor_sync(0xffffffffu, svv, 8);
    kk += __shfl_xor_sync(0xffffffffu, kk, 4);
    kk += __shfl_xor_sync(0xffffffffu, kk, 2);
    kk += __shfl_xor_sync(0xffffffffu, kk, 1);
    const int j = (lane >> 3) & 3;
    if ((lane & 7) == 0 && q0 + j < c.K) P[q0 + j] = kk;
  }
}

// One tree level: R_d[a][q] = R_{d+1}[2a][q] + R_{d+1}[2a+1][q], q < Kdim[d] (src = P when d + 1 == kappa).
__global__ void k_apply_tree(ApplyCtx c, int d) {
  const long long nd = 1LL << d;
  const int Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const double *src = d + 1 == c.kappa ? c.P : c.R + c.Roff[d + 1];
  double *dst = c.R + c.Roff[d];
  const long long tot = nd * Kd;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < tot; p += (long long)gridDim.x * blockDim.x) {
    const long long a = p / Kd; const int q = (int)(p - a * Kd);
    dst[p] = src[(2 * a) * K1 + q] + src[(2 * a + 1) * K1 + q];
  }
}

__global__ void __launch_bounds__(AT) k_apply_leaf_down(ApplyCtx c) {
  __shared__ double sw[AKMAX];
  __shared__ long long scol[AKMAX];
  const long long leaf = blockIdx.x;
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  const int t = threadIdx.x;
  // w_l[q] (q in slot e) = t of the sibling of the depth-e ancestor: R_e[(leaf >> (kappa - e)) ^ 1][q]
  for (int q = t; q < c.K; q += AT) {
    int e = 1;
    while (c.dt->Kdim[e] <= q) e++;
    const long long ia = leaf >> (c.kappa - e);            // index of the depth-e ancestor within its depth
    const double *Re = e == c.kappa ? c.P : c.R + c.Roff[e];
    const int Ke = c.dt->Kdim[e];
    const long long src = apply_colsrc(c, leaf, q);
    scol[q] = src >= 0 ? src : 0;
    sw[q] = src >= 0 ? Re[(ia ^ 1) * Ke + q] : 0.0;
  }
  __syncthreads();
  // ys_l += E_l w_l: invalid columns carry weight 0 and read column 0 (no branch: the loads of 8 columns are in
  // flight together)
  for (int i = t; i < m; i += AT) {
    double s = c.ys[lo + i];
    const double *xr = c.Xh + lo + i;
    int q = 0;
    for (; q + 16 <= c.K; q += 16) {
      double ev[16];
#pragma unroll
      for (int j = 0; j < 16; j++) ev[j] = __ldg(xr + scol[q + j] * c.ldx);
#pragma unroll
      for (int j = 0; j < 16; j++) s = fma(ev[j], sw[q + j], s);
    }
    for (; q < c.K; q++) s = fma(__ldg(xr + scol[q] * c.ldx), sw[q], s);
    c.y[c.perm[lo + i]] = s;
  }
}

}  // namespace

hodlr_status hodlr_apply_impl(hodlr_s *h, const double *x, double *y) {
  const int kappa = h->kappa;
  const long long n = h->n, nl = h->nleaves;
  const int K = kappa > 0 ? h->dt.Kdim[kappa] : 0;
  if (h->leaf_max > AVMAX || K > AKMAX)
    return hodlr_set_error(HODLR_EINVAL, "apply: leaf size %d > %d or K = %d > %d", h->leaf_max, AVMAX, K, AKMAX);
  ApplyCtx c;
  c.kp = h->kp; c.n = n; c.ninternal = h->ninternal; c.nleaves = nl; c.ldx = h->ldx; c.kappa = kappa; c.K = K;
  c.xs = h->xs; c.lo = h->lo; c.hi = h->hi; c.perm = h->perm; c.Xh = h->Xh; c.rank = h->rank; c.dt = h->d_dt;
  c.x = x; c.y = y;
  c.kps = h->d_kps; c.nseg = h->nseg;
  long long rtot = 0;
  for (int d = 0; d <= kappa && d < HODLR_MAXDEPTH + 2; d++) {
    c.Roff[d] = rtot;
    if (d >= 1 && d < kappa) rtot += (1LL << d) * (long long)h->dt.Kdim[d];
  }
  const size_t need = (size_t)n + (size_t)nl * (size_t)(K > 0 ? K : 1) + (size_t)(rtot > 0 ? rtot : 1);
  if (h->apply_ws_n < need) {
    h->apply_ws = (double *)hodlr_dalloc(h, sizeof(double) * need);
    if (!h->apply_ws) return hodlr_set_error(HODLR_ENOMEM, "apply: workspace");
    h->apply_ws_n = need;
  }
  c.ys = h->apply_ws; c.P = c.ys + n; c.R = c.P + nl * (long long)(K > 0 ? K : 1);
  HCUDA(cudaMemcpyAsync(h->d_dt, &h->dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));   // Kdim after the ACA
  k_apply_leaf_up<<<(unsigned)nl, AT, 0, h->st>>>(c);
  HLAUNCH(h, "k_apply_leaf_up");
  for (int d = kappa - 1; d >= 1; d--) {
    const long long tot = (1LL << d) * (long long)h->dt.Kdim[d];
    const int grid = (int)std::min<long long>((tot + 255) / 256, 4096);
    k_apply_tree<<<grid > 0 ? grid : 1, 256, 0, h->st>>>(c, d);
    HLAUNCH(h, "k_apply_tree");
  }
  k_apply_leaf_down<<<(unsigned)nl, AT, 0, h->st>>>(c);
  HLAUNCH(h, "k_apply_leaf_down");
  return HODLR_OK;
}
