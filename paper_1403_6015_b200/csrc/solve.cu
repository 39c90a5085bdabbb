// solve.cu -- G11/G12: x = C^{-1} y by applying the inverse factors (eq-fac)
// in projected form:
//   up   (leaves)  v_l = A_l^{-1} b_l,  g_l = E_l^T v_l,  h_l = b_l . v_l
//   up   (node c)  t_c = S_c^{-1} [g_c2[s]; g_c1[s]]
//                  g_c = g_c1[a] + g_c2[a] - B_c[r:]^T t_c[:r] - B_c[:r]^T t_c[r:]
//                  h_c = h_c1 + h_c2 - g_c1[s] . t_c[:r] - g_c2[s] . t_c[r:]
//   down (node c)  f = t_c + T_c w_c;  w_c1 = [w_c, -f[:r]],  w_c2 = [w_c, -f[r:]]
//   down (leaves)  x_l = A_l^{-1} (b_l + E_l w_l)
// h_root = y^T C^{-1} y gives the log-likelihood without the down pass (eq. 1).
//
// One persistent cooperative kernel (one 512-thread CTA per SM) runs the phases separated by grid barriers:
// leaf up -> tree up, level by level -> tree down, level by level -> leaf down.  Leaf phases use the stored
// X = L^{-1} (two triangular matrix-vector products) and stage X and the ancestor panel E_l in shared memory
// with cp.async, prefetching the next leaf's X while E is used and its E while X is used.  Tree nodes: one
// warp each (t_c by S_c^{-1} + 2 compensated refinement steps; compensated accumulations).
// Under subtree sharding the kernel is split at the exchange of the depth-t projections.
#include "hodlr_internal.cuh"
#include <cooperative_groups.h>
#include <type_traits>
#include <stdio.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

namespace {

constexpr int LT = 256;           // threads per CTA (two CTAs per SM)
constexpr int NWL = LT / 32;      // warps per CTA
constexpr int VMAX = 8 * 32;      // leaf rows handled (leaf_max < 2 leaf <= 256)
static_assert(VMAX <= LT, "one leaf row per thread (y_fetch)");

struct SolveCtx {
  long long n, ninternal, nleaves;
  int kappa, K, T;
  int grank, tsplit;
  const long long *lo, *hi, *perm;
  const double *Xh; long long ldx;
  const int *rank;
  const DepthTab *dt;
  const double *Lf; long long lstride;
  const double *Uf; const int *lperm;   // LU leaves (kernel not SPD, R20): A^{-1} b = XU^T (XL (P b)), XU = Uf tiles
                                        // read from global memory, P b = b[lperm]; NULL for Cholesky leaves
  const double *Spool, *BTpool;
  double *V;        // per-level node vectors (g on the way up, w on the way down)
  double *Tv;       // per-node t_c (q hi, q lo doubles; depth-d offset nodeT[d])
  double *hv;       // per-node h = y_c^T K_cc^{-1} y_c as a double-double pair (heap id)
  const double *y;
  double *x;
  double *xsorted;  // sharded solve: this rank's solution rows in sorted order (NULL on one GPU)
  int *flags;
  long long leaf0, nown;    // this rank's leaves
  long long tree_scratch;   // doubles of per-warp scratch for the tree-up nodes
  int tree_warps;           // warps per CTA that take tree-up nodes (scratch must fit)
  unsigned long long *stamps;   // HODLR_TRACE: %globaltimer after each phase (block 0), or NULL
  int R;                    // right-hand sides of this launch (columns r of y / x at r * ldy)
  long long xdoubles;       // X tile staging (doubles) at the start of the dynamic shared memory
  int xglobal;              // leaves too large to stage X (p > ~235): the triangular products read X from global
  long long ldy;
  long long vcol, tcol, hcol;   // per-column strides of V, Tv and hv
  int aug;                  // the factorization carries a fused right-hand side: B_c / T_c rows have Kf[d] = Kdim[d] + 1
                            // entries with the ancestor columns at offset 1 (column 0 belongs to that right-hand side)
  int fused;                // this solve IS that right-hand side: t_c = T_c[:, 0] from the factorization (no up pass)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

struct Phases {
  int leaf_up;      // run the leaf up pass
  int up_hi, up_lo; // tree up levels d = up_hi down to up_lo (none if up_hi < up_lo)
  int down;         // run the tree down levels and the leaf down pass
};

__device__ __forceinline__ void own_range(const SolveCtx &c, int d, long long &i0, long long &cnt) {
  if (d < c.tsplit) { i0 = 0; cnt = 1LL << d; }
  else { cnt = 1LL << (d - c.tsplit); i0 = (long long)c.grank * cnt; }
}

__device__ __forceinline__ void cp16(double *dst, const double *src) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N)); }

__device__ __forceinline__ int leaf_colsrc(const SolveCtx &c, long long id, int q) {
  if (q >= c.K) return -1;
  int e = 1;
  while (c.dt->Kdim[e] <= q) e++;
  const int qq = q - c.dt->Kdim[e - 1];
  const long long b = ((id + 1) >> (c.kappa - e + 1)) - 1;     // ancestor at depth e - 1 (heap order)
  return qq < c.rank[b] ? (int)(c.dt->colbase[e] + qq) : -1;
}

// ---------------------------------------------------------------------------------------------
// leaf staging: X = L^{-1} tiles (one commit group); the panel E_l is read from global memory (L2-resident
// across the right-hand sides of a leaf)
// ---------------------------------------------------------------------------------------------
__device__ void issue_x(const SolveCtx &c, long long leaf, double *sX) {
  const double *Xg = c.Lf + leaf * c.lstride;
  if (c.xglobal) { cp_commit(); return; }
  const int nx2 = (c.T * (c.T + 1) / 2) * 32;
  for (int p = threadIdx.x; p < nx2; p += LT) cp16(sX + 2 * p, Xg + 2 * p);
  cp_commit();
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// out = X in (lower) on the FP64 tensor pipe: warp I owns tile row I, C(I) = sum_{k <= I} X(I,k) B_k with B_k the
// 8-vector in_k replicated over the 8 columns (A fragments straight from the fragment-order tiles:
// conflict-free).  Two accumulators alternate over k.
__device__ void tri_mv(const double *X, int T, const double *in, double *out, double *) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  for (int I = warp; I < T; I += NWL) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
    int k = 0;
    for (; k + 1 <= I; k += 2) {
      const double *t0 = X + tix(I, k) * 64, *t1 = X + tix(I, k + 1) * 64;
      dmma(c0, c1, t0[lane], in[8 * k + tq]);
      dmma(e0, e1, t1[lane], in[8 * k + 8 + tq]);
      dmma(c0, c1, t0[32 + lane], in[8 * k + 4 + tq]);
      dmma(e0, e1, t1[32 + lane], in[8 * k + 12 + tq]);
    }
    if (k <= I) {
      const double *t0 = X + tix(I, k) * 64;
      dmma(c0, c1, t0[lane], in[8 * k + tq]);
      dmma(c0, c1, t0[32 + lane], in[8 * k + 4 + tq]);
    }
    if (tq == 0) out[8 * I + g] = c0 + e0;
  }
  __syncthreads();
}

// out = X^T in: warp J owns tile column J, C(J) = sum_{I >= J} X(I,J)^T B_I; the A fragment of X(I,J)^T
// (row g, column tq) is tile element (tq, g) at fo(tq, g) (2 wavefronts per half, the minimum for 64-bit).
__device__ void tri_mvt(const double *X, int T, const double *in, double *out, double *) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  const int a0 = fo(tq, g), a1 = fo(tq + 4, g);
  for (int J = warp; J < T; J += NWL) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
    int I = J;
    for (; I + 1 < T; I += 2) {
      const double *t0 = X + tix(I, J) * 64, *t1 = X + tix(I + 1, J) * 64;
      dmma(c0, c1, t0[a0], in[8 * I + tq]);
      dmma(e0, e1, t1[a0], in[8 * I + 8 + tq]);
      dmma(c0, c1, t0[a1], in[8 * I + 4 + tq]);
      dmma(e0, e1, t1[a1], in[8 * I + 12 + tq]);
    }
    if (I < T) {
      const double *t0 = X + tix(I, J) * 64;
      dmma(c0, c1, t0[a0], in[8 * I + tq]);
      dmma(c0, c1, t0[a1], in[8 * I + 4 + tq]);
    }
    __syncwarp();
    if (tq == 0) out[8 * J + g] = c0 + e0;
  }
  __syncthreads();
}

constexpr int KMAX_SOLVE = 512;
#ifndef SOLVE_RMAX
#define SOLVE_RMAX 32     // right-hand sides per solve launch
#endif
#ifndef SOLVE_UPB
#define SOLVE_UPB 4       // leaf up: panel columns per warp batch (multiple of 4)
#endif
#ifndef SOLVE_DNU
#define SOLVE_DNU 16      // leaf down: panel columns loaded together per lane
#endif
struct LeafSmem {
  double sb[VMAX], su[VMAX], red[4 * VMAX], sw[KMAX_SOLVE];
  int colsrc[KMAX_SOLVE];
};

// y entries of (leaf, column r) for this thread's row (R <= LT: at most one row per thread), gathered through perm;
// issued one (leaf, column) ahead so the dependent loads (lo/hi -> perm -> y) overlap the current one.
__device__ __forceinline__ double y_fetch(const SolveCtx &c, long long leaf, int r) {
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  return (int)threadIdx.x < m ? c.y[r * c.ldy + c.perm[lo + threadIdx.x]] : 0.0;
}

// ---------------------------------------------------------------------------------------------
// leaf up over this CTA's leaves (leaf0 + blockIdx.x + k gridDim.x); per leaf X is staged once and reused by every
// right-hand side r: u = X b_r, v = X^T u, h_r = b_r . v, g_r = E^T v (E from global memory; after the first
// column of a leaf it is an L2 hit).  The next leaf's X is copied during the last column.
// ---------------------------------------------------------------------------------------------
__device__ void leaf_up_phase(const SolveCtx &c, double *sX, LeafSmem &S) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int Rr = 8 * c.T, K = c.K;
  long long leaf = c.leaf0 + blockIdx.x;
  const long long end = c.leaf0 + c.nown;
  if (leaf >= end) return;
  issue_x(c, leaf, sX);
  double ycur = y_fetch(c, leaf, 0);
  for (; leaf < end; leaf += gridDim.x) {
    const long long nxt = leaf + gridDim.x;
    const long long id = c.ninternal + leaf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    for (int q = t; q < K; q += LT) S.colsrc[q] = leaf_colsrc(c, id, q);
    for (int r = 0; r < c.R; r++) {
      {
        const double v = ycur;
        if (r + 1 < c.R) ycur = y_fetch(c, leaf, r + 1);
        else if (nxt < end) ycur = y_fetch(c, nxt, 0);
        if (t < Rr) {
          S.sb[t] = v;
          if (!isfinite(v)) atomicOr(&c.flags[3], 1);
        }
      }
      if (r == 0) cp_wait<0>();                // X of this leaf
      __syncthreads();
      if (c.Uf) {                              // LU leaves: u = XL (P b), v = XU^T u
        const int *lp = c.lperm + leaf * Rr;
        for (int i = t; i < Rr; i += LT) S.red[VMAX + i] = S.sb[lp[i]];
        __syncthreads();
        tri_mv(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.red + VMAX, S.su, nullptr);
        tri_mvt(c.Uf + leaf * c.lstride, c.T, S.su, S.red, nullptr);
      } else {
        tri_mv(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.sb, S.su, S.red);      // u = X b
        tri_mvt(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.su, S.red, nullptr);  // v = X^T u  (into red[0..R))
      }
      if (r + 1 == c.R && nxt < end) issue_x(c, nxt, sX);   // X is free
      double hs = 0.0;
      for (int i = t; i < m; i += LT) hs += S.sb[i] * S.red[i];
      hs = warp_sum(hs);
      if (lane == 0) S.red[2 * VMAX + warp] = hs;
      double *g = c.V + r * c.vcol + c.dt->nodeV[c.kappa] + leaf * (long long)K;
      // g = E^T v from global memory: a warp takes 4 consecutive columns at once (all their loads in flight
      // together), lanes over rows; the 4 partial sums are reduced by a transposed butterfly (6 shuffles), after
      // which lanes 8j .. 8j+7 hold column q0 + j
      const int hi4 = lane & 16, hi3 = lane & 8;
      for (int q0 = SOLVE_UPB * warp; q0 < K; q0 += SOLVE_UPB * NWL) {
        constexpr int RU = 4;                  // rows per lane per chunk (128-row chunks)
        double pv[SOLVE_UPB];
        const double *ecol[SOLVE_UPB];
        bool cv[SOLVE_UPB];
#pragma unroll
        for (int j = 0; j < SOLVE_UPB; j++) {
          const int src = q0 + j < K ? S.colsrc[q0 + j] : -1;
          cv[j] = src >= 0;
          ecol[j] = c.Xh + (long long)(src >= 0 ? src : 0) * c.ldx + lo;
          pv[j] = 0.0;
        }
        for (int r0 = 0; r0 < Rr; r0 += 32 * RU) {
          double ev[SOLVE_UPB][RU];
#pragma unroll
          for (int j = 0; j < SOLVE_UPB; j++)
#pragma unroll
            for (int u = 0; u < RU; u++) {
              const int i = r0 + lane + 32 * u;
              ev[j][u] = (cv[j] && i < m) ? __ldg(ecol[j] + i) : 0.0;
            }
#pragma unroll
          for (int j = 0; j < SOLVE_UPB; j++)
#pragma unroll
            for (int u = 0; u < RU; u++) {
              const int i = r0 + lane + 32 * u;
              pv[j] = fma(ev[j][u], i < m ? S.red[i] : 0.0, pv[j]);
            }
        }
#pragma unroll
        for (int b4 = 0; b4 < SOLVE_UPB; b4 += 4) {
          double s0v = hi4 ? pv[b4] : pv[b4 + 2], s1v = hi4 ? pv[b4 + 1] : pv[b4 + 3];
          double k0 = hi4 ? pv[b4 + 2] : pv[b4], k1 = hi4 ? pv[b4 + 3] : pv[b4 + 1];
          k0 += __shfl_xor_sync(0xffffffffu, s0v, 16);
          k1 += __shfl_xor_sync(0xffffffffu, s1v, 16);
          const double sv = hi3 ? k0 : k1;
          double kk = hi3 ? k1 : k0;
          kk += __shfl_xor_sync(0xffffffffu, sv, 8);
          kk += __shfl_xor_sync(0xffffffffu, kk, 4);
          kk += __shfl_xor_sync(0xffffffffu, kk, 2);
          kk += __shfl_xor_sync(0xffffffffu, kk, 1);
          const int j = b4 + ((lane >> 3) & 3);
          if ((lane & 7) == 0 && q0 + j < K) g[q0 + j] = kk;
        }
      }
      __syncthreads();
      if (t == 0) {
        double h = 0.0;
        for (int w = 0; w < NWL; w++) h += S.red[2 * VMAX + w];
        double *hv = c.hv + r * c.hcol;
        hv[2 * id] = h; hv[2 * id + 1] = 0.0;
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// leaf down: x_l = A_l^{-1} (b_l + E_l w_l) for every right-hand side r; X staged once per leaf
__device__ void leaf_down_phase(const SolveCtx &c, double *sX, LeafSmem &S) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int Rr = 8 * c.T, K = c.K;
  long long leaf = c.leaf0 + blockIdx.x;
  const long long end = c.leaf0 + c.nown;
  if (leaf >= end) return;
  issue_x(c, leaf, sX);
  double ycur = y_fetch(c, leaf, 0);
  static_assert(KMAX_SOLVE <= 2 * LT, "w prefetch: two columns per thread");
  const double *wbase = c.V + c.dt->nodeV[c.kappa];
  double w0 = t < K ? wbase[leaf * (long long)K + t] : 0.0, w1 = t + LT < K ? wbase[leaf * (long long)K + t + LT] : 0.0;
  for (; leaf < end; leaf += gridDim.x) {
    const long long nxt = leaf + gridDim.x;
    const long long id = c.ninternal + leaf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    for (int q = t; q < K; q += LT) S.colsrc[q] = leaf_colsrc(c, id, q);
    for (int r = 0; r < c.R; r++) {
      __syncthreads();                         // previous column's users of sw / sb / colsrc are done
      if (t < K) S.sw[t] = w0;                 // w of this (leaf, column), fetched one ahead
      if (t + LT < K) S.sw[t + LT] = w1;
      {
        const long long nl = r + 1 < c.R ? leaf : nxt;
        const int nr = r + 1 < c.R ? r + 1 : 0;
        if (nl < end) {
          const double *wb = wbase + nr * c.vcol + nl * (long long)K;
          w0 = t < K ? wb[t] : 0.0;
          w1 = t + LT < K ? wb[t + LT] : 0.0;
        }
        const double v = ycur;
        if (nl < end) ycur = y_fetch(c, nl, nr);
        if (t < Rr) S.sb[t] = v;
      }
      __syncthreads();
      // b + E w from global memory: warp w takes row group w % RG (one row per lane) and column split w / RG;
      // SOLVE_DNU columns' loads in flight per lane; the CS column-split partials are summed in a fixed order
      const int RG = (Rr + 31) / 32, CS = NWL / RG;
      const int rg = warp % RG, cs = warp / RG;
      const int i = 32 * rg + lane;
      if (cs < CS) {
        double s2 = 0.0;
        const int q0 = (K * cs) / CS, q1 = (K * (cs + 1)) / CS;
        const double *ebase = c.Xh + lo + i;
        int q = q0;
        for (; q + SOLVE_DNU <= q1; q += SOLVE_DNU) {
          double ev[SOLVE_DNU];
#pragma unroll
          for (int j = 0; j < SOLVE_DNU; j++) {
            const int src = S.colsrc[q + j];
            ev[j] = (src >= 0 && i < m) ? __ldg(ebase + (long long)src * c.ldx) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < SOLVE_DNU; j++) s2 = fma(ev[j], S.sw[q + j], s2);
        }
        for (; q < q1; q++) {
          const int src = S.colsrc[q];
          if (src >= 0 && i < m) s2 = fma(__ldg(ebase + (long long)src * c.ldx), S.sw[q], s2);
        }
        S.red[cs * Rr + i] = s2;
      }
      __syncthreads();
      for (int rr = t; rr < Rr; rr += LT) {
        double acc = 0.0;
        for (int k2 = 0; k2 < CS; k2++) acc += S.red[k2 * Rr + rr];
        S.sb[rr] += acc;
      }
      if (r == 0) cp_wait<0>();                // X of this leaf
      __syncthreads();
      if (c.Uf) {                              // LU leaves (R20)
        const int *lp = c.lperm + leaf * Rr;
        for (int i = t; i < Rr; i += LT) S.red[VMAX + i] = S.sb[lp[i]];
        __syncthreads();
        tri_mv(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.red + VMAX, S.su, nullptr);
        tri_mvt(c.Uf + leaf * c.lstride, c.T, S.su, S.sb, nullptr);
      } else {
        tri_mv(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.sb, S.su, S.red);
        tri_mvt(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.su, S.sb, S.red);
      }
      if (r + 1 == c.R && nxt < end) issue_x(c, nxt, sX);
      if (c.xsorted) for (int i2 = t; i2 < m; i2 += LT) c.xsorted[lo + i2] = S.sb[i2];
      else for (int i2 = t; i2 < m; i2 += LT) c.x[r * c.ldy + c.perm[lo + i2]] = S.sb[i2];
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Eight right-hand sides at a time (the batched kernel k_solve<8>): every DMMA m8n8k4 then carries 8 different
// vectors in its B operand instead of one replicated vector, the panel products E^T V and E W become 8-column
// DMMA products, and X and E_l are read once per leaf for all columns.  Rows beyond the leaf are zero.
// ---------------------------------------------------------------------------------------------
constexpr int VP = VMAX + 4;            // row stride of the 8-column vectors (bank padding)
struct LeafSmem8 {
  double b[8][VP], u[8][VP];
  union { double v[8][VP]; double w[8][KMAX_SOLVE + 4]; };
  int colsrc[KMAX_SOLVE];
  double hred[8];
};

// out_c = X in_c for the 8 columns c (warp I owns tile row I; C fragment: column 2tq, 2tq+1, row 8I + g)
__device__ void tri_mv8(const double *X, int T, const double (*in)[VP], double (*out)[VP]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  for (int I = warp; I < T; I += NWL) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
    int k = 0;
    for (; k + 1 <= I; k += 2) {
      const double *t0 = X + tix(I, k) * 64, *t1 = X + tix(I, k + 1) * 64;
      dmma(c0, c1, t0[lane], in[g][8 * k + tq]);
      dmma(e0, e1, t1[lane], in[g][8 * k + 8 + tq]);
      dmma(c0, c1, t0[32 + lane], in[g][8 * k + 4 + tq]);
      dmma(e0, e1, t1[32 + lane], in[g][8 * k + 12 + tq]);
    }
    if (k <= I) {
      const double *t0 = X + tix(I, k) * 64;
      dmma(c0, c1, t0[lane], in[g][8 * k + tq]);
      dmma(c0, c1, t0[32 + lane], in[g][8 * k + 4 + tq]);
    }
    out[2 * tq][8 * I + g] = c0 + e0;
    out[2 * tq + 1][8 * I + g] = c1 + e1;
  }
  __syncthreads();
}

// out_c = X^T in_c (warp J owns tile column J)
__device__ void tri_mvt8(const double *X, int T, const double (*in)[VP], double (*out)[VP]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  const int a0 = fo(tq, g), a1 = fo(tq + 4, g);
  for (int J = warp; J < T; J += NWL) {
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
    int I = J;
    for (; I + 1 < T; I += 2) {
      const double *t0 = X + tix(I, J) * 64, *t1 = X + tix(I + 1, J) * 64;
      dmma(c0, c1, t0[a0], in[g][8 * I + tq]);
      dmma(e0, e1, t1[a0], in[g][8 * I + 8 + tq]);
      dmma(c0, c1, t0[a1], in[g][8 * I + 4 + tq]);
      dmma(e0, e1, t1[a1], in[g][8 * I + 12 + tq]);
    }
    if (I < T) {
      const double *t0 = X + tix(I, J) * 64;
      dmma(c0, c1, t0[a0], in[g][8 * I + tq]);
      dmma(c0, c1, t0[a1], in[g][8 * I + 4 + tq]);
    }
    out[2 * tq][8 * J + g] = c0 + e0;
    out[2 * tq + 1][8 * J + g] = c1 + e1;
  }
  __syncthreads();
}

// b[c][i] = y of column r0 + c (c < nr) at sorted row lo + i, zero elsewhere
__device__ void load_b8(const SolveCtx &c, long long lo, int m, int r0, int nr, double (*b)[VP]) {
  const int Rr = 8 * c.T;
  for (int p = threadIdx.x; p < 8 * Rr; p += LT) {
    const int cc = p / Rr, i = p - cc * Rr;
    double v = 0.0;
    if (cc < nr && i < m) {
      v = c.y[(r0 + cc) * c.ldy + c.perm[lo + i]];
      if (!isfinite(v)) atomicOr(&c.flags[3], 1);
    }
    b[cc][i] = v;
  }
}

__device__ void leaf_up_phase8(const SolveCtx &c, double *sX, LeafSmem8 &S) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, tq = lane & 3;
  const int K = c.K;
  long long leaf = c.leaf0 + blockIdx.x;
  const long long end = c.leaf0 + c.nown;
  if (leaf >= end) return;
  issue_x(c, leaf, sX);
  for (; leaf < end; leaf += gridDim.x) {
    const long long nxt = leaf + gridDim.x;
    const long long id = c.ninternal + leaf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    for (int q = t; q < K; q += LT) S.colsrc[q] = leaf_colsrc(c, id, q);
    for (int r0 = 0; r0 < c.R; r0 += 8) {
      const int nr = min(8, c.R - r0);
      load_b8(c, lo, m, r0, nr, S.b);
      if (r0 == 0) cp_wait<0>();
      __syncthreads();
      tri_mv8(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.b, S.u);               // u = X b
      tri_mvt8(c.xglobal ? c.Lf + leaf * c.lstride : sX, c.T, S.u, S.v);              // v = X^T u
      if (r0 + 8 >= c.R && nxt < end) issue_x(c, nxt, sX);   // X is free
      {                                          // h_c = b_c . v_c: warp c
        double hs = 0.0;
        for (int i = lane; i < m; i += 32) hs = fma(S.b[warp][i], S.v[warp][i], hs);
        hs = warp_sum(hs);
        if (lane == 0 && warp < nr) {
          double *hv = c.hv + (r0 + warp) * c.hcol;
          hv[2 * id] = hs; hv[2 * id + 1] = 0.0;
        }
      }
      // G (8 x K) = V^T E: warp takes 8 panel columns q0 .. q0+7 at a time; A = V^T (row c, col = leaf row),
      // B = E (row = leaf row, col = panel column), both k = 4 leaf rows per DMMA
      for (int q0 = 8 * warp; q0 < K; q0 += 8 * NWL) {
        const int src = q0 + g < K ? S.colsrc[q0 + g] : -1;
        const double *ecol = c.Xh + (long long)(src >= 0 ? src : 0) * c.ldx + lo;
        double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
        for (int kb = 0; kb < m; kb += 32) {       // 8 DMMA steps (32 rows) per batch, loads first
          double ev[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int i = kb + 4 * u + tq;
            ev[u] = (src >= 0 && i < m) ? __ldg(ecol + i) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; u += 2) {
            dmma(c0, c1, S.v[g][kb + 4 * u + tq], ev[u]);
            dmma(e0, e1, S.v[g][kb + 4 * u + 4 + tq], ev[u + 1]);
          }
        }
        // C[c = g][q0 + 2tq (+1)]
        if (g < nr) {
          double *gp = c.V + (r0 + g) * c.vcol + c.dt->nodeV[c.kappa] + leaf * (long long)K;
          if (q0 + 2 * tq < K) gp[q0 + 2 * tq] = c0 + e0;
          if (q0 + 2 * tq + 1 < K) gp[q0 + 2 * tq + 1] = c1 + e1;
        }
      }
      __syncthreads();
    }
  }
  cp_wait<0>();
  __syncthreads();
}

__device__ void leaf_down_phase8(const SolveCtx &c, double *sX, LeafSmem8 &S) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, g = lane >> 2, tq = lane & 3;
  const int K = c.K, T = c.T;
  long long leaf = c.leaf0 + blockIdx.x;
  const long long end = c.leaf0 + c.nown;
  if (leaf >= end) return;
  issue_x(c, leaf, sX);
  const double *wbase = c.V + c.dt->nodeV[c.kappa];
  for (; leaf < end; leaf += gridDim.x) {
    const long long nxt = leaf + gridDim.x;
    const long long id = c.ninternal + leaf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    for (int q = t; q < K; q += LT) S.colsrc[q] = leaf_colsrc(c, id, q);
    for (int r0 = 0; r0 < c.R; r0 += 8) {
      const int nr = min(8, c.R - r0);
      __syncthreads();
      load_b8(c, lo, m, r0, nr, S.b);
      for (int p = t; p < 8 * K; p += LT) {      // w of the 8 columns (zero for c >= nr)
        const int cc = p / K, q = p - cc * K;
        S.w[cc][q] = cc < nr ? wbase[(r0 + cc) * c.vcol + leaf * (long long)K + q] : 0.0;
      }
      for (int p = t; p < 8 * 4; p += LT) S.w[p >> 2][K + (p & 3)] = 0.0;   // (k padding of the last DMMA step)
      __syncthreads();
      // b += E W: warp takes tile rows I (8 leaf rows), A = E (row 8I + g, col = panel column), B = W
      for (int I = warp; I < T; I += NWL) {
        const int i = 8 * I + g;
        double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
        for (int q0 = 0; q0 < K; q0 += 16) {
          double ev[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int q = q0 + 4 * u + tq;
            const int src = q < K ? S.colsrc[q] : -1;
            ev[u] = (src >= 0 && i < m) ? __ldg(c.Xh + (long long)src * c.ldx + lo + i) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; u += 2) {
            const int qa = q0 + 4 * u + tq, qb = qa + 4;
            dmma(c0, c1, ev[u], qa < K ? S.w[g][qa] : 0.0);
            dmma(e0, e1, ev[u + 1], qb < K ? S.w[g][qb] : 0.0);
          }
        }
        S.b[2 * tq][i] += c0 + e0;
        S.b[2 * tq + 1][i] += c1 + e1;
      }
      if (r0 == 0) cp_wait<0>();
      __syncthreads();
      tri_mv8(c.xglobal ? c.Lf + leaf * c.lstride : sX, T, S.b, S.u);
      tri_mvt8(c.xglobal ? c.Lf + leaf * c.lstride : sX, T, S.u, S.b);
      if (r0 + 8 >= c.R && nxt < end) issue_x(c, nxt, sX);
      for (int p = t; p < 8 * m; p += LT) {
        const int cc = p / m, i = p - cc * m;
        if (cc < nr) c.x[(r0 + cc) * c.ldy + c.perm[lo + i]] = S.b[cc][i];
      }
    }
  }
  cp_wait<0>();
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// tree nodes (one warp each)
// ---------------------------------------------------------------------------------------------
// t = S^{-1} rhs as (th, tl): explicit inverse S^{-1} (from the factor phase) + 2 refinement steps with
// compensated residuals.  All vectors in the warp's shared scratch.
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

__device__ void tree_up_node(const SolveCtx &c, int d, long long i, int col, double *scr, int lane) {
  const long long node = (1LL << d) - 1 + i;
  double *const V = c.V + col * c.vcol, *const Tvc = c.Tv + col * c.tcol, *const hv = c.hv + col * c.hcol;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const int ldb = c.dt->Kf[d];               // B_c row stride (ancestor columns at offset c.aug)
  const double *g1 = V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  const double *g2 = g1 + K1;
  const double *Sg = c.Spool + c.dt->nodeS[d] + i * (long long)(2 * q * q + q);
  const double *B = c.BTpool + c.dt->nodeBT[d] + i * 3LL * q * ldb + c.aug;
  double *S0 = scr;
  double *Si = S0 + q * q, *rhs = Si + q * q + q, *th = rhs + q, *tl = th + q, *tmp = tl + q;
  {
    const int np = 2 * q * q + q;
    int p = lane;
    for (; p + 96 < np; p += 128) {            // 4 independent loads in flight per lane
      const double a0 = Sg[p], a1 = Sg[p + 32], a2 = Sg[p + 64], a3 = Sg[p + 96];
      S0[p] = a0; S0[p + 32] = a1; S0[p + 64] = a2; S0[p + 96] = a3;
    }
    for (; p < np; p += 32) S0[p] = Sg[p];
  }
  for (int u = lane; u < r; u += 32) { rhs[u] = g2[Kd + u]; rhs[r + u] = g1[Kd + u]; }
  __syncwarp();
  dd_solve_warp(S0, Si, q, rhs, th, tl, tmp, lane);
  double *tg = Tvc + c.dt->nodeT[d] + i * 2LL * q;
  for (int u = lane; u < q; u += 32) { tg[u] = th[u]; tg[q + u] = tl[u]; }
  if (lane == 0) {
    Acc2 A = acc2(hv[2 * (2 * node + 1)]);
    acc_add_dd(A, hv[2 * (2 * node + 2)], hv[2 * (2 * node + 2) + 1]);
    A.c += hv[2 * (2 * node + 1) + 1];
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g1[Kd + u], th[u], tl[u]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -g2[Kd + u], th[r + u], tl[r + u]);
    acc_dd(A, hv[2 * node], hv[2 * node + 1]);
  }
  double *gc = V + c.dt->nodeV[d] + i * (long long)Kd;
  // 4 entries a per lane at once (a = a0 + 32 x): the B loads of all four are independent and issued together
  for (int a0 = lane; a0 < Kd; a0 += 128) {
    Acc2 A[4];
#pragma unroll
    for (int x = 0; x < 4; x++) {
      const int a = a0 + 32 * x;
      A[x] = acc2(a < Kd ? g1[a] : 0.0);
      acc_add(A[x], a < Kd ? g2[a] : 0.0);
    }
    for (int u = 0; u < r; u++) {
      double b1[4], b2[4];
#pragma unroll
      for (int x = 0; x < 4; x++) {
        const int a = a0 + 32 * x, ac = a < Kd ? a : 0;
        b1[x] = B[(long long)(r + u) * ldb + ac]; b2[x] = B[(long long)u * ldb + ac];
      }
#pragma unroll
      for (int x = 0; x < 4; x++) { acc_fma_dd(A[x], -b1[x], th[u], tl[u]); acc_fma_dd(A[x], -b2[x], th[r + u], tl[r + u]); }
    }
#pragma unroll
    for (int x = 0; x < 4; x++) if (a0 + 32 * x < Kd) gc[a0 + 32 * x] = acc_val(A[x]);
  }
  __syncwarp();
}

// Same as tree_up_node with the whole CTA on one node (levels with few nodes): every thread stages, warp 0
// solves, all threads form g_c; the arithmetic and its order per output are identical.
__device__ void tree_up_node_cta(const SolveCtx &c, int d, long long i, int col, double *scr) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const long long node = (1LL << d) - 1 + i;
  double *const V = c.V + col * c.vcol, *const Tvc = c.Tv + col * c.tcol, *const hv = c.hv + col * c.hcol;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const int ldb = c.dt->Kf[d];
  const double *g1 = V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  const double *g2 = g1 + K1;
  const double *Sg = c.Spool + c.dt->nodeS[d] + i * (long long)(2 * q * q + q);
  const double *B = c.BTpool + c.dt->nodeBT[d] + i * 3LL * q * ldb + c.aug;
  double *S0 = scr;
  double *Si = S0 + q * q, *rhs = Si + q * q + q, *th = rhs + q, *tl = th + q, *tmp = tl + q;
  for (int p = t; p < 2 * q * q + q; p += LT) S0[p] = Sg[p];
  for (int u = t; u < r; u += LT) { rhs[u] = g2[Kd + u]; rhs[r + u] = g1[Kd + u]; }
  __syncthreads();
  if (warp == 0) {
    dd_solve_warp(S0, Si, q, rhs, th, tl, tmp, lane);
    double *tg = Tvc + c.dt->nodeT[d] + i * 2LL * q;
    for (int u = lane; u < q; u += 32) { tg[u] = th[u]; tg[q + u] = tl[u]; }
    if (lane == 0) {
      Acc2 A = acc2(hv[2 * (2 * node + 1)]);
      acc_add_dd(A, hv[2 * (2 * node + 2)], hv[2 * (2 * node + 2) + 1]);
      A.c += hv[2 * (2 * node + 1) + 1];
      for (int u = 0; u < r; u++) acc_fma_dd(A, -g1[Kd + u], th[u], tl[u]);
      for (int u = 0; u < r; u++) acc_fma_dd(A, -g2[Kd + u], th[r + u], tl[r + u]);
      acc_dd(A, hv[2 * node], hv[2 * node + 1]);
    }
  }
  __syncthreads();
  double *gc = V + c.dt->nodeV[d] + i * (long long)Kd;
  for (int a = t; a < Kd; a += LT) {
    Acc2 A = acc2(g1[a]);
    acc_add(A, g2[a]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)(r + u) * ldb + a], th[u], tl[u]);
    for (int u = 0; u < r; u++) acc_fma_dd(A, -B[(long long)u * ldb + a], th[r + u], tl[r + u]);
    gc[a] = acc_val(A);
  }
  __syncthreads();
}

// f = t_c + T_c w_c with `parts` lanes per row u (interleaved a), partials combined by xor shuffles.
// t_c (hi, lo) of row u: from the up pass, or -- for the right-hand side fused into the factorization -- column 0
// of T_c = S_c^{-1} B_c (the factorization's compensated pair)
__device__ __forceinline__ void t_of(const SolveCtx &c, const double *tg, const double *Th, const double *Tl, int ldb,
                                     int q, int u, double &hi, double &lo) {
  if (c.fused) { hi = Th[(long long)u * ldb - c.aug]; lo = Tl[(long long)u * ldb - c.aug]; }
  else { hi = tg[u]; lo = tg[q + u]; }
}

__device__ void tree_down_node(const SolveCtx &c, int d, long long i, int col, int lane) {
  double *const V = c.V + col * c.vcol, *const Tvc = c.Tv + col * c.tcol;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const int ldb = c.dt->Kf[d];
  const double *wc = V + c.dt->nodeV[d] + i * (long long)Kd;
  const long long qK = (long long)q * ldb;
  const double *Th = c.BTpool + c.dt->nodeBT[d] + i * 3LL * qK + qK + c.aug;    // ancestor columns of T_c
  const double *Tl = Th + qK;
  const double *tg = Tvc + c.dt->nodeT[d] + i * 2LL * q;
  double *w1 = V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  double *w2 = w1 + K1;
  int parts = 1;
  while (parts * 2 * q <= 32 && parts < 16) parts *= 2;
  const int part = lane % parts;
  for (int u0 = 0; u0 < q; u0 += 32 / parts) {
    const int u = u0 + lane / parts;
    Acc2 A = acc2(0.0);
    if (u < q) {
      if (part == 0) { double th0, tl0; t_of(c, tg, Th, Tl, ldb, q, u, th0, tl0); A = acc2(th0); A.c += tl0; }
      const double *thu = Th + (long long)u * ldb, *tlu = Tl + (long long)u * ldb;
      int a = part;
      for (; a + 3 * parts < Kd; a += 4 * parts) {      // 4 iterations of loads in flight
        const double w0 = wc[a], w1v = wc[a + parts], w2v = wc[a + 2 * parts], w3 = wc[a + 3 * parts];
        const double h0 = thu[a], h1 = thu[a + parts], h2 = thu[a + 2 * parts], h3 = thu[a + 3 * parts];
        const double l0 = tlu[a], l1 = tlu[a + parts], l2 = tlu[a + 2 * parts], l3 = tlu[a + 3 * parts];
        acc_fma_dd(A, w0, h0, l0); acc_fma_dd(A, w1v, h1, l1); acc_fma_dd(A, w2v, h2, l2); acc_fma_dd(A, w3, h3, l3);
      }
      for (; a < Kd; a += parts) acc_fma_dd(A, wc[a], thu[a], tlu[a]);
    }
    for (int o = 1; o < parts; o <<= 1) {
      const double s2 = __shfl_xor_sync(0xffffffffu, A.s, o), c2 = __shfl_xor_sync(0xffffffffu, A.c, o);
      acc_add(A, s2); A.c += c2;
    }
    if (u < q && part == 0) {
      const double f = acc_val(A);
      if (u < r) w1[Kd + u] = -f; else w2[Kd + u - r] = -f;
    }
  }
  for (int a = lane; a < Kd; a += 32) { const double v = wc[a]; w1[a] = v; w2[a] = v; }
}

// Down pass of node i at depth d: f_u = t_u + sum_a w_c[a] T[u, a] (compensated), w_c1 = [w_c; -f_u (u < r)],
// w_c2 = [w_c; -f_u (u >= r)].  One warp takes the rows u = u0, u0 + ustep, ... in batches of 4 with the lanes over
// a (all loads of a batch in flight together, then a 5-round dd butterfly per row).  Warp per node (u0 = 0,
// ustep = 1) or, for levels with few nodes, a CTA per node (u0 = warp, ustep = warps).
__device__ void tree_down_rows(const SolveCtx &c, int d, long long i, int col, int lane, int u0, int ustep, bool copy_w) {
  double *const V = c.V + col * c.vcol, *const Tvc = c.Tv + col * c.tcol;
  const int r = c.dt->rdep[d + 1], q = 2 * r, Kd = c.dt->Kdim[d], K1 = c.dt->Kdim[d + 1];
  const int ldb = c.dt->Kf[d];
  const double *wc = V + c.dt->nodeV[d] + i * (long long)Kd;
  const long long qK = (long long)q * ldb;
  const double *Th = c.BTpool + c.dt->nodeBT[d] + i * 3LL * qK + qK + c.aug;
  const double *Tl = Th + qK;
  const double *tg = Tvc + c.dt->nodeT[d] + i * 2LL * q;
  double *w1 = V + c.dt->nodeV[d + 1] + (2 * i) * (long long)K1;
  double *w2 = w1 + K1;
  constexpr int UB = 4;
  for (int ub = u0; ub < q; ub += UB * ustep) {
    Acc2 A[UB];
#pragma unroll
    for (int x = 0; x < UB; x++) A[x] = acc2(0.0);
    for (int a0 = 0; a0 < Kd; a0 += 64) {      // 2 entries per lane per row and chunk
      const int aa = a0 + lane, ab = a0 + 32 + lane;
      const double wa = aa < Kd ? wc[aa] : 0.0, wb = ab < Kd ? wc[ab] : 0.0;
      double h[UB][2], l[UB][2];
#pragma unroll
      for (int x = 0; x < UB; x++) {
        const int u = ub + x * ustep;
        const bool ok = u < q;
        const double *thu = Th + (long long)(ok ? u : 0) * ldb, *tlu = Tl + (long long)(ok ? u : 0) * ldb;
        h[x][0] = (ok && aa < Kd) ? thu[aa] : 0.0; l[x][0] = (ok && aa < Kd) ? tlu[aa] : 0.0;
        h[x][1] = (ok && ab < Kd) ? thu[ab] : 0.0; l[x][1] = (ok && ab < Kd) ? tlu[ab] : 0.0;
      }
#pragma unroll
      for (int x = 0; x < UB; x++) { acc_fma_dd(A[x], wa, h[x][0], l[x][0]); acc_fma_dd(A[x], wb, h[x][1], l[x][1]); }
    }
#pragma unroll
    for (int x = 0; x < UB; x++)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, A[x].s, o), c2 = __shfl_xor_sync(0xffffffffu, A[x].c, o);
        acc_add(A[x], s2); A[x].c += c2;
      }
    if (lane == 0) {
#pragma unroll
      for (int x = 0; x < UB; x++) {
        const int u = ub + x * ustep;
        if (u >= q) break;
        double th0, tl0;
        t_of(c, tg, Th, Tl, ldb, q, u, th0, tl0);
        acc_add(A[x], th0); A[x].c += tl0;
        const double f = acc_val(A[x]);
        if (u < r) w1[Kd + u] = -f; else w2[Kd + u - r] = -f;
      }
    }
  }
  if (copy_w) for (int a = lane; a < Kd; a += 32) { const double v = wc[a]; w1[a] = v; w2[a] = v; }
}

// ---------------------------------------------------------------------------------------------
// the persistent cooperative kernel
// ---------------------------------------------------------------------------------------------
// RB = 1: one right-hand side at a time through the leaves (two CTAs per SM); RB = 8: the leaves take 8 columns per
// pass (k_solve<8>, larger shared state: one CTA per SM).  The tree levels are the same code.
template <int RB, bool XG = false>
__global__ void __launch_bounds__(LT, (RB == 1 ? 2 : 1)) k_solve(SolveCtx c0, Phases ph) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  // RB = 1: the leaf scratch is static; RB = 8: it is too large for static shared memory and sits after the X tiles
  __shared__ typename std::conditional<RB == 1, LeafSmem, int>::type S1;
  auto &S = *[&]() {
    if constexpr (RB == 1) return &S1;
    else return reinterpret_cast<LeafSmem8 *>(sm + c0.xdoubles);
  }();
  __shared__ DepthTab sdt;                     // the per-depth tables, read by every tree node
  for (int i = threadIdx.x; i < (int)(sizeof(DepthTab) / 8); i += LT) ((long long *)&sdt)[i] = ((const long long *)c0.dt)[i];
  __syncthreads();
  SolveCtx c = c0;
  c.xglobal = XG;                              // compile-time: the staged-X path carries no run-time test
  c.dt = &sdt;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *sX = sm;
  const long long gw = (long long)blockIdx.x * NWL + warp, nw = (long long)gridDim.x * NWL;
  const bool stamp = c.stamps && blockIdx.x == 0 && threadIdx.x == 0;
  int ns = 0;
  const int R = c.R;
  if (stamp) c.stamps[ns++] = gtimer();
  if (ph.leaf_up) {
    if constexpr (RB == 1) leaf_up_phase(c, sX, S); else leaf_up_phase8(c, sX, S);
    grid.sync();
    if (stamp) c.stamps[ns++] = gtimer();
  }
  {
    // work items of a level: (node, right-hand side) pairs, node fastest
    const long long gwt = (long long)blockIdx.x * c.tree_warps + warp, nwt = (long long)gridDim.x * c.tree_warps;
    for (int d = ph.up_hi; d >= ph.up_lo; d--) {
      long long i0, cnt;
      own_range(c, d, i0, cnt);
      const long long items = cnt * R;
      if (items <= gridDim.x) {                // few items: one CTA each
        if (blockIdx.x < items) tree_up_node_cta(c, d, i0 + blockIdx.x % cnt, (int)(blockIdx.x / cnt), sm);
      } else if (warp < c.tree_warps) {
        for (long long j = gwt; j < items; j += nwt)
          tree_up_node(c, d, i0 + j % cnt, (int)(j / cnt), sm + (size_t)warp * c.tree_scratch, lane);
      }
      grid.sync();
      if (stamp) c.stamps[ns++] = gtimer();
    }
  }
  if (!ph.down) return;
  for (int d = 0; d < c.kappa; d++) {
    long long i0, cnt;
    own_range(c, d, i0, cnt);
    const long long items = cnt * R;
    if (items >= 8 && items <= gridDim.x) {   // few (but not very few) items: one CTA each, its warps split the rows
      if (blockIdx.x < items)
        tree_down_rows(c, d, i0 + blockIdx.x % cnt, (int)(blockIdx.x / cnt), lane, warp, NWL, warp == 0);
    } else {
      for (long long j = gw; j < items; j += nw) tree_down_node(c, d, i0 + j % cnt, (int)(j / cnt), lane);
    }
    grid.sync();
    if (stamp) c.stamps[ns++] = gtimer();
  }
  if constexpr (RB == 1) leaf_down_phase(c, sX, S); else leaf_down_phase8(c, sX, S);
  if (stamp) c.stamps[ns++] = gtimer();
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

}  // namespace

// every rank returns the full solution: allgather the sorted row slices, un-permute into x
static hodlr_status unshard(hodlr_s *h, double *x) {
  hodlr_status st;
    const long long id = (1LL << h->tsplit) - 1 + h->grank;
    const long long rlo = h->h_lo[id], rm = h->h_hi[id] - rlo;
    double *send = h->xshard + h->n, *recv = send + h->rows_max;
    k_pack_rows<<<(int)((rm + 255) / 256), 256, 0, h->st>>>(h->xshard, rlo, rm, send);
    HLAUNCH(h, "k_pack_rows");
    st = hodlr_allgather(h, send, recv, sizeof(double) * h->rows_max);
    if (st != HODLR_OK) return st;
    const long long tot = (long long)h->nranks * h->rows_max;
    k_unshard<<<(int)((tot + 255) / 256), 256, 0, h->st>>>(recv, h->d_rowlo, h->nranks, h->rows_max, h->n, h->perm, x);
    HLAUNCH(h, "k_unshard");
    return HODLR_OK;
}

// y, x: nrhs columns with leading dimension ld (device; x may be NULL when up_only).  up_only: stop after the up pass
// (h_root = y^T C^{-1} y of column r in hvec[r * 2 nnodes]).  fused: y is the right-hand side the factorization
// carried (hodlr_factor_solve, nrhs = 1): its leaf and tree up passes are already in the factors (Pi_c[0, :] = g_c,
// T_c[:, 0] = t_c), so only the down passes run.  Up to SOLVE_RMAX columns per launch share every staged leaf
// inverse X and every L2-resident panel E_l, and the tree levels run their (node, column) pairs in parallel.
hodlr_status hodlr_solve_impl(hodlr_s *h, const double *y, double *x, int64_t nrhs, int64_t ld, bool up_only, bool fused) {
  const int kappa = h->kappa;
  DepthTab &dt = h->dt;
  if (h->leaf_max > VMAX || dt.Kdim[kappa] > KMAX_SOLVE)
    return hodlr_set_error(HODLR_EINVAL, "solve: leaf size %d > %d or K = %d > %d", h->leaf_max, VMAX, dt.Kdim[kappa], KMAX_SOLVE);
  // per-launch columns: one when sharded (the exchanges are per column) or fused
  const int RM = (h->nranks > 1 || fused) ? 1 : (int)std::min<int64_t>(nrhs, SOLVE_RMAX);
  if (!h->Vpool || h->solve_cols < RM) {
    long long vTot = 0, tTot = 0;
    for (int e = 0; e <= kappa; e++) { dt.nodeV[e] = vTot; vTot += (1LL << e) * (long long)dt.Kdim[e]; }
    for (int d = 0; d < kappa; d++) { dt.nodeT[d] = tTot; tTot += (1LL << d) * 4LL * dt.rdep[d + 1]; }
    h->vcol = vTot > 0 ? vTot : 1; h->tcol = tTot > 0 ? tTot : 1; h->hcol = 2 * h->nnodes;
    h->Vpool = (double *)hodlr_dalloc(h, sizeof(double) * h->vcol * RM);
    h->Tvec = (double *)hodlr_dalloc(h, sizeof(double) * h->tcol * RM);
    h->hvec = (double *)hodlr_dalloc(h, sizeof(double) * h->hcol * RM);
    if (!h->Vpool || !h->Tvec || !h->hvec) return hodlr_set_error(HODLR_ENOMEM, "solve: device allocation failed");
    h->solve_cols = RM;
    HCUDA(cudaMemcpyAsync(h->d_dt, &dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));
  }
  SolveCtx c;
  c.n = h->n; c.ninternal = h->ninternal; c.nleaves = h->nleaves; c.kappa = kappa; c.K = dt.Kdim[kappa];
  c.T = h->ltiles; c.grank = h->grank; c.tsplit = h->tsplit;
  c.lo = h->lo; c.hi = h->hi; c.perm = h->perm; c.Xh = h->Xh; c.ldx = h->ldx; c.rank = h->rank; c.dt = h->d_dt;
  c.Lf = h->Lf; c.lstride = h->lstride; c.Spool = h->Spool; c.BTpool = h->BTpool;
  c.Uf = h->nonspd ? h->Uf : nullptr; c.lperm = h->nonspd ? h->lperm : nullptr;
  c.V = h->Vpool; c.Tv = h->Tvec; c.hv = h->hvec; c.y = y; c.x = x; c.flags = h->dflags;
  c.vcol = h->vcol; c.tcol = h->tcol; c.hcol = h->hcol; c.ldy = ld;
  c.aug = h->aug; c.fused = fused ? 1 : 0;
  hodlr_own_nodes(h, kappa, &c.leaf0, &c.nown);
  c.xsorted = nullptr;
  if (h->nranks > 1 && !up_only) {
    if (!h->xshard) {
      h->xshard = (double *)hodlr_dalloc(h, sizeof(double) * ((size_t)h->n + (size_t)h->rows_max * (h->nranks + 1)));
      if (!h->xshard) return hodlr_set_error(HODLR_ENOMEM, "solve: device allocation failed");
    }
    c.xsorted = h->xshard;
  }
  // dynamic shared memory: the leaf staging (X tiles) or the tree-up scratch of every warp
  const int Rr = 8 * h->ltiles;
  size_t qmax = 0;
  for (int d = 0; d < kappa; d++) qmax = std::max(qmax, 2 * (size_t)dt.rdep[d + 1]);
  c.tree_scratch = (long long)std::max<size_t>(1, 2 * qmax * qmax + 5 * qmax);   // kappa = 0: no tree
  int maxsm = 0, nsm = 0;
  HCUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  HCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
  const bool rb8 = RM > 1 && !h->nonspd;         // LU leaves: the one-column leaf phases (R20)
  const void *kfun = rb8 ? (const void *)k_solve<8> : (const void *)k_solve<1>;   // (X global: <RB, true> below)
  cudaFuncAttributes fa;
  HCUDA(cudaFuncGetAttributes(&fa, kfun));     // (static shared memory: the same for both X modes)
  const size_t static_smem = fa.sharedSizeBytes;
  const size_t avail = ((size_t)maxsm - static_smem - 256) / sizeof(double);
  // Stage only X (68 KB at p = 128) and read E from global memory: two CTAs per SM overlap one leaf's loads with
  // the other's arithmetic (measured faster than staging X + E at one CTA per SM)
  size_t x_db0 = 64 * (size_t)(h->ltiles * (h->ltiles + 1) / 2);
  const size_t x_extra = rb8 ? (sizeof(LeafSmem8) + 7) / 8 : 0;
  c.xglobal = x_db0 + x_extra > avail ? 1 : 0;   // (leaves of more than ~235 points: X read from global memory)
  if (c.xglobal) {
    x_db0 = 0;
    kfun = rb8 ? (const void *)k_solve<8, true> : (const void *)k_solve<1, true>;
  }
  c.xdoubles = (long long)x_db0;
  // RB = 8: the 8-column leaf scratch follows the X tiles in dynamic shared memory
  const size_t x_db = x_db0 + x_extra;
  const size_t need = std::max(x_db, (size_t)c.tree_scratch);
  if (need > avail)
    return hodlr_set_error(HODLR_EINVAL, "solve: leaf inverse (%d rows) or coupling size %zu exceeds shared memory", Rr, qmax);
  const size_t half = rb8 ? avail : std::min(avail, (size_t)(((size_t)maxsm / 2 - static_smem - 1024) / sizeof(double)));
  const size_t dsm_d = std::max(x_db, std::min(half, (size_t)NWL * (size_t)c.tree_scratch));
  c.tree_warps = (int)std::min<size_t>(NWL, dsm_d / (size_t)c.tree_scratch);
  const size_t dsm = sizeof(double) * dsm_d;
  static int trace = -1;
  if (trace < 0) { const char *ev = getenv("HODLR_TRACE"); trace = ev && atoi(ev) ? 1 : 0; }
  c.stamps = nullptr;
  if (trace) {
    if (!h->stamps) h->stamps = (unsigned long long *)hodlr_dalloc(h, sizeof(unsigned long long) * 128);
    c.stamps = h->stamps;
  }
  HCUDA(hodlr_allow_smem(kfun, h->dev));
  int per_sm = 0;
  HCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfun, LT, dsm));
  if (per_sm < 1) return hodlr_set_error(HODLR_EINVAL, "solve: kernel does not fit on an SM");
  const int grid = nsm * std::min(per_sm, 2);             // persistent: every CTA resident (cooperative launch)
  auto launch = [&](Phases ph) -> hodlr_status {
    void *args[] = {(void *)&c, (void *)&ph};
    HCUDA(cudaLaunchCooperativeKernel(kfun, dim3(grid), dim3(LT), args, dsm, h->st));
    HLAUNCH(h, "k_solve");
    return HODLR_OK;
  };
  ph_begin(h, PH_SLEAF_UP);
  hodlr_status st = HODLR_OK;
  for (int64_t j0 = 0; j0 < nrhs && st == HODLR_OK; j0 += RM) {
    c.R = (int)std::min<int64_t>(RM, nrhs - j0);
    c.y = y + j0 * ld; c.x = x ? x + j0 * ld : nullptr;
    if (fused) {
      st = launch(Phases{0, -1, 0, 1});
    } else if (h->nranks > 1 && h->tsplit > 0) {
      // leaf up + own subtree levels, exchange of the depth-t projections, then the rest
      st = launch(Phases{1, kappa - 1, h->tsplit, 0});
      if (st != HODLR_OK) return st;
      const int t = h->tsplit;
      const long long Kt = dt.Kdim[t];
      double *gb = h->Vpool + dt.nodeV[t];
      st = hodlr_allgather(h, gb + h->grank * Kt, gb, sizeof(double) * (Kt > 0 ? Kt : 1));
      if (st != HODLR_OK) return st;
      double *hb = h->hvec + 2 * ((1LL << t) - 1);
      st = hodlr_allgather(h, hb + 2 * h->grank, hb, sizeof(double) * 2);
      if (st != HODLR_OK) return st;
      st = launch(Phases{0, t - 1, 0, up_only ? 0 : 1});
    } else {
      st = launch(Phases{1, kappa - 1, 0, up_only ? 0 : 1});
    }
    if (st != HODLR_OK) return st;
    if (h->nranks > 1 && !up_only) st = unshard(h, c.x);
  }
  if (st != HODLR_OK) return st;
  ph_end(h, PH_SLEAF_UP);
  if (trace && c.stamps) {       // per-phase device times (block 0's view, after each grid barrier)
    unsigned long long s[80];
    HCUDA(cudaMemcpyAsync(s, c.stamps, sizeof(s), cudaMemcpyDeviceToHost, h->st));
    HCUDA(cudaStreamSynchronize(h->st));
    const int nst = (up_only ? 1 + kappa : 2 + 2 * kappa) + 1;
    fprintf(stderr, "[hodlr solve phases us]");
    for (int k = 1; k < nst && k < 64; k++) fprintf(stderr, " %.1f", 1e-3 * (double)(s[k] - s[k - 1]));
    fprintf(stderr, "\n");
  }
  return HODLR_OK;
}
