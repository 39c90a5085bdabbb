// factor.cu -- G4/G5/G7: the "Factor" phase (Fig. 6) in projected-Gram form.
//
// Paper: apply K_kappa^{-1} (leaf blocks) and then every finer level's block inverse to each
// coarser left factor (Fig. 6 lines 8-12), forming S_c = [[I, V^T K_c2^{-1} V], [U^T K_c1^{-1} U, I]]
// at each node (equation_Low_Rank_Update + SMW).
//
// B200 form (same factorization, never materialises the processed panel):
// for every node a define Pi_a = E_a^T K_aa^{-1} E_a where E_a = the original ACA left factors of
// all ancestors of a (and a itself) restricted to the rows of a.
//   leaf:  Pi_l = Z^T Z,  Z = L^{-1} E_l,  A_l = L L^T     (leaf_mma.cu fast path, k_leaf_factor fallback)
//   node c at depth d with children c1, c2, s = depth-(d+1) columns, a = columns of depths <= d:
//     S_c = [[I, Pi_c2[s,s]], [Pi_c1[s,s], I]],  B_c = [Pi_c2[s,a]; Pi_c1[s,a]],  T_c = S_c^{-1} B_c
//     Pi_c = Pi_c1[a,a] + Pi_c2[a,a] - B_c[r:]^T T_c[:r] - B_c[:r]^T T_c[r:]   (k_tree_factor)
// because E^T K_cc^{-1} E = E^T D^{-1} E - E^T D^{-1} L S^{-1} R D^{-1} E with D = diag(K_c1, K_c2),
// L = blockdiag(U, V), R = [[0, V^T], [U^T, 0]] (SMW).  log det C = sum_l 2 sum log L_ii +
// sum_c log det S_c (Sylvester + multiplicativity).
// The Schur updates cancel heavily (the top-level S_c reach cond ~1e11), so T_c is kept as a
// double-double pair and Pi_c is accumulated with compensated arithmetic.
#include "hodlr_internal.cuh"
#include <cooperative_groups.h>
#include <vector>
#ifndef TREE_PLAIN_LEVELS
#define TREE_PLAIN_LEVELS 3
#endif
#ifndef TREE_DEEP64_SMEM
#define TREE_DEEP64_SMEM (20 * 1024)   // deep runs whose nodes need at most this run 64-thread CTAs, 11-12 per SM
#endif
#ifndef TREE_DEEP_SMEM
#define TREE_DEEP_SMEM (36 * 1024)  // deep-run levels keep 6 CTAs per SM (their shared memory per node at most this)
#endif
#ifndef TREE_NARROW_MIN
#define TREE_NARROW_MIN (4 * 148)   // levels with at least this many nodes (and q <= 16) use the 128-thread CTAs
#endif
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

namespace cg = cooperative_groups;

namespace {

constexpr int LT = 256;      // threads per leaf CTA (fallback kernel)
constexpr int TT = 256;      // threads per tree CTA

__device__ __forceinline__ long long P(long long i, long long j) { return i * (i + 1) / 2 + j; }

// ---------------------------------------------------------------------------------------------
// Fallback leaf kernel (any leaf size; scalar FP64): Cholesky, Z = L^{-1} E, Pi = Z^T Z.
// Outputs in the shared storage formats (L tiles + Linv tiles, packed Pi).
// ---------------------------------------------------------------------------------------------
struct LeafCtx {
  KParams kp;
  long long n, ninternal, nleaves;
  int kappa, K, ldz, T;
  const double *xs;
  const long long *lo, *hi;
  const double *Xh; long long ldx;
  const int *rank;
  const DepthTab *dt;
  double *Lf; long long lstride;
  double *Pi;               // leaf Pi storage, packed K(K+1)/2 per leaf
  double *leaf_ld;
  int *flags;
  double *scratch;          // per-CTA fallback storage when shared memory is too small
  long long scratch_per_cta;
  int use_smem;
  int mmax;                 // max leaf size
  long long leaf0, nown;    // this rank's leaves [leaf0, leaf0 + nown)
  long long lsz;            // packed triangle capacity mmax(mmax+1)/2 + 1
  int aug;                  // fused right-hand side: column 0 of the panel is y (gathered through perm)
  const double *y; const long long *perm;
  const KParams *kps; long long nseg;     // batched handle (kp_of), or NULL
};

// Threads: any multiple of 32 up to 1024 (256 with everything in shared memory; 1024 and one CTA per SM when the
// leaf lives in global scratch, so that all CTAs' scratch -- 148 x ~0.4 MB -- stays in L2: with 592 CTAs of 256
// threads the 247 MB of scratch thrashed L2, 106 GB of DRAM traffic and 105 ms for the paper's n = 10^6 / leaf 128 row).
__global__ void __launch_bounds__(1024) k_leaf_factor(LeafCtx c) {
  extern __shared__ double sm[];
  __shared__ long long colsrc[1024];
  __shared__ int bad;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nth = blockDim.x, nw = nth >> 5;
  const int K = c.K, ldz = c.ldz;
  double *colj = sm;                           // mmax: the current Cholesky column
  double *base = c.use_smem ? sm + c.mmax : c.scratch + (long long)blockIdx.x * c.scratch_per_cta;
  for (long long leaf = c.leaf0 + blockIdx.x; leaf < c.leaf0 + c.nown; leaf += gridDim.x) {
    const long long id = c.ninternal + leaf, lo = c.lo[id], m = c.hi[id] - lo;
    const KParams kp = kp_of(c.kp, c.kps, c.nseg, lo);
    double *xl = base;                       // m
    double *L = base + c.mmax;               // packed lower m(m+1)/2
    double *Z = L + c.lsz;                   // m x ldz
    double *Zb = Z + (long long)c.mmax * ldz;   // 8 x ldz: one row block of Z = X E before it replaces E's rows
    for (long long i = t; i < m; i += nth) xl[i] = c.xs[lo + i];
    if (t == 0) bad = 0;
    __syncthreads();
    for (long long i = warp; i < m; i += nw) {          // assemble the packed lower triangle, a warp per row
      double *Li = L + P(i, 0);
      for (long long j = lane; j <= i; j += 32) {
        double v = kp.dim > 1 ? kval_nd_fast(kp, c.xs, lo + i, lo + j) : kval(kp, xl[i] - xl[j]);
        if (i == j) v += sig2(kp, lo + i);
        Li[j] = v;
      }
    }
    __syncthreads();
    for (long long j = 0; j < m; j++) {        // right-looking Cholesky A = L L^T
      // The scaled column j also goes to shared memory (colj): the trailing update reads both of its factors
      // there, so its only global accesses are the coalesced read-modify-writes of the packed rows, four rows per
      // warp in flight.
      const double d = L[P(j, j)];
      const bool ok = d > 0.0;
      const double ljj = sqrt(ok ? d : 1.0);
      for (long long i = j + 1 + t; i < m; i += nth) { const double v = L[P(i, j)] / ljj; colj[i] = v; L[P(i, j)] = v; }
      __syncthreads();
      if (t == 0) { L[P(j, j)] = ljj; if (!ok) bad = 1; }
      constexpr int NR = 4;                       // rows per warp in flight
      for (int i0 = (int)j + 1 + warp; i0 < (int)m; i0 += NR * nw) {
        double *Lr[NR]; double lr[NR]; int er[NR];
#pragma unroll
        for (int q = 0; q < NR; q++) {
          const int iq = i0 + q * nw;
          const bool v = iq < (int)m;
          Lr[q] = L + P(v ? iq : i0, 0); lr[q] = v ? colj[iq] : 0.0; er[q] = v ? iq : (int)j;   // er = j: no such row
        }
        const int ke = max(max(er[0], er[1]), max(er[2], er[3]));
        for (int k = (int)j + 1 + lane; k <= ke; k += 32) {
          const double ck = colj[k];
          double v[NR];
#pragma unroll
          for (int q = 0; q < NR; q++) v[q] = k <= er[q] ? Lr[q][k] : 0.0;
#pragma unroll
          for (int q = 0; q < NR; q++) if (k <= er[q]) Lr[q][k] = v[q] - lr[q] * ck;
        }
      }
      __syncthreads();
    }
    if (t == 0) {
      double s = 0.0;
      for (long long j = 0; j < m; j++) s += log(L[P(j, j)]);
      c.leaf_ld[leaf] = 2.0 * s;
      if (bad) { atomicAdd(&c.flags[1], 1); atomicMin(&c.flags[2], (int)id); }
    }
    // X = L^{-1} as fragment-order tiles (identity padding beyond m): forward substitution L x = e_j, four lanes
    // per column (each a quarter of the row's dot product, summed by shuffles; fallback path -- the fast path forms
    // X on the tensor pipe)
    const int T = c.T, NT = T * (T + 1) / 2;
    double *Lg = c.Lf + leaf * c.lstride;
    for (long long p = t; p < (long long)NT * 64; p += nth) Lg[p] = 0.0;
    __syncthreads();
    {
      const int sub = lane & 3;
      const unsigned gmask = 0xFu << (lane & ~3);
      for (int j = t >> 2; j < 8 * T; j += nth >> 2) {
        if (j >= m) { if (sub == 0) Lg[tix(j >> 3, j >> 3) * 64 + fo(j & 7, j & 7)] = 1.0; continue; }
        const int Jt = j >> 3, jc = j & 7;
        for (int i = j; i < m; i++) {
          const double *Li = L + P(i, 0);
          double s = 0.0;
          const double *Xc = Lg + fo(sub, jc);                       // rows sub and sub + 4 of each tile of column j
          for (int Kt = Jt; 8 * Kt < i; Kt++) {
            const double *Xt = Xc + tix(Kt, Jt) * 64;
            const int k0 = 8 * Kt + sub, k1 = k0 + 4;
            if (k0 >= j && k0 < i) s += Li[k0] * Xt[0];
            if (k1 >= j && k1 < i) s += Li[k1] * Xt[16];
          }
          s += __shfl_xor_sync(gmask, s, 1);
          s += __shfl_xor_sync(gmask, s, 2);
          if (sub == 0) Lg[tix(i >> 3, Jt) * 64 + fo(i & 7, jc)] = ((i == j ? 1.0 : 0.0) - s) / Li[i];
          __syncwarp(gmask);
        }
      }
    }
    if (K > 0) {
      if (t == 0) {   // column map: [rhs,] depth 1 .. kappa; zero beyond each block's rank
        long long a = id;
        for (int e = c.kappa; e >= 1; e--) {
          long long b = (a - 1) / 2;
          int rb = c.rank[b];
          for (int q = 0; q < c.dt->rdep[e]; q++)
            colsrc[c.aug + c.dt->Kdim[e - 1] + q] = q < rb ? c.dt->colbase[e] + q : -1;
          a = b;
        }
        if (c.aug) colsrc[0] = -2;
      }
      __syncthreads();                 // colsrc, and X complete
      for (int col = warp; col < K; col += nw) {          // E: the leaf's rows of its ancestors' factor columns
        const long long src = colsrc[col];
        for (long long ib = 0; ib < m; ib += 256) {       // 8 loads in flight per lane
          double v[8];
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const long long i = ib + lane + 32 * q;
            v[q] = 0.0;
            if (i < m) {
              if (src >= 0) v[q] = c.Xh[src * c.ldx + lo + i];
              else if (src == -2) v[q] = c.y[c.perm[lo + i]];
            }
          }
#pragma unroll
          for (int q = 0; q < 8; q++) {
            const long long i = ib + lane + 32 * q;
            if (i < m) { if (src == -2 && !isfinite(v[q])) atomicOr(&c.flags[3], 1); Z[i * ldz + col] = v[q]; }
          }
        }
      }
      __syncthreads();
      // Z <- X E in place, row blocks from the bottom up (block I needs E's rows <= 8 I + 7 only; the block is
      // staged in Zb so that every thread has read E's rows of the block before they are replaced)
      for (int I = (int)((m - 1) >> 3); I >= 0; I--) {
        const int rows = (int)(m - 8 * I < 8 ? m - 8 * I : 8);
        for (int o = t; o < rows * K; o += nth) {
          const int r = o / K, col = o - r * K, i = 8 * I + r;
          double s = 0.0;
          const double *Xr = Lg + tix(I, 0) * 64 + r * 4;            // row r of the tiles (I, 0 .. I): fo(r, c)
          const double *Zc = Z + col;
          for (int J = 0; J < I; J++, Xr += 64, Zc += 8 * ldz) {
#pragma unroll
            for (int cc = 0; cc < 8; cc++) s += Xr[(cc >> 2) * 32 + (cc & 3)] * Zc[cc * ldz];
          }
          for (int cc = 0; cc <= r; cc++) s += Xr[(cc >> 2) * 32 + (cc & 3)] * Zc[cc * ldz];
          Zb[r * ldz + col] = s;
        }
        __syncthreads();
        for (int o = t; o < rows * K; o += nth) {
          const int r = o / K, col = o - r * K;
          Z[(long long)(8 * I + r) * ldz + col] = Zb[r * ldz + col];
        }
        __syncthreads();
      }
      double *Pl = c.Pi + leaf * ((long long)K * (K + 1) / 2);   // Pi_l = Z^T Z, packed lower
      const long long npk = (long long)K * (K + 1) / 2;
      for (long long p = t; p < npk; p += nth) {
        long long a = (long long)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
        while (a * (a + 1) / 2 > p) a--;
        while ((a + 1) * (a + 2) / 2 <= p) a++;
        long long b = p - a * (a + 1) / 2;
        double s = 0.0;
        for (long long i = 0; i < m; i++) s += Z[i * ldz + a] * Z[i * ldz + b];
        Pl[p] = s;
      }
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------------------------
// Leaves of a kernel that is not positive definite (MQ, BIHARM; NEXT-2, R20): A_l = P^T L U by LU with
// partial pivoting (the oracle's O5': row of max |.|, first index on ties), log|det A_l| = sum log|U_ii|, the sign of
// det A_l counted into flags[10] when negative.  Stored for the solve: XL = L^{-1} (unit lower) in Lf, XU = U^{-T}
// (lower) in Uf, both as fragment-order tiles (identity padding), and the row order lperm (P b = b[lperm]), so that
// A_l^{-1} b = XU^T (XL (P b)).  Pi_l = E^T W with W = A_l^{-1} E by the LU substitutions (packed lower: row index a
// = the E side, column b = the W side, as the oracle's B entries E_s^T X_J).  One CTA per leaf; A in shared memory
// when it fits, W and the unpermuted panel E in the CTA's global scratch (L2-resident).
// ---------------------------------------------------------------------------------------------
struct LuCtx {
  LeafCtx b;
  double *Uf;              // XU tiles (lstride doubles per leaf)
  int *lperm;              // 8T ints per leaf
  int a_smem;              // A in shared memory
  double *scr; long long scr_per_cta;
};

__global__ void __launch_bounds__(LT) k_leaf_factor_lu(LuCtx lc) {
  extern __shared__ double sm[];
  __shared__ long long colsrc[1024];
  __shared__ int prm[256];
  __shared__ int s_bad, s_neg, s_p;
  const LeafCtx &c = lc.b;
  const int t = threadIdx.x, lane = t & 31;
  const int K = c.K, ldz = c.ldz, T = c.T, R8 = 8 * T;
  double *scr = lc.scr + (long long)blockIdx.x * lc.scr_per_cta;
  for (long long leaf = c.leaf0 + blockIdx.x; leaf < c.leaf0 + c.nown; leaf += gridDim.x) {
    const long long id = c.ninternal + leaf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    const KParams kp = kp_of(c.kp, c.kps, c.nseg, lo);
    double *A = lc.a_smem ? sm : scr;                          // m x m, row-major
    double *W = scr + (lc.a_smem ? 0 : (long long)m * m);      // m x ldz: P E, then A^{-1} E
    double *Eg = W + (long long)m * ldz;                      // m x ldz: E (sorted row order)
    for (int p = t; p < m * m; p += LT) {
      const int i = p / m, j = p - i * m;
      double v = kp.dim > 1 ? kval_nd_fast(kp, c.xs, lo + i, lo + j) : kval(kp, c.xs[lo + i] - c.xs[lo + j]);
      if (i == j) v += sig2(kp, lo + i);
      A[p] = v;
    }
    for (int i = t; i < 256; i += LT) prm[i] = i;
    if (t == 0) { s_bad = 0; s_neg = 0; }
    __syncthreads();
    for (int k = 0; k < m; k++) {
      if (t < 32) {                                            // pivot: first max |A[i][k]|, i >= k
        double best = -1.0; int p = m;
        for (int i = k + lane; i < m; i += 32) { const double v = fabs(A[i * m + k]); if (v > best) { best = v; p = i; } }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double b2 = __shfl_xor_sync(0xffffffffu, best, o); const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
          if (b2 > best || (b2 == best && p2 < p)) { best = b2; p = p2; }
        }
        if (lane == 0) {
          s_p = p;
          if (p != k) { const int tq = prm[k]; prm[k] = prm[p]; prm[p] = tq; s_neg ^= 1; }
        }
      }
      __syncthreads();
      const int p = s_p;
      if (p != k) for (int j = t; j < m; j += LT) { const double tq = A[k * m + j]; A[k * m + j] = A[p * m + j]; A[p * m + j] = tq; }
      __syncthreads();
      const double ukk = A[k * m + k];
      if (t == 0) { if (ukk == 0.0) s_bad = 1; if (ukk < 0.0) s_neg ^= 1; }
      const double iu = ukk != 0.0 ? ukk : 1.0;
      for (int i = k + 1 + t; i < m; i += LT) A[i * m + k] = A[i * m + k] / iu;
      __syncthreads();
      const int w = m - k - 1;
      for (int e = t; e < w * w; e += LT) {
        const int i = k + 1 + e / w, j = k + 1 + e % w;
        A[i * m + j] = fma(-A[i * m + k], A[k * m + j], A[i * m + j]);
      }
      __syncthreads();
    }
    if (t == 0) {
      double s = 0.0;
      for (int i = 0; i < m; i++) s += log(fabs(A[i * m + i]));
      c.leaf_ld[leaf] = s;
      if (s_bad) { atomicAdd(&c.flags[1], 1); atomicMin(&c.flags[2], (int)id); }
      else if (s_neg) atomicAdd(&c.flags[10], 1);
    }
    // XL = L^{-1} and XU = U^{-T} as fragment-order tiles (identity beyond m), one thread per column j
    const int NT = T * (T + 1) / 2;
    double *Lg = c.Lf + leaf * c.lstride, *Ug = lc.Uf + leaf * c.lstride;
    for (long long p = t; p < (long long)NT * 64; p += LT) { Lg[p] = 0.0; Ug[p] = 0.0; }
    for (int i = t; i < R8; i += LT) lc.lperm[leaf * R8 + i] = i < m ? prm[i] : i;
    __syncthreads();
    for (int j = t; j < R8; j += LT) {
      if (j >= m) {
        Lg[tix(j >> 3, j >> 3) * 64 + fo(j & 7, j & 7)] = 1.0;
        Ug[tix(j >> 3, j >> 3) * 64 + fo(j & 7, j & 7)] = 1.0;
        continue;
      }
      for (int i = j; i < m; i++) {                            // L x = e_j (unit diagonal)
        double s = i == j ? 1.0 : 0.0;
        for (int k = j; k < i; k++) s -= A[i * m + k] * Lg[tix(k >> 3, j >> 3) * 64 + fo(k & 7, j & 7)];
        Lg[tix(i >> 3, j >> 3) * 64 + fo(i & 7, j & 7)] = s;
      }
      for (int i = j; i < m; i++) {                            // U^T z = e_j: z_i = (d_ij - sum_k U[k][i] z_k) / U_ii
        double s = i == j ? 1.0 : 0.0;
        for (int k = j; k < i; k++) s -= A[k * m + i] * Ug[tix(k >> 3, j >> 3) * 64 + fo(k & 7, j & 7)];
        Ug[tix(i >> 3, j >> 3) * 64 + fo(i & 7, j & 7)] = s / A[i * m + i];
      }
    }
    if (K > 0) {
      if (t == 0) {   // column map: [rhs,] depth 1 .. kappa; zero beyond each block's rank
        long long a = id;
        for (int e = c.kappa; e >= 1; e--) {
          long long b = (a - 1) / 2;
          int rb = c.rank[b];
          for (int q = 0; q < c.dt->rdep[e]; q++)
            colsrc[c.aug + c.dt->Kdim[e - 1] + q] = q < rb ? c.dt->colbase[e] + q : -1;
          a = b;
        }
        if (c.aug) colsrc[0] = -2;
      }
      __syncthreads();
      for (long long p = t; p < (long long)K * m; p += LT) {
        const long long col = p / m, i = p - col * m, src = colsrc[col];
        double v = 0.0;
        if (src >= 0) v = c.Xh[src * c.ldx + lo + i];
        else if (src == -2) { v = c.y[c.perm[lo + i]]; if (!isfinite(v)) atomicOr(&c.flags[3], 1); }
        Eg[i * ldz + col] = v;
      }
      __syncthreads();
      for (int col = t; col < K; col += LT) {                  // W = U^{-1} L^{-1} P E
        for (int i = 0; i < m; i++) {
          double s = Eg[(long long)prm[i] * ldz + col];
          for (int k = 0; k < i; k++) s -= A[i * m + k] * W[(long long)k * ldz + col];
          W[(long long)i * ldz + col] = s;
        }
        for (int i = m - 1; i >= 0; i--) {
          double s = W[(long long)i * ldz + col];
          for (int k = i + 1; k < m; k++) s -= A[i * m + k] * W[(long long)k * ldz + col];
          W[(long long)i * ldz + col] = s / A[i * m + i];
        }
      }
      __syncthreads();
      double *Pl = c.Pi + leaf * ((long long)K * (K + 1) / 2);   // Pi_l = E^T W, packed lower
      const long long npk = (long long)K * (K + 1) / 2;
      for (long long p = t; p < npk; p += LT) {
        long long a = (long long)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
        while (a * (a + 1) / 2 > p) a--;
        while ((a + 1) * (a + 2) / 2 <= p) a++;
        const long long b = p - a * (a + 1) / 2;
        double s = 0.0;
        for (int i = 0; i < m; i++) s = fma(Eg[(long long)i * ldz + a], W[(long long)i * ldz + b], s);
        Pl[p] = s;
      }
    }
    __syncthreads();
  }
}

}  // namespace
#include "tree_node.cuh"
namespace {

__device__ __forceinline__ GlobalPi global_pi(const TreeCtx &c, long long i) {
  const long long K1 = c.K1, sz = K1 * (K1 + 1) / 2;
  GlobalPi g; g.P1 = c.Pi1 + (2 * i) * sz; g.P2 = c.Pi1 + (2 * i + 1) * sz; g.Kd = c.Kd;
  return g;
}

// PIDD = false: the plain Pi update (the deepest levels); true: as the level's c.dd says.  DESIGN.md 6.2.
template <bool PIDD>
__global__ void __launch_bounds__(TT, 3) k_tree_factor(TreeCtx c) {
  extern __shared__ double sm[];
  const long long i = c.i0 + blockIdx.x;
  tree_node<true, GlobalPi, 32, PIDD>(c, i, sm, global_pi(c, i));
}

// Levels with many small nodes: 128-thread CTAs (6 per SM) -- finer barrier domains, more independent nodes
// in flight per SM.  Same device code.
#ifndef TREE_PLAIN_LEVELS
#define TREE_PLAIN_LEVELS 3
#endif
#ifndef TREE_DEEP64_SMEM
#define TREE_DEEP64_SMEM (20 * 1024)   // deep runs whose nodes need at most this run 64-thread CTAs, 11-12 per SM
#endif
#ifndef TREE_DEEP_SMEM
#define TREE_DEEP_SMEM (36 * 1024)  // deep-run levels keep 6 CTAs per SM (their shared memory per node at most this)
#endif
#ifndef TREE_NARROW_MINB
#define TREE_NARROW_MINB 6
#endif
template <bool PIDD>
__global__ void __launch_bounds__(TT / 2, TREE_NARROW_MINB) k_tree_factor_narrow(TreeCtx c) {
  extern __shared__ double sm[];
  const long long i = c.i0 + blockIdx.x;
  tree_node<true, GlobalPi, 16, PIDD>(c, i, sm, global_pi(c, i));   // (q <= 16 only)
}

// The upper levels (few nodes each) in ONE persistent cooperative launch: CTAs stride over the nodes of a level, a
// grid barrier separates the levels (deepest first).  These levels were launch- and cold-start-bound one kernel per
// level (~50 us each regardless of their node count: every level's few CTAs start on SMs whose instruction caches
// hold other kernels' code -- tree_node is ~10k instructions); here every SM warms its cache once.
// The deep levels (many nodes, q <= 16) in ONE persistent launch of 128-thread CTAs: nodes are handed out by an atomic
// counter, deepest level first, and a node waits (tree_node) for its children's progress flags, so the partial last
// wave of one level is filled by the next level's nodes instead of each level's launch ending in a tail.  Deadlock-free:
// a node only waits for nodes handed out before it (to resident CTAs of the cooperative launch).
// NTD threads per node: 128, or 64 for runs of small nodes (12 per SM instead of 6: the per-node phases are latency)
template <bool PIDD, int NTD>
__global__ void __launch_bounds__(NTD, 768 / NTD) k_tree_deep(const TreeCtx *__restrict__ ctxs, int nlev,
                                                              unsigned *next) {
  extern __shared__ double sm[];
  __shared__ long long s_j;
  __shared__ int s_L;
  for (;;) {
    if (threadIdx.x == 0) {
      long long j = (long long)atomicAdd(next, 1u);
      int L = 0;
      while (L < nlev && j >= ctxs[L].cnt) { j -= ctxs[L].cnt; L++; }
      s_j = j; s_L = L;
    }
    __syncthreads();
    const int L = s_L;
    const long long j = s_j;
    __syncthreads();
    if (L >= nlev) return;
    const TreeCtx c = ctxs[L];
    tree_node<true, GlobalPi, 16, PIDD>(c, c.i0 + j, sm, global_pi(c, c.i0 + j));
  }
}

// Levels are not separated by grid barriers: a node waits (tree_node) for its children's progress flags, so a parent's
// Gauss-Jordan overlaps the children's Pi updates.  Deadlock-free: every CTA takes its nodes deepest level first, and
// the cooperative launch keeps every CTA resident.
template <bool DD>
__global__ void __launch_bounds__(TT, 2) k_tree_top(const TreeCtx *__restrict__ ctxs, int nlev) {
  extern __shared__ double sm[];
  for (int L = 0; L < nlev; L++) {
    const TreeCtx c = ctxs[L];
    for (long long j = blockIdx.x; j < c.cnt; j += gridDim.x) tree_node<DD>(c, c.i0 + j, sm, global_pi(c, c.i0 + j));
  }
}

// log det partial = leaves (left to right), then internal nodes of depth >= tsplit by depth kappa-1..tsplit,
// left to right; per-thread Neumaier over a contiguous segment, combined in order by thread 0.
// out[0] = partial, out[1] = failures seen by this rank.
constexpr int LDR_T = 1024;      // k_logdet_reduce threads
__device__ __forceinline__ void neu_add(double &S, double &C, double x) {   // Neumaier: S + C += x
  const double tt = S + x;
  if (fabs(S) >= fabs(x)) C += (S - tt) + x; else C += (x - tt) + S;
  S = tt;
}
__global__ void __launch_bounds__(LDR_T) k_logdet_reduce(const double *leaf_ld, const double *node_ld, long long nleaves,
                                                         int kappa, int tsplit, const int *flags, double *out) {
  __shared__ double ss[LDR_T], cc[LDR_T], s2[32], c2[32];
  const long long nnode = nleaves - (1LL << tsplit);     // internal nodes of depth >= tsplit
  const long long N = nleaves + nnode;
  const int t = threadIdx.x;
  long long per = (N + LDR_T - 1) / LDR_T, v0 = t * per, v1 = v0 + per < N ? v0 + per : N;
  double s = 0.0, comp = 0.0;
  // value v: leaf v, then the internal nodes of depth kappa-1 .. tsplit left to right (offset o = v - nleaves lies
  // in depth d when 2^kappa - 2^(d+1) <= o < 2^kappa - 2^d); 8 loads in flight, folded in order
  auto val = [&](long long v) -> double {
    if (v < nleaves) return leaf_ld[v];
    const long long o = v - nleaves, w = (1LL << kappa) - o;           // 2^d < w <= 2^(d+1)
    const int d = 63 - __clzll(w - 1);                                // floor(log2(w - 1))
    return node_ld[(1LL << d) - 1 + (o - ((1LL << kappa) - (2LL << d)))];
  };
  long long v = v0;
  for (; v + 8 <= v1; v += 8) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = val(v + k);
#pragma unroll
    for (int k = 0; k < 8; k++) neu_add(s, comp, x[k]);
  }
  for (; v < v1; v++) neu_add(s, comp, val(v));
  ss[t] = s; cc[t] = comp;
  __syncthreads();
  if (t < 32) {                          // fixed order: lane l folds partials 32l .. 32l+31, lane 0 folds the lanes
    double S = 0.0, Cc = 0.0;
    for (int j = 32 * t; j < 32 * t + 32; j++) { neu_add(S, Cc, ss[j]); Cc += cc[j]; }
    s2[t] = S; c2[t] = Cc;
    __syncwarp();
    if (t == 0) {
      double S2 = 0.0, C2 = 0.0;
      for (int j = 0; j < 32; j++) { neu_add(S2, C2, s2[j]); C2 += c2[j]; }
      out[0] = S2 + C2;
      out[1] = (double)flags[1];
    }
  }
}

// log det = sum of the ranks' partials (rank order) + the top-level nodes (depth tsplit-1..0, left to right);
// failures of any rank make every rank report ENOTPD.
__global__ void k_logdet_final(const double *gathered, int nranks, const double *node_ld, int tsplit, int *flags,
                               double *out) {
  if (threadIdx.x != 0) return;
  double S = 0.0, Cc = 0.0, fails = 0.0;
  auto add = [&](double x) {
    double tt = S + x;
    if (fabs(S) >= fabs(x)) Cc += (S - tt) + x; else Cc += (x - tt) + S;
    S = tt;
  };
  for (int r = 0; r < nranks; r++) { add(gathered[2 * r]); fails += gathered[2 * r + 1]; }
  for (int d = tsplit - 1; d >= 0; d--)
    for (long long i = 0; i < (1LL << d); i++) add(node_ld[(1LL << d) - 1 + i]);
  *out = S + Cc;
  if (nranks > 1 && fails > flags[1]) {
    if (flags[1] == 0) flags[2] = -1;       // failure on another rank
    flags[1] = (int)fails;
  }
}

// Batched handle: per-problem log det (problem s = blockIdx.x: its leaves left to right, then its internal nodes by
// depth kappa-1 .. tbatch, left to right -- k_logdet_reduce's order on its subtree) and y^T C_s^-1 y from the fused
// right-hand side (the aug entry of the problem root's Pi; NaN without one).  out[s], out[B + s].
__global__ void k_logdet_segments(const double *leaf_ld, const double *node_ld, int kappa, int t, const double *Pi_t,
                                  long long pi_sz, int aug, double *out) {
  __shared__ double ss[256], cc[256];
  const int s = blockIdx.x, B = gridDim.x;
  const long long Ls = 1LL << (kappa - t);               // leaves per problem
  const long long N = Ls + (Ls - 1);
  const int th = threadIdx.x;
  const long long per = (N + 255) / 256, v0 = th * per, v1 = v0 + per < N ? v0 + per : N;
  double S = 0.0, comp = 0.0;
  int dl = kappa - t - 1; long long u = 0;                // (local depth, index) of internal value v, advanced in step
  if (v0 > Ls && v0 < v1) { u = v0 - Ls; while (u >= (1LL << dl)) { u -= (1LL << dl); dl--; } }
  for (long long v = v0; v < v1; v++) {
    double x;
    if (v < Ls) x = leaf_ld[s * Ls + v];
    else {
      x = node_ld[(1LL << (t + dl)) - 1 + (long long)s * (1LL << dl) + u];
      if (++u == (1LL << dl)) { u = 0; dl--; }
    }
    const double tt = S + x;
    if (fabs(S) >= fabs(x)) comp += (S - tt) + x; else comp += (x - tt) + S;
    S = tt;
  }
  ss[th] = S; cc[th] = comp;
  __syncthreads();
  if (th == 0) {
    double T = 0.0, C = 0.0;
    for (int j = 0; j < 256; j++) {
      const double x = ss[j], tt = T + x;
      if (fabs(T) >= fabs(x)) C += (T - tt) + x; else C += (x - tt) + T;
      T = tt;
      C += cc[j];
    }
    out[s] = T + C;
    out[B + s] = aug ? Pi_t[(long long)s * pi_sz] : NAN;
  }
}

}  // namespace

hodlr_status hodlr_batch_parts(hodlr_s *h, double *d_out) {
  const int t = h->tbatch, kappa = h->kappa;
  const long long Kt = h->dt.Kf[t];
  k_logdet_segments<<<h->nbatch, 256, 0, h->st>>>(h->leaf_ld, h->node_ld, kappa, t, h->Pipool + h->dt.piOff[t],
                                                  Kt * (Kt + 1) / 2, h->aug, d_out);
  HLAUNCH(h, "k_logdet_segments");
  return HODLR_OK;
}

// Leaf factor storage (T = ceil(leaf_max / 8) tile rows, or 8 / 16 on the fast path): allocated at build time
// because the leaf Cholesky runs during the build.
hodlr_status hodlr_leaf_alloc(hodlr_s *h) {
  const int mmax = h->leaf_max;
  const int Pfast = mmax <= 64 ? 64 : (mmax <= 128 ? 128 : 0);
  const long long nl = h->nleaves;
  h->ltiles = Pfast ? Pfast / 8 : (mmax + 7) / 8;
  h->lstride = (long long)(h->ltiles * (h->ltiles + 1) / 2) * 64;      // tiles of X = L^{-1}
  h->Lf = (double *)hodlr_dalloc(h, sizeof(double) * h->lstride * nl);
  if (h->nonspd) {                 // LU leaves: U^{-T} tiles and the row order (R20)
    h->Uf = (double *)hodlr_dalloc(h, sizeof(double) * h->lstride * nl);
    h->lperm = (int *)hodlr_dalloc(h, sizeof(int) * 8 * (size_t)h->ltiles * nl);
    if (!h->Uf || !h->lperm) return hodlr_set_error(HODLR_ENOMEM, "leaf factor allocation failed");
  }
  h->leaf_ld = (double *)hodlr_dalloc(h, sizeof(double) * nl);
  if (!h->Lf || !h->leaf_ld) return hodlr_set_error(HODLR_ENOMEM, "leaf factor allocation failed");
  HCUDA(cudaMemsetAsync(h->leaf_ld, 0, sizeof(double) * nl, h->st));      // other ranks' leaves count 0
  return HODLR_OK;
}


static TreeCtx tree_ctx(hodlr_s *h, int d, long long i0) {
  const DepthTab &dt = h->dt;
  TreeCtx tc;
  tc.cnt = 0;
  // factor-side widths: Kf = Kdim (+ 1 with a fused right-hand side, which is then index 0 of every Pi)
  tc.d = d; tc.i0 = i0; tc.r = dt.rdep[d + 1]; tc.q = 2 * tc.r; tc.Kd = dt.Kf[d]; tc.K1 = dt.Kf[d + 1];
  tc.ldk = (tc.Kd + 3) & ~3;
  // Pi update in plain FP64 at the TREE_PLAIN_LEVELS deepest levels of each problem (local depth = d - tbatch, so a
  // batched handle and a single one do the same arithmetic per node), compensated above
  tc.dd = (d - h->tbatch) < (h->kappa - h->tbatch) - TREE_PLAIN_LEVELS ? 1 : 0;
  tc.Pi1 = h->Pipool + dt.piOff[d + 1]; tc.Pic = h->Pipool + dt.piOff[d];
  tc.Sst = h->Spool + dt.nodeS[d]; tc.BT = h->BTpool + dt.nodeBT[d];
  tc.node_ld = h->node_ld; tc.flags = h->dflags; tc.nonspd = h->nonspd;
  tc.ready = nullptr; tc.wait = 0; tc.r_up = d > 0 ? dt.rdep[d] : 0;
  return tc;
}

hodlr_status hodlr_factor_impl(hodlr_s *h) {
  const int kappa = h->kappa;
  DepthTab &dt = h->dt;
  for (int e = 0; e <= kappa; e++) dt.Kf[e] = dt.Kdim[e] + h->aug;
  const int K = dt.Kf[kappa];              // panel columns per leaf (+ the fused right-hand side)
  const long long nl = h->nleaves;
  // ---- storage ----
  const int mmax = h->leaf_max;
  h->node_ld = (double *)hodlr_dalloc(h, sizeof(double) * (h->ninternal > 0 ? h->ninternal : 1));
  if (!h->d_ready) h->d_ready = (int *)hodlr_dalloc(h, sizeof(int) * (size_t)(h->ninternal + 2));   // + k_tree_deep's counter
  if (!h->d_ready) return hodlr_set_error(HODLR_ENOMEM, "factor: device allocation failed");
  h->d_logdet = (double *)hodlr_dalloc(h, sizeof(double));
  long long piTot = 0, sTot = 0, btTot = 0;
  for (int e = kappa; e >= 0; e--) {
    dt.piOff[e] = piTot;
    piTot += (1LL << e) * ((long long)dt.Kf[e] * (dt.Kf[e] + 1) / 2);
  }
  for (int d = 0; d < kappa; d++) {
    long long q = 2LL * dt.rdep[d + 1];
    dt.nodeS[d] = sTot; sTot += (1LL << d) * (2 * q * q + q);
    dt.nodeBT[d] = btTot; btTot += (1LL << d) * 3 * q * dt.Kf[d];
  }
  h->Pipool = (double *)hodlr_dalloc(h, sizeof(double) * (piTot > 0 ? piTot : 1));
  h->d_treectx = (TreeCtx *)hodlr_dalloc(h, sizeof(TreeCtx) * TREE_TOP_MAXLEV);
  h->Spool = (double *)hodlr_dalloc(h, sizeof(double) * (sTot > 0 ? sTot : 1));
  h->BTpool = (double *)hodlr_dalloc(h, sizeof(double) * (btTot > 0 ? btTot : 1));
  double *ldx = (double *)hodlr_dalloc(h, sizeof(double) * 2 * (h->nranks + 1));   // log det exchange
  if (!h->node_ld || !h->d_logdet || !h->Pipool || !h->d_treectx || !h->Spool || !h->BTpool || !ldx)
    return hodlr_set_error(HODLR_ENOMEM, "factor: device allocation failed");
  HCUDA(cudaMemsetAsync(h->node_ld, 0, sizeof(double) * (h->ninternal > 0 ? h->ninternal : 1), h->st));
  HCUDA(cudaMemcpyAsync(h->d_dt, &dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));
  if (K > 1024) return hodlr_set_error(HODLR_EINVAL, "factor: K = %d ancestor columns exceeds 1024", K);
  int maxsm = 0;
  HCUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  // ---- leaves ----
  HCUDA(cudaStreamWaitEvent(h->st, h->ev_chol, 0));     // leaf Cholesky issued during the build
  ph_begin(h, PH_LEAF);
  bool fast = false;
  if (!h->nonspd) {
    hodlr_status fs = hodlr_leaf_factor_mma(h, K, h->Pipool + dt.piOff[kappa], &fast);   // needs the Cholesky kernel
    if (fs != HODLR_OK) return fs;
  }
  if (h->nonspd) {                 // LU leaves (R20)
    LuCtx lu;
    LeafCtx &lc = lu.b;
    lc.kp = h->kp; lc.n = h->n; lc.ninternal = h->ninternal; lc.nleaves = nl; lc.kappa = kappa; lc.K = K;
    lc.ldz = K | 1; lc.T = h->ltiles; lc.xs = h->xs; lc.lo = h->lo; lc.hi = h->hi; lc.Xh = h->Xh; lc.ldx = h->ldx;
    lc.rank = h->rank; lc.dt = h->d_dt; lc.Lf = h->Lf; lc.lstride = h->lstride; lc.Pi = h->Pipool + dt.piOff[kappa];
    lc.leaf_ld = h->leaf_ld; lc.flags = h->dflags; lc.aug = h->aug; lc.y = h->y_aug; lc.perm = h->perm;
    lc.kps = h->d_kps; lc.nseg = h->nseg; lc.mmax = mmax;
    hodlr_own_nodes(h, kappa, &lc.leaf0, &lc.nown);
    lu.Uf = h->Uf; lu.lperm = h->lperm;
    if (mmax > 256 || K > 1024) return hodlr_set_error(HODLR_EINVAL, "factor: LU leaves need leaf size <= 256, K <= 1024");
    const size_t a_bytes = sizeof(double) * (size_t)mmax * mmax;
    lu.a_smem = a_bytes <= (size_t)maxsm - 16 * 1024 ? 1 : 0;
    const int grid = (int)std::min<long long>(lc.nown, 148 * 2);
    lu.scr_per_cta = (lu.a_smem ? 0 : (long long)mmax * mmax) + 2LL * mmax * lc.ldz;
    lu.scr = (double *)hodlr_dalloc_tmp(h, sizeof(double) * (size_t)lu.scr_per_cta * grid);
    if (!lu.scr) return hodlr_set_error(HODLR_ENOMEM, "factor: scratch allocation failed");
    if (lu.a_smem) HCUDA(hodlr_allow_smem((const void *)k_leaf_factor_lu, h->dev));
    k_leaf_factor_lu<<<grid, LT, lu.a_smem ? a_bytes : 0, h->st>>>(lu);
    HLAUNCH(h, "k_leaf_factor_lu");
    fast = true;
  }
  if (!fast) {
    LeafCtx lc;
    lc.kp = h->kp; lc.n = h->n; lc.ninternal = h->ninternal; lc.nleaves = nl; lc.kappa = kappa; lc.K = K;
    lc.ldz = K | 1; lc.T = h->ltiles; lc.xs = h->xs; lc.lo = h->lo; lc.hi = h->hi; lc.Xh = h->Xh; lc.ldx = h->ldx; lc.rank = h->rank;
    lc.dt = h->d_dt; lc.Lf = h->Lf; lc.lstride = h->lstride; lc.Pi = h->Pipool + dt.piOff[kappa];
    lc.leaf_ld = h->leaf_ld; lc.flags = h->dflags;
    lc.aug = h->aug; lc.y = h->y_aug; lc.perm = h->perm;
    lc.kps = h->d_kps; lc.nseg = h->nseg;
    lc.mmax = mmax;
    hodlr_own_nodes(h, kappa, &lc.leaf0, &lc.nown);
    lc.lsz = (long long)mmax * (mmax + 1) / 2 + 1;
    size_t need = sizeof(double) * (2 * (size_t)mmax + lc.lsz + (size_t)(mmax + 8) * lc.ldz);   // colj, xl, L, Z, Zb
    int grid = (int)lc.nown, nthreads = LT;
    lc.scratch = nullptr; lc.scratch_per_cta = 0;
    if (need <= (size_t)maxsm - 12 * 1024) {
      lc.use_smem = 1;
      HCUDA(hodlr_allow_smem((const void *)k_leaf_factor, h->dev));
    } else {
      lc.use_smem = 0; need = sizeof(double) * (size_t)mmax;     // colj only; xl, L, Z in global scratch
      if (need > (size_t)maxsm - 12 * 1024) return hodlr_set_error(HODLR_EINVAL, "factor: leaf size %d too large", mmax);
      int nsm = 148;
      HCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
      grid = (int)(lc.nown < nsm ? lc.nown : nsm); nthreads = 1024;      // one CTA per SM: the scratch stays in L2
      lc.scratch_per_cta = mmax + lc.lsz + (long long)(mmax + 8) * lc.ldz;
      lc.scratch = (double *)hodlr_dalloc(h, sizeof(double) * lc.scratch_per_cta * grid);
      if (!lc.scratch) return hodlr_set_error(HODLR_ENOMEM, "factor: scratch allocation failed");
    }
    k_leaf_factor<<<grid, nthreads, need, h->st>>>(lc);
    HLAUNCH(h, "k_leaf_factor");
  }
  ph_end(h, PH_LEAF);
  // ---- tree, bottom-up ----
  ph_begin(h, PH_TREE);
  size_t tree_smem_max = 0;
  for (int d = 0; d < kappa; d++) {
    const int q = 2 * dt.rdep[d + 1], ldk = (dt.Kf[d] + 3) & ~3;
    tree_smem_max = std::max(tree_smem_max, sizeof(double) * (size_t)tree_smem_doubles(q, ldk));
  }
  if (tree_smem_max > (size_t)maxsm - 2048)
    return hodlr_set_error(HODLR_EINVAL, "factor: coupling system too large for shared memory");
  // (the device maximum, set on every call: a process-wide "already set" guard is neither per-device nor
  // thread-safe, and concurrent handles needing different sizes would race on a per-call value)
  if (kappa > 0) {
    HCUDA(hodlr_allow_smem((const void *)k_tree_factor<true>, h->dev));
    HCUDA(hodlr_allow_smem((const void *)k_tree_factor<false>, h->dev));
    HCUDA(hodlr_allow_smem((const void *)k_tree_factor_narrow<true>, h->dev));
    HCUDA(hodlr_allow_smem((const void *)k_tree_factor_narrow<false>, h->dev));
  }
  int nsm = 148;
  HCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
  std::vector<TreeCtx> top;           // the current run of upper levels for k_tree_top
  auto flush_top = [&]() -> hodlr_status {
    if (top.empty()) return HODLR_OK;
    size_t smem = 0;
    long long maxcnt = 0;
    for (const TreeCtx &tc : top) {
      smem = std::max(smem, sizeof(double) * (size_t)tree_smem_doubles(tc.q, tc.ldk));
      maxcnt = std::max(maxcnt, tc.cnt);
    }
    if (top.size() > (size_t)TREE_TOP_MAXLEV) return hodlr_set_error(HODLR_EINVAL, "factor: tree level table overflow");
    for (size_t L = 0; L < top.size(); L++) { top[L].ready = h->d_ready; top[L].wait = L > 0 ? 1 : 0; }
    HCUDA(cudaMemsetAsync(h->d_ready, 0, sizeof(int) * (size_t)(h->ninternal + 2), h->st));
    HCUDA(cudaMemcpyAsync(h->d_treectx, top.data(), sizeof(TreeCtx) * top.size(), cudaMemcpyHostToDevice, h->st));
    HCUDA(hodlr_allow_smem((const void *)k_tree_top<true>, h->dev));
    int per_sm = 0;
    HCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tree_top<true>, TT, smem));
    if (per_sm < 1) return hodlr_set_error(HODLR_EINVAL, "factor: coupling system too large for one SM");
    long long gmax = (long long)nsm * per_sm;
    if (h->coop_ctas > 0) gmax = std::min<long long>(gmax, h->coop_ctas);
    const int grid = (int)std::min<long long>(maxcnt, gmax);
    const TreeCtx *pc = h->d_treectx;
    int nlev = (int)top.size();
    void *args[] = {(void *)&pc, (void *)&nlev};
    HCUDA(cudaLaunchCooperativeKernel((const void *)k_tree_top<true>, dim3(grid), dim3(TT), args, smem, h->st));
    HLAUNCH(h, "k_tree_top");
    top.clear();
    return HODLR_OK;
  };
  std::vector<TreeCtx> deep;          // the current run of deep levels for k_tree_deep
  auto flush_deep = [&]() -> hodlr_status {
    if (deep.empty()) return HODLR_OK;
    if (deep.size() > (size_t)TREE_TOP_MAXLEV) return hodlr_set_error(HODLR_EINVAL, "factor: tree level table overflow");
    size_t smem = 0;
    long long tot = 0;
    bool anydd = false;
    for (size_t L = 0; L < deep.size(); L++) {
      deep[L].ready = h->d_ready; deep[L].wait = L > 0 ? 1 : 0;
      smem = std::max(smem, sizeof(double) * (size_t)tree_smem_doubles(deep[L].q, deep[L].ldk));
      tot += deep[L].cnt;
      anydd = anydd || deep[L].dd;
    }
    const bool small = smem <= TREE_DEEP64_SMEM;
    const int ntd = small ? 64 : TT / 2;
    const void *kf = small ? (anydd ? (const void *)k_tree_deep<true, 64> : (const void *)k_tree_deep<false, 64>)
                           : (anydd ? (const void *)k_tree_deep<true, TT / 2> : (const void *)k_tree_deep<false, TT / 2>);
    HCUDA(cudaMemsetAsync(h->d_ready, 0, sizeof(int) * (size_t)(h->ninternal + 2), h->st));
    HCUDA(cudaMemcpyAsync(h->d_treectx, deep.data(), sizeof(TreeCtx) * deep.size(), cudaMemcpyHostToDevice, h->st));
    HCUDA(hodlr_allow_smem(kf, h->dev));
    int per_sm = 0;
    HCUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, ntd, smem));
    if (per_sm < 1) return hodlr_set_error(HODLR_EINVAL, "factor: coupling system too large for one SM");
    long long gmax = (long long)nsm * per_sm;
    if (h->coop_ctas > 0) gmax = std::min<long long>(gmax, h->coop_ctas);
    const int grid = (int)std::min<long long>(tot, gmax);
    const TreeCtx *pc = h->d_treectx;
    int nlev = (int)deep.size();
    unsigned *nx = (unsigned *)(h->d_ready + h->ninternal);
    void *args[] = {(void *)&pc, (void *)&nlev, (void *)&nx};
    HCUDA(cudaLaunchCooperativeKernel(kf, dim3(grid), dim3(ntd), args, smem, h->st));
    HLAUNCH(h, "k_tree_deep");
    deep.clear();
    return HODLR_OK;
  };
  for (int d = kappa - 1; d >= 0; d--) {
    if (d + 1 == h->tsplit && h->nranks > 1) {     // every rank gets the Pi of all depth-t subtree roots
      hodlr_status fs = flush_deep();
      if (fs != HODLR_OK) return fs;
      fs = flush_top();
      if (fs != HODLR_OK) return fs;
      const long long Kt = dt.Kf[d + 1], sz = Kt * (Kt + 1) / 2;
      double *base = h->Pipool + dt.piOff[d + 1];
      hodlr_status xs = hodlr_allgather(h, base + h->grank * sz, base, sizeof(double) * sz);
      if (xs != HODLR_OK) return xs;
    }
    long long i0, cnt;
    hodlr_own_nodes(h, d, &i0, &cnt);
    TreeCtx tc = tree_ctx(h, d, i0);
    tc.cnt = cnt;
    if (cnt < TREE_NARROW_MIN) {                  // upper levels: batched into k_tree_top
      hodlr_status fs = flush_deep();
      if (fs != HODLR_OK) return fs;
      top.push_back(tc);
      continue;
    }
    const size_t smem = sizeof(double) * (size_t)tree_smem_doubles(tc.q, tc.ldk);
    const bool narrow = tc.q <= 16;
    if (narrow && smem <= TREE_DEEP_SMEM) {      // deep run (k_tree_deep): levels of one Pi precision per launch
      if (!deep.empty() && deep.back().dd != tc.dd) {
        hodlr_status fs = flush_deep();
        if (fs != HODLR_OK) return fs;
      }
      deep.push_back(tc);
      continue;
    }
    {
      hodlr_status fs = flush_deep();
      if (fs != HODLR_OK) return fs;
    }
    if (narrow) {
      if (tc.dd) k_tree_factor_narrow<true><<<(int)cnt, TT / 2, smem, h->st>>>(tc);
      else k_tree_factor_narrow<false><<<(int)cnt, TT / 2, smem, h->st>>>(tc);
    } else {
      if (tc.dd) k_tree_factor<true><<<(int)cnt, TT, smem, h->st>>>(tc);
      else k_tree_factor<false><<<(int)cnt, TT, smem, h->st>>>(tc);
    }
    HLAUNCH(h, "k_tree_factor");
  }
  {
    hodlr_status fs = flush_deep();
    if (fs != HODLR_OK) return fs;
    fs = flush_top();
    if (fs != HODLR_OK) return fs;
  }
  // log det: this rank's leaves and subtree nodes (others are 0), exchanged with the failure counts, then the
  // top-level nodes (computed redundantly by every rank) once
  k_logdet_reduce<<<1, LDR_T, 0, h->st>>>(h->leaf_ld, h->node_ld, nl, kappa, h->tsplit, h->dflags, ldx + 2 * h->nranks);
  HLAUNCH(h, "k_logdet_reduce");
  {
    hodlr_status xs = hodlr_allgather(h, ldx + 2 * h->nranks, ldx, sizeof(double) * 2);
    if (xs != HODLR_OK) return xs;
  }
  k_logdet_final<<<1, 32, 0, h->st>>>(ldx, h->nranks, h->node_ld, h->tsplit, h->dflags, h->d_logdet);
  HLAUNCH(h, "k_logdet_final");
  ph_end(h, PH_TREE);
  return HODLR_OK;
}
