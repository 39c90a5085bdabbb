// leaf_mma.cu -- G4/G5 fast path: per-leaf Cholesky, panel solve and projected Gram on the FP64
// tensor pipe (mma.sync f64, "DMMA"), one CTA per leaf, everything resident on chip.  Two kernels:
// k_leaf_chol (no dependence on the ACA: runs on a side stream during the build) and k_leaf_zsyrk
// (Z and Pi after the ACA).
//
// For a leaf l with rows [lo, lo+m), m <= P (P = 64 or 128), and its ancestor-factor panel
// E_l = Xh[l rows, K columns] (Fig. 6 lines 7-12):
//   A_l = K[l,l] + s2 I = L L^T   left-looking over 8-column tiles: C(I,J) = A(I,J) - sum_k L(I,k) L(J,k)^T
//                                  accumulated in registers (DMMA m8n8k4), 8x8 POTRF + triangular inverse
//                                  of the diagonal tile by one warp, panel L(I,J) = C(I,J) Linv(J)^T
//   Z   = L^{-1} E_l              each warp owns <= 2 8-column tiles of Z and sweeps them down the 16 row
//                                  blocks entirely in registers (Z_b <- Linv(b) Z_b; Z_i -= L(i,b) Z_b),
//                                  no block-level synchronisation
//   Pi_l = Z^T Z                  SYRK with DMMA m16n8k8, 16x16 register blocks
// Layout: L tiles in "fragment order" (element (r, c) of an 8x8 tile at (c>>2)*32 + r*4 + (c&3), so an
// A/B fragment half is 32 contiguous doubles); Z column-major with leading dimension P + 4 (conflict-free
// fragment loads).  Rows m..P-1 are padded with the identity (A) and zeros (E).
#include "hodlr_internal.cuh"
#include "tree_node.cuh"
#include <stdio.h>
#include <algorithm>
#include <stdlib.h>

namespace {


__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma16(double *c, double a0, double a1, double a2, double a3, double b0, double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}
// offset of this lane's C/D pair (row lane>>2, cols 2(lane&3), +1) inside a fragment-order tile
__device__ __forceinline__ int cpos(int lane) { int q = lane & 3; return (q >> 1) * 32 + (lane >> 2) * 4 + 2 * (q & 1); }

// From an 8x8 tile held in C layout (c0, c1 at row lane>>2, cols 2(lane&3)+{0,1}) produce the two B-operand
// halves (row (lane&3) + 4h, col lane>>2).
__device__ __forceinline__ void c_to_b(double c0, double c1, int lane, double &b0, double &b1) {
  const int col = lane >> 2, sel = col & 1;
  const int s0 = 4 * (lane & 3) + (col >> 1), s1 = s0 + 16;
  const double x0 = __shfl_sync(0xffffffffu, c0, s0), x1 = __shfl_sync(0xffffffffu, c1, s0);
  const double y0 = __shfl_sync(0xffffffffu, c0, s1), y1 = __shfl_sync(0xffffffffu, c1, s1);
  b0 = sel ? x1 : x0;
  b1 = sel ? y1 : y0;
}

// (I, J) of packed lower tile index ti, for T <= 16 (136 tiles); statically initialised (per device at module
// load, so no host-side "tables ready" state)
__constant__ unsigned char c_tileI[136] = {0,1,1,2,2,2,3,3,3,3,4,4,4,4,4,5,5,5,5,5,5,6,6,6,6,6,6,6,7,7,7,7,7,7,7,7,8,8,8,8,8,8,8,8,8,9,9,9,9,9,9,9,9,9,9,10,10,10,10,10,10,10,10,10,10,10,11,11,11,11,11,11,11,11,11,11,11,11,12,12,12,12,12,12,12,12,12,12,12,12,12,13,13,13,13,13,13,13,13,13,13,13,13,13,13,14,14,14,14,14,14,14,14,14,14,14,14,14,14,14,15,15,15,15,15,15,15,15,15,15,15,15,15,15,15,15};
__constant__ unsigned char c_tileJ[136] = {0,0,1,0,1,2,0,1,2,3,0,1,2,3,4,0,1,2,3,4,5,0,1,2,3,4,5,6,0,1,2,3,4,5,6,7,0,1,2,3,4,5,6,7,8,0,1,2,3,4,5,6,7,8,9,0,1,2,3,4,5,6,7,8,9,10,0,1,2,3,4,5,6,7,8,9,10,11,0,1,2,3,4,5,6,7,8,9,10,11,12,0,1,2,3,4,5,6,7,8,9,10,11,12,13,0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,0,1,2,3,4,5,6,7,8,9,10,11,12,13,14,15};

struct LeafMmaCtx {
  KParams kp;
  long long n, ninternal;
  int kappa, K, Kp, Kz;
  const double *xs;
  const long long *lo, *hi;
  const double *Xh; long long ldx;
  const int *rank;
  const DepthTab *dt;
  double *Lf; long long lstride;
  double *Pi;
  double *leaf_ld;
  int *flags;
  long long leaf0;          // first leaf of this launch (this rank's subtree)
  int aug;                  // fused right-hand side (hodlr_factor_solve): panel column 0 is y[perm[rows]]
  const double *y; const long long *perm;
  const KParams *kps; long long nseg;     // batched handle (kp_of), or NULL
};

// Panel entry of the fused right-hand side: y of sorted row lo + row (0 beyond the leaf); flags non-finite y.
__device__ __forceinline__ double rhs_val(const LeafMmaCtx &c, long long lo, int row, int m) {
  if (row >= m) return 0.0;
  const double v = c.y[c.perm[lo + row]];
  if (!isfinite(v)) atomicOr(&c.flags[3], 1);
  return v;
}

// One warp, every lane computes the same 8x8 POTRF redundantly (no shuffles on the critical path),
// then writes its fragment positions of L and of L^{-1}.
__device__ void potrf8(double *tile, double *linv, double *diag8, int *bad) {
  const int lane = threadIdx.x & 31;
  double a[8][8];
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j <= i; j++) a[i][j] = tile[fo(i, j)];
  double inv[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    double d = a[j][j];
    if (!(d > 0.0)) { if (lane == 0) *bad = 1; d = 1.0; }
    // 1/sqrt(d): hardware approximation (rsqrt.approx.f64) + 2 Newton steps (no slow-path call)
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = r * fma(-0.5 * d * r, r, 1.5);
    r = r * fma(-0.5 * d * r, r, 1.5);
    inv[j] = r;
    a[j][j] = d * r;
#pragma unroll
    for (int i = j + 1; i < 8; i++) a[i][j] *= r;
#pragma unroll
    for (int k = j + 1; k < 8; k++)
#pragma unroll
      for (int i = k; i < 8; i++) a[i][k] -= a[i][j] * a[k][j];
  }
  // every lane holds the same factor: all lanes store every element (same address, same value)
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) tile[fo(i, j)] = j <= i ? a[i][j] : 0.0;
  if (lane < 8) diag8[lane] = tile[fo(lane, lane)];
  // L^{-1}: lane cc < 8 computes column cc by forward substitution (the 8 columns in parallel)
  if (lane < 8) {
    const int cc = lane;
    double y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      double s = (i == cc) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; k++) s = fma(-a[i][k], y[k], s);
      y[i] = i < cc ? 0.0 : s * inv[i];
    }
#pragma unroll
    for (int i = 0; i < 8; i++) linv[fo(i, cc)] = y[i];
  }
  __syncwarp();
}

// Column map of leaf `id`: local column q (depth e block, Kdim[e-1] <= q < Kdim[e]) -> global Xh column, or -1
// beyond the rank of that ancestor's block.  One thread per column (no serial walk).
// With a fused right-hand side, column 0 is that vector (-2) and the ancestor columns follow.
__device__ __forceinline__ long long leaf_colsrc(const LeafMmaCtx &c, long long id, int q) {
  if (q >= c.K) return -1;
  if (q < c.aug) return -2;
  q -= c.aug;
  int e = 1;
  while (c.dt->Kdim[e] <= q) e++;
  const int qq = q - c.dt->Kdim[e - 1];
  const long long b = ((id + 1) >> (c.kappa - e + 1)) - 1;     // ancestor at depth e - 1 (heap order)
  return qq < c.rank[b] ? c.dt->colbase[e] + qq : -1;
}

// ---------------------------------------------------------------------------------------------
// Kernel 1 (does not depend on the ACA; launched on a side stream during the build):
//   A_l = K[l,l] + s2 I = L L^T, left-looking over 8-column tiles, 2 CTAs per SM; then X = L^{-1}
//   (column sweeps on the FP64 tensor pipe); writes the tiles of X and the log det partial 2 sum log L_ii.
//   Only X is kept: Z = X E is a GEMM and the solve's triangular solves become matrix-vector products
//   (explicit triangular inverse: DESIGN.md R6).
// ---------------------------------------------------------------------------------------------
#ifndef CHOL_LOOKAHEAD
#define CHOL_LOOKAHEAD 1
#endif
#ifdef CHOL_TRACE
__device__ unsigned long long g_chol_stamps[2][6];
#define CSTAMP(k) if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 4000)) { unsigned long long v_; \
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v_)); g_chol_stamps[blockIdx.x ? 1 : 0][k] = v_; }
#else
#define CSTAMP(k)
#endif
// CTA size: 8 warps for 128-point leaves (2 CTAs per SM); 2 warps for 64-point leaves, 8 CTAs per SM -- a 64-point
// leaf's chain of 8 diagonal steps is latency, so more leaves in flight (the batched config-4 factorization:
// 131072 such leaves).
#ifndef CHOL64_NT
#define CHOL64_NT 64
#endif
#ifndef CHOL64_MINB
#define CHOL64_MINB (512 / CHOL64_NT)
#endif
template <int P> struct CholCfg {
  static constexpr int NT = P == 64 ? CHOL64_NT : 256, MINB = P == 64 ? CHOL64_MINB : 2;
};
template <int P, int SEO>
__global__ void __launch_bounds__(CholCfg<P>::NT, CholCfg<P>::MINB) k_leaf_chol(LeafMmaCtx c) {
  constexpr int NTH = CholCfg<P>::NT, NW = NTH / 32;
  constexpr int T = P / 8;
  constexpr int NTILE = T * (T + 1) / 2;
  extern __shared__ double sm[];
  __shared__ int bad;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double *sL = sm;                              // NTILE * 64
  double *sLi = sL + NTILE * 64;                // T * 64
  double *sx = sLi + T * 64;                    // P
  double *sdiag = sx + P;                       // P
  const long long leaf = c.leaf0 + blockIdx.x;
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const KParams kp = kp_of(c.kp, c.kps, c.nseg, lo);
  const int m = (int)(c.hi[id] - lo);
  CSTAMP(0)
  if (t == 0) bad = 0;
  for (int i = t; i < P; i += NTH) sx[i] = i < m ? c.xs[lo + i] : 0.0;
  __syncthreads();
  // assemble A_l = K[l,l] + s2 I into the lower tiles (fragment order), identity padding beyond m.  With the
  // look-ahead schedule only tile columns 0 and 1 are assembled up front; column J+2 is assembled by warps 1-7
  // during step J (while warp 0 factors the diagonal tile), hiding the kernel evaluations behind the POTRFs.
  auto asm_tile = [&](int I, int J) {
    const int ti = tix(I, J);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int r = lane >> 2, cc = (lane & 3) + 4 * h;
      const int i = 8 * I + r, j = 8 * J + cc;
      double v;
      if (i < m && j < m) {
        v = SEO == KV_ND ? kval_nd_fast(kp, c.xs, lo + i, lo + j) : kval_t<SEO>(kp, sx[i] - sx[j]);
        if (i == j) v += sig2(kp, lo + i);
      }
      else v = (i == j) ? 1.0 : 0.0;
      sL[ti * 64 + 32 * h + lane] = v;
    }
  };
#if CHOL_LOOKAHEAD
  for (int ti = warp; ti < 2 * T - 1; ti += NW) asm_tile(ti < T ? ti : ti - T + 1, ti < T ? 0 : 1);   // columns 0, 1
#else
  for (int ti = warp; ti < NTILE; ti += NW) asm_tile(c_tileI[ti], c_tileJ[ti]);
#endif
  __syncthreads();
  CSTAMP(1)
  // ---------------- Cholesky, left-looking over tile columns J ----------------
  // Per column: warp 0 forms the diagonal tile C(J,J) and factors it (POTRF + inverse) while warps 1-7
  // form the sub-diagonal tiles C(I,J) = A(I,J) - sum_{k<J} L(I,k) L(J,k)^T; then all warps apply
  // Linv(J)^T to the panel.
  const int cp = cpos(lane);
#if CHOL_LOOKAHEAD
  // Look-ahead schedule (one block barrier per column): in step J every warp applies Linv(J) to its panel tiles
  // L(I,J) = C(I,J) Linv(J)^T (warp 0 takes I = J+1 first), then warp 0 -- without waiting for the others --
  // forms the next diagonal tile C(J+1,J+1) = A - sum_{k<=J} L(J+1,k) L(J+1,k)^T and factors it (POTRF +
  // inverse), while warps 1-7, after a named barrier that warp 0 only arrives at, form the sub-diagonal tiles
  // C(I,J+1), I > J+1.  The factorization is the same left-looking one; only the order of independent work changes.
  auto diag_update = [&](int J) {              // warp 0: C(J,J) -= sum_{k<J} L(J,k) L(J,k)^T, then POTRF
    const double *tJ = sL + tix(J, 0) * 64;
    double *tc = sL + tix(J, J) * 64;
    double d0 = tc[cp], d1 = tc[cp + 1], e0 = 0.0, e1 = 0.0;
    int k = 0;
    for (; k + 1 < J; k += 2) {
      dmma(d0, d1, -tJ[k * 64 + lane], tJ[k * 64 + lane]);
      dmma(e0, e1, -tJ[(k + 1) * 64 + lane], tJ[(k + 1) * 64 + lane]);
      dmma(d0, d1, -tJ[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
      dmma(e0, e1, -tJ[(k + 1) * 64 + 32 + lane], tJ[(k + 1) * 64 + 32 + lane]);
    }
    if (k < J) {
      dmma(d0, d1, -tJ[k * 64 + lane], tJ[k * 64 + lane]);
      dmma(e0, e1, -tJ[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
    }
    __syncwarp();
    tc[cp] = d0 + e0; tc[cp + 1] = d1 + e1;
    __syncwarp();
    potrf8(tc, sLi + J * 64, sdiag + 8 * J, &bad);
  };
  auto offdiag_update = [&](int I, int J) {    // C(I,J) -= sum_{k<J} L(I,k) L(J,k)^T
    const double *tJ = sL + tix(J, 0) * 64;
    double *tc = sL + tix(I, J) * 64;
    double d0 = tc[cp], d1 = tc[cp + 1], e0 = 0.0, e1 = 0.0;
    const double *tI = sL + tix(I, 0) * 64;
    int k = 0;
    for (; k + 1 < J; k += 2) {
      dmma(d0, d1, -tI[k * 64 + lane], tJ[k * 64 + lane]);
      dmma(e0, e1, -tI[(k + 1) * 64 + lane], tJ[(k + 1) * 64 + lane]);
      dmma(d0, d1, -tI[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
      dmma(e0, e1, -tI[(k + 1) * 64 + 32 + lane], tJ[(k + 1) * 64 + 32 + lane]);
    }
    if (k < J) {
      dmma(d0, d1, -tI[k * 64 + lane], tJ[k * 64 + lane]);
      dmma(e0, e1, -tI[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
    }
    __syncwarp();
    tc[cp] = d0 + e0; tc[cp + 1] = d1 + e1;
  };
  auto panel = [&](int I, int J) {             // L(I,J) = C(I,J) Linv(J)^T
    const double *Li = sLi + J * 64;
    double *tl = sL + tix(I, J) * 64;
    const double a0 = tl[lane], a1 = tl[32 + lane];
    double d0 = 0.0, d1 = 0.0;
    dmma(d0, d1, a0, Li[lane]);
    dmma(d0, d1, a1, Li[32 + lane]);
    __syncwarp();
    tl[cp] = d0; tl[cp + 1] = d1;
  };
  if (warp == 0) diag_update(0);               // column 0: nothing to subtract
  __syncthreads();
  for (int J = 0; J < T; J++) {
    if (J + 1 >= T) break;                     // the last column has no panel
    if (warp == 0) {
      panel(J + 1, J);
      __syncwarp();
      __threadfence_block();
      asm volatile("bar.arrive 1, %0;" :: "n"(NTH) : "memory");    // L(J+1, J) is in shared memory
      diag_update(J + 1);
    } else {
      for (int I = J + 1 + warp; I < T; I += NW - 1) panel(I, J);
      asm volatile("bar.sync 1, %0;" :: "n"(NTH) : "memory");
      for (int I = J + 1 + warp; I < T; I += NW - 1) offdiag_update(I, J + 1);
      for (int I = J + 1 + warp; I < T; I += NW - 1) asm_tile(I, J + 2);     // column J+2 (I >= J+2)
    }
    __syncthreads();
  }
#else
  for (int J = 0; J < T; J++) {
    const double *tJ = sL + tix(J, 0) * 64;
    if (warp == 0) {
      double *tc = sL + tix(J, J) * 64;
      double d0 = tc[cp], d1 = tc[cp + 1], e0 = 0.0, e1 = 0.0;
      int k = 0;
      for (; k + 1 < J; k += 2) {
        dmma(d0, d1, -tJ[k * 64 + lane], tJ[k * 64 + lane]);
        dmma(e0, e1, -tJ[(k + 1) * 64 + lane], tJ[(k + 1) * 64 + lane]);
        dmma(d0, d1, -tJ[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
        dmma(e0, e1, -tJ[(k + 1) * 64 + 32 + lane], tJ[(k + 1) * 64 + 32 + lane]);
      }
      if (k < J) {
        dmma(d0, d1, -tJ[k * 64 + lane], tJ[k * 64 + lane]);
        dmma(e0, e1, -tJ[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
      }
      __syncwarp();
      tc[cp] = d0 + e0; tc[cp + 1] = d1 + e1;
      __syncwarp();
      potrf8(tc, sLi + J * 64, sdiag + 8 * J, &bad);
    } else {
      for (int I = J + warp; I < T; I += NW - 1) {
        double *tc = sL + tix(I, J) * 64;
        double d0 = tc[cp], d1 = tc[cp + 1], e0 = 0.0, e1 = 0.0;
        const double *tI = sL + tix(I, 0) * 64;
        int k = 0;
        for (; k + 1 < J; k += 2) {
          dmma(d0, d1, -tI[k * 64 + lane], tJ[k * 64 + lane]);
          dmma(e0, e1, -tI[(k + 1) * 64 + lane], tJ[(k + 1) * 64 + lane]);
          dmma(d0, d1, -tI[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
          dmma(e0, e1, -tI[(k + 1) * 64 + 32 + lane], tJ[(k + 1) * 64 + 32 + lane]);
        }
        if (k < J) {
          dmma(d0, d1, -tI[k * 64 + lane], tJ[k * 64 + lane]);
          dmma(e0, e1, -tI[k * 64 + 32 + lane], tJ[k * 64 + 32 + lane]);
        }
        tc[cp] = d0 + e0; tc[cp + 1] = d1 + e1;
      }
    }
    __syncthreads();
    // panel: L(I,J) = C(I,J) Linv(J)^T for I > J
    const double *Li = sLi + J * 64;
    for (int I = J + 1 + warp; I < T; I += NW) {
      double *tl = sL + tix(I, J) * 64;
      const double a0 = tl[lane], a1 = tl[32 + lane];
      double d0 = 0.0, d1 = 0.0;
      dmma(d0, d1, a0, Li[lane]);
      dmma(d0, d1, a1, Li[32 + lane]);
      __syncwarp();
      tl[cp] = d0; tl[cp + 1] = d1;
    }
    __syncthreads();
  }
#endif
  CSTAMP(2)
  if (warp == 0) {          // 2 sum log L_ii: per-lane partials, then a fixed-order warp reduction
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += log(sdiag[i]);
    s2 = warp_sum(s2);
    if (lane == 0) {
      c.leaf_ld[leaf] = 2.0 * s2;
      if (bad) { atomicAdd(&c.flags[1], 1); atomicMin(&c.flags[2], (int)id); }
    }
  }
  // ---- X = L^{-1} (lower, fragment-order tiles) written straight to global: column sweep with E = I,
  // tile column J by one warp (pairs J = warp, T-1-warp balance the work), L read from shared memory ----
  double *Xg = c.Lf + leaf * c.lstride;
  {
    const int g = lane >> 2, q2 = 2 * (lane & 3);
    const int cp = cpos(lane);
    for (int pass = 0;; pass++) {
      // 2 NW >= T: columns J = warp, then T-1-warp (balanced: column J costs T - J tiles); else J = warp + pass NW
      int J;
      if (2 * NW >= T) {
        if (pass >= 2) break;
        J = pass ? T - 1 - warp : warp;
        if (J >= T || (pass && J < NW)) break;
      } else {
        J = warp + pass * NW;
        if (J >= T) break;
      }
      double z[T][2];
#pragma unroll
      for (int i = 0; i < T; i++) {
        z[i][0] = (i == J && g == q2) ? 1.0 : 0.0;
        z[i][1] = (i == J && g == q2 + 1) ? 1.0 : 0.0;
      }
#pragma unroll
      for (int b = 0; b < T; b++) {
        if (b < J) continue;
        const double *Li = sLi + b * 64;
        double b0, b1;
        c_to_b(z[b][0], z[b][1], lane, b0, b1);
        double d0 = 0.0, d1 = 0.0;
        dmma(d0, d1, Li[lane], b0);
        dmma(d0, d1, Li[32 + lane], b1);
        z[b][0] = d0; z[b][1] = d1;
        c_to_b(d0, d1, lane, b0, b1);
#pragma unroll
        for (int i = b + 1; i < T; i++) {
          const double *tA = sL + tix(i, b) * 64;
          dmma(z[i][0], z[i][1], -tA[lane], b0);
          dmma(z[i][0], z[i][1], -tA[32 + lane], b1);
        }
      }
#pragma unroll
      for (int i = 0; i < T; i++) {
        if (i < J) continue;
        double2 v; v.x = z[i][0]; v.y = z[i][1];
        *(double2 *)(Xg + tix(i, J) * 64 + cp) = v;
      }
    }
  }
  __syncthreads();
  CSTAMP(3)
}

// ---------------------------------------------------------------------------------------------
// Kernel 2 (after the ACA): Z = X E_l (X = L^{-1}) and Pi_l = Z^T Z.  16 warps; X tiles and E staged with
// 16-byte cp.async; every warp computes 8-column tiles of Z as a GEMM on the FP64 tensor pipe.
// ---------------------------------------------------------------------------------------------
constexpr int ZTH = 512;
constexpr int ZW = ZTH / 32;

// XG (wide panels, K up to ~208): X tiles are read straight from global memory (L2) as DMMA operands and
// only Z lives in shared memory.
template <int P, bool XG = false>
__global__ void __launch_bounds__(ZTH, 1) k_leaf_zsyrk(LeafMmaCtx c) {
  constexpr int T = P / 8;
  constexpr int NTILE = T * (T + 1) / 2;
  constexpr int LDR = P + 4;
  extern __shared__ double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int K = c.K, Kp = c.Kp, Kc = Kp / 8, Kz = c.Kz;
  const long long leaf = c.leaf0 + blockIdx.x;
  const double *sX = XG ? c.Lf + leaf * c.lstride : sm;   // NTILE * 64: tiles of X = L^{-1}
  double *sZ = XG ? sm : sm + NTILE * 64;       // Kz * LDR (column-major)
  long long *colsrc = (long long *)(sZ + (long long)Kz * LDR);   // Kz
  const long long id = c.ninternal + leaf, lo = c.lo[id];
  const int m = (int)(c.hi[id] - lo);
  if (!XG) {
    const double *Lg = c.Lf + leaf * c.lstride;
    for (int p = t; p < NTILE * 32; p += ZTH) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(sm + 2 * p);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(Lg + 2 * p));
    }
  }
  for (int q = t; q < Kz; q += ZTH) colsrc[q] = leaf_colsrc(c, id, q);
  __syncthreads();
  const bool al16 = ((c.ldx | lo) & 1) == 0;      // 16-byte aligned column segments (row pairs)
  if (al16) {
    for (int p = t; p < Kz * (P / 2); p += ZTH) {
      const int col = p / (P / 2), row = 2 * (p - col * (P / 2));
      const long long src = colsrc[col];
      double *dst = sZ + col * LDR + row;
      if (src >= 0 && row + 1 < m) {
        unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(c.Xh + src * c.ldx + lo + row));
      } else if (src == -2) {
        dst[0] = rhs_val(c, lo, row, m); dst[1] = rhs_val(c, lo, row + 1, m);
      } else {
        dst[0] = (src >= 0 && row < m) ? c.Xh[src * c.ldx + lo + row] : 0.0;
        dst[1] = 0.0;
      }
    }
  } else {
    for (int p = t; p < Kz * P; p += ZTH) {
      const int col = p / P, row = p - col * P;
      const long long src = colsrc[col];
      double *dst = sZ + col * LDR + row;
      *dst = src == -2 ? rhs_val(c, lo, row, m) : ((src >= 0 && row < m) ? c.Xh[src * c.ldx + lo + row] : 0.0);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // ---------------- Z = X E (X = L^{-1}): GEMM, one 8-column tile of Z per warp, all row blocks as
  // independent register accumulators (no sequential dependence) ----------------
  {
    const int g = lane >> 2, q2 = 2 * (lane & 3), kq = lane & 3;
    for (int cc = warp; cc < Kc; cc += ZW) {
      double acc[T][2];
#pragma unroll
      for (int i = 0; i < T; i++) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
      const double *zc = sZ + (8 * cc + g) * LDR;        // B operand: E(8 kb + kq (+4), 8 cc + g)
#pragma unroll
      for (int kb = 0; kb < T; kb++) {
        const double b0 = zc[8 * kb + kq], b1 = zc[8 * kb + 4 + kq];
#pragma unroll
        for (int i = kb; i < T; i++) {
          const double *tA = sX + tix(i, kb) * 64;
          dmma(acc[i][0], acc[i][1], tA[lane], b0);
          dmma(acc[i][0], acc[i][1], tA[32 + lane], b1);
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < T; i++) {
        sZ[(8 * cc + q2) * LDR + 8 * i + g] = acc[i][0];
        sZ[(8 * cc + q2 + 1) * LDR + 8 * i + g] = acc[i][1];
      }
    }
  }
  __syncthreads();
  if (K == 0) return;
  // ---------------- Pi_l = Z^T Z: 16x16 output blocks, DMMA m16n8k8 ----------------
  const int Kc16 = Kz / 16;
  const int nblk = Kc16 * (Kc16 + 1) / 2;
  double *Pl = c.Pi + leaf * ((long long)K * (K + 1) / 2);
  const int kend = (m + 7) & ~7;
  const int g = lane >> 2, tq = lane & 3;
  for (int blk = warp; blk < nblk; blk += ZW) {
    const int BI = c_tileI[blk], BJ = c_tileJ[blk];
    double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
    const double *pa0 = sZ + (16 * BI + g) * LDR + tq;
    const double *pa1 = pa0 + 8 * LDR;
    const double *pb0 = sZ + (16 * BJ + g) * LDR + tq;
    const double *pb1 = pb0 + 8 * LDR;
    for (int k0 = 0; k0 < kend; k0 += 8) {
      const double a0 = pa0[k0], a1 = pa1[k0], a2 = pa0[k0 + 4], a3 = pa1[k0 + 4];
      dmma16(acc0, a0, a1, a2, a3, pb0[k0], pb0[k0 + 4]);
      dmma16(acc1, a0, a1, a2, a3, pb1[k0], pb1[k0 + 4]);
    }
    // acc0: rows 16BI + g (+8), cols 16BJ + 2tq (+1); acc1: same rows, cols + 8
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const double v = q < 4 ? acc0[q] : acc1[q - 4];
      const int row = 16 * BI + g + ((q & 2) ? 8 : 0);
      const int col = 16 * BJ + 2 * tq + (q & 1) + (q >= 4 ? 8 : 0);
      if (row < K && col < K && row >= col) Pl[(long long)row * (row + 1) / 2 + col] = v;
    }
  }
}

// Persistent form of k_leaf_zsyrk (X staged): one CTA per SM walks the leaves leaf0 + blockIdx.x + k gridDim.x;
// the next leaf's X tiles are copied (cp.async) while this leaf's Pi = Z^T Z runs, and its panel E as soon as Z is
// free, so only the E copy is exposed per leaf (no CTA turnaround either).
// NT threads: 512 (16 warps, one CTA per SM) in general; 256 (8 warps, 4 CTAs per SM) for 64-point leaves with at
// most 64 panel columns -- there a leaf has too few Z tiles for 16 warps and the per-leaf barriers dominate, so
// four leaves per SM are in flight instead of one (the batched config-4 factorization: 131072 such leaves).
template <int P, int NT>
__global__ void __launch_bounds__(NT, NT == 512 ? 1 : 4) k_leaf_zsyrk_p(LeafMmaCtx c, long long nown) {
  constexpr int ZTH = NT, ZW = NT / 32;
  constexpr int T = P / 8;
  constexpr int NTILE = T * (T + 1) / 2;
  constexpr int LDR = P + 4;
  extern __shared__ double sm[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int K = c.K, Kp = c.Kp, Kc = Kp / 8, Kz = c.Kz;
  double *sX = sm;                              // NTILE * 64: tiles of X = L^{-1}
  double *sZ = sm + NTILE * 64;                 // Kz * LDR (column-major)
  long long *colsrc = (long long *)(sZ + (long long)Kz * LDR);   // Kz
  auto issue_x = [&](long long lf) {
    const double *Lg = c.Lf + lf * c.lstride;
    for (int p = t; p < NTILE * 32; p += ZTH) {
      unsigned sa = (unsigned)__cvta_generic_to_shared(sX + 2 * p);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(Lg + 2 * p));
    }
  };
  auto issue_e = [&](long long lf) {            // colsrc of lf must be in shared memory (after a barrier)
    const long long id = c.ninternal + lf, lo = c.lo[id];
    const int m = (int)(c.hi[id] - lo);
    const bool al16 = ((c.ldx | lo) & 1) == 0;
    if (al16) {
      for (int p = t; p < Kz * (P / 2); p += ZTH) {
        const int col = p / (P / 2), row = 2 * (p - col * (P / 2));
        const long long src = colsrc[col];
        double *dst = sZ + col * LDR + row;
        if (src >= 0 && row + 1 < m) {
          unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(sa), "l"(c.Xh + src * c.ldx + lo + row));
        } else if (src == -2) {
          dst[0] = rhs_val(c, lo, row, m); dst[1] = rhs_val(c, lo, row + 1, m);
        } else {
          dst[0] = (src >= 0 && row < m) ? c.Xh[src * c.ldx + lo + row] : 0.0;
          dst[1] = 0.0;
        }
      }
    } else {
      for (int p = t; p < Kz * P; p += ZTH) {
        const int col = p / P, row = p - col * P;
        const long long src = colsrc[col];
        double *dst = sZ + col * LDR + row;
        *dst = src == -2 ? rhs_val(c, lo, row, m) : ((src >= 0 && row < m) ? c.Xh[src * c.ldx + lo + row] : 0.0);
      }
    }
  };
  long long leaf = c.leaf0 + blockIdx.x;
  const long long end = c.leaf0 + nown;
  if (leaf >= end) return;
  for (int q = t; q < Kz; q += ZTH) colsrc[q] = leaf_colsrc(c, c.ninternal + leaf, q);
  issue_x(leaf);
  __syncthreads();
  issue_e(leaf);
  asm volatile("cp.async.commit_group;\n" ::);
  for (; leaf < end; leaf += gridDim.x) {
    const long long nxt = leaf + gridDim.x;
    const long long id = c.ninternal + leaf;
    const int m = (int)(c.hi[id] - c.lo[id]);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // ---------------- Z = X E ----------------
    {
      const int g = lane >> 2, q2 = 2 * (lane & 3), kq = lane & 3;
      for (int cc = warp; cc < Kc; cc += ZW) {
        double acc[T][2];
#pragma unroll
        for (int i = 0; i < T; i++) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
        const double *zc = sZ + (8 * cc + g) * LDR;
#pragma unroll
        for (int kb = 0; kb < T; kb++) {
          const double b0 = zc[8 * kb + kq], b1 = zc[8 * kb + 4 + kq];
#pragma unroll
          for (int i = kb; i < T; i++) {
            const double *tA = sX + tix(i, kb) * 64;
            dmma(acc[i][0], acc[i][1], tA[lane], b0);
            dmma(acc[i][0], acc[i][1], tA[32 + lane], b1);
          }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < T; i++) {
          sZ[(8 * cc + q2) * LDR + 8 * i + g] = acc[i][0];
          sZ[(8 * cc + q2 + 1) * LDR + 8 * i + g] = acc[i][1];
        }
      }
    }
    __syncthreads();
    if (nxt < end) { issue_x(nxt); asm volatile("cp.async.commit_group;\n" ::); }   // X is free
    if (K > 0) {
      // ---------------- Pi_l = Z^T Z: 16x16 output blocks, DMMA m16n8k8 ----------------
      const int Kc16 = Kz / 16;
      const int nblk = Kc16 * (Kc16 + 1) / 2;
      double *Pl = c.Pi + leaf * ((long long)K * (K + 1) / 2);
      const int kend = (m + 7) & ~7;
      const int g = lane >> 2, tq = lane & 3;
      for (int blk = warp; blk < nblk; blk += ZW) {
        const int BI = c_tileI[blk], BJ = c_tileJ[blk];
        double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0};
        const double *pa0 = sZ + (16 * BI + g) * LDR + tq;
        const double *pa1 = pa0 + 8 * LDR;
        const double *pb0 = sZ + (16 * BJ + g) * LDR + tq;
        const double *pb1 = pb0 + 8 * LDR;
        for (int k0 = 0; k0 < kend; k0 += 8) {
          const double a0 = pa0[k0], a1 = pa1[k0], a2 = pa0[k0 + 4], a3 = pa1[k0 + 4];
          dmma16(acc0, a0, a1, a2, a3, pb0[k0], pb0[k0 + 4]);
          dmma16(acc1, a0, a1, a2, a3, pb1[k0], pb1[k0 + 4]);
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const double v = q < 4 ? acc0[q] : acc1[q - 4];
          const int row = 16 * BI + g + ((q & 2) ? 8 : 0);
          const int col = 16 * BJ + 2 * tq + (q & 1) + (q >= 4 ? 8 : 0);
          if (row < K && col < K && row >= col) Pl[(long long)row * (row + 1) / 2 + col] = v;
        }
      }
    }
    if (nxt < end) for (int q = t; q < Kz; q += ZTH) colsrc[q] = leaf_colsrc(c, c.ninternal + nxt, q);
    __syncthreads();                            // Z and colsrc free / ready
    if (nxt < end) { issue_e(nxt); asm volatile("cp.async.commit_group;\n" ::); }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

}  // namespace

// Leaf fast path applies for leaf <= 128 (P = 64 or 128).
static int leaf_P(const hodlr_s *h) { return h->leaf_max <= 64 ? 64 : (h->leaf_max <= 128 ? 128 : 0); }

static LeafMmaCtx leaf_ctx(hodlr_s *h, int K, double *Pi_leaf) {
  LeafMmaCtx c;
  c.kp = h->kp; c.n = h->n; c.ninternal = h->ninternal; c.kappa = h->kappa; c.K = K; c.Kp = (K + 7) / 8 * 8;
  c.Kz = (K + 15) / 16 * 16;
  c.xs = h->xs; c.lo = h->lo; c.hi = h->hi; c.Xh = h->Xh; c.ldx = h->ldx; c.rank = h->rank; c.dt = h->d_dt;
  c.Lf = h->Lf; c.lstride = h->lstride; c.Pi = Pi_leaf; c.leaf_ld = h->leaf_ld; c.flags = h->dflags;
  c.aug = h->aug; c.y = h->y_aug; c.perm = h->perm;
  c.kps = h->d_kps; c.nseg = h->nseg;
  long long cnt;
  hodlr_own_nodes(h, h->kappa, &c.leaf0, &cnt);
  return c;
}

// Leaf Cholesky (kernel 1) on `stream`; *launched reports whether the fast path applies.
hodlr_status hodlr_leaf_chol_mma(hodlr_s *h, cudaStream_t stream, bool *launched) {
  *launched = false;
  const int P = leaf_P(h);
  if (P == 0 || h->nleaves == 0) return HODLR_OK;
  const int T = P / 8, NTILE = T * (T + 1) / 2;
  const size_t smem = sizeof(double) * ((size_t)NTILE * 64 + T * 64 + 2 * P);
  LeafMmaCtx c = leaf_ctx(h, 0, nullptr);
  int maxsm = 0;      // attributes are set to the device maximum (same value from every thread; see factor.cu)
  HCUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
#define LAUNCH_CHOL(PP, SE_)                                                                                    \
  do {                                                                                                         \
    HCUDA(hodlr_allow_smem((const void *)k_leaf_chol<PP, SE_>, h->dev));  \
    k_leaf_chol<PP, SE_><<<(int)(h->nleaves >> h->tsplit), CholCfg<PP>::NT, smem, stream>>>(c);                           \
  } while (0)
  const int kv = kv_of_kp(h->kp);
  if (P == 64) {
    if (kv == KV_SE) LAUNCH_CHOL(64, KV_SE); else if (kv == KV_M52) LAUNCH_CHOL(64, KV_M52);
    else if (kv == KV_ND) LAUNCH_CHOL(64, KV_ND); else LAUNCH_CHOL(64, KV_ANY);
  } else {
    if (kv == KV_SE) LAUNCH_CHOL(128, KV_SE); else if (kv == KV_M52) LAUNCH_CHOL(128, KV_M52);
    else if (kv == KV_ND) LAUNCH_CHOL(128, KV_ND); else LAUNCH_CHOL(128, KV_ANY);
  }
#undef LAUNCH_CHOL
  HLAUNCH(h, "k_leaf_chol");
#ifdef CHOL_TRACE
  {
    unsigned long long ts[2][6];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(ts, g_chol_stamps, sizeof(ts));
    for (int b = 0; b < 2; b++)
      fprintf(stderr, "[chol CTA %d] assemble %.2f factor %.2f logdet+X %.2f us\n", b ? 4000 : 0,
              1e-3 * (ts[b][1] - ts[b][0]), 1e-3 * (ts[b][2] - ts[b][1]), 1e-3 * (ts[b][3] - ts[b][2]));
  }
#endif
  *launched = true;
  return HODLR_OK;
}

// Z = L^{-1} E and Pi_l = Z^T Z (kernel 2) if the fast path applies (the Cholesky ran); *used reports it.
hodlr_status hodlr_leaf_factor_mma(hodlr_s *h, int K, double *Pi_leaf, bool *used) {
  *used = false;
  const int P = leaf_P(h);
  if (P == 0 || !h->chol_done) return HODLR_OK;
  const int Kp = (K + 7) / 8 * 8;
  if (Kp / 8 > 2 * ZW) return HODLR_OK;              // <= 2 8-column tiles of Z per warp (shared memory decides)
  const int Kz = (K + 15) / 16 * 16;
  if (Kz / 16 > 16) return HODLR_OK;                 // SYRK block tables cover 16 x 16 blocks
  const int T = P / 8, NTILE = T * (T + 1) / 2, LDR = P + 4;
  int maxsm = 0;
  HCUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->dev));
  size_t smem = sizeof(double) * ((size_t)NTILE * 64 + (size_t)Kz * LDR + Kz);
  bool wide = false;                                 // X from global memory when X + Z do not fit
  if (smem + 64 > (size_t)maxsm) { smem = sizeof(double) * ((size_t)Kz * LDR + Kz); wide = true; }
  if (smem + 64 > (size_t)maxsm) return HODLR_OK;
  LeafMmaCtx c = leaf_ctx(h, K, Pi_leaf);
  const int grid = (int)(h->nleaves >> h->tsplit);
#define LAUNCH_ZS(PP, XGV)                                                                                     \
  do {                                                                                                        \
    HCUDA(hodlr_allow_smem((const void *)k_leaf_zsyrk<PP, XGV>, h->dev)); \
    k_leaf_zsyrk<PP, XGV><<<grid, ZTH, smem, h->st>>>(c);                                                      \
  } while (0)
#define LAUNCH_ZSP(PP, NT, PER_SM)                                                                             \
  do {                                                                                                        \
    HCUDA(hodlr_allow_smem((const void *)k_leaf_zsyrk_p<PP, NT>, h->dev));   \
    k_leaf_zsyrk_p<PP, NT><<<std::min(grid, (PER_SM) * nsm), NT, smem, h->st>>>(c, (long long)grid);            \
  } while (0)
  int nsm = 148, maxsm_sm = 0;
  HCUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
  HCUDA(cudaDeviceGetAttribute(&maxsm_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->dev));
  const bool small = P == 64 && Kp <= 64 && 4 * (smem + 1024) <= (size_t)maxsm_sm;
  if (P == 64) { if (wide) LAUNCH_ZS(64, true); else if (small) LAUNCH_ZSP(64, 256, 4); else LAUNCH_ZSP(64, 512, 1); }
  else { if (wide) LAUNCH_ZS(128, true); else LAUNCH_ZSP(128, 512, 1); }
#undef LAUNCH_ZS
#undef LAUNCH_ZSP
  HLAUNCH(h, "k_leaf_zsyrk");
  *used = true;
  return HODLR_OK;
}
