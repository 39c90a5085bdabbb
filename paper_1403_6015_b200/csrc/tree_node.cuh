// tree_node.cuh -- the coupling-system node of the projected-Gram factorization,
// shared by the per-level tree kernel (factor.cu, children's Pi in global memory) and the fused leaf-pair
// kernel (leaf_mma.cu, children's Pi formed on chip):  S_c (Gauss-Jordan with partial pivoting, log|det|),
// T_c = S_c^{-1} B_c refined in compensated arithmetic, Pi_c = Pi_c1 + Pi_c2 - B^T T (compensated).
#pragma once
#include "hodlr_internal.cuh"
#ifndef TREE_GJ_WARP_MAX
#define TREE_GJ_WARP_MAX 8       // largest q eliminated by one warp in registers (larger: the whole CTA, one barrier
                                 // per step -- measured 66 us faster over cfg3's tree than one warp for 8 < q <= 32)
#endif
#ifndef TREE_GJ_REGS
#define TREE_GJ_REGS 16          // largest q of the register Gauss-Jordan (gj_regs up to 8, gj_cols up to 16)
#endif

struct TreeCtx {
  int d;                    // depth of the nodes of this launch
  long long i0;             // first node (index within depth d) of this launch
  long long cnt;            // nodes of depth d this launch computes (i0 .. i0 + cnt)
  int r, q, Kd, K1, ldk;    // ldk: row stride of B / T in shared memory (Kd rounded up to 4)
  int dd;                   // compensated (double-double) Pi update at this level
  int nonspd;               // kernel not positive definite: det S_c < 0 is counted, not a failure (R20)
  int *ready;               // k_tree_top: per-node progress flags (heap id; 1 = the parent's rows of Pi_c written,
                            // 2 = node done), or NULL (levels separated by kernel boundaries)
  int wait;                 // wait for the children's flags (their level ran in the same k_tree_top launch)
  int r_up;                 // rows of Pi_c the parent's coupling system and B read first: its rank r (= rdep[d])
  const double *Pi1;        // children Pi base (depth d+1), packed K1(K1+1)/2 per node
  double *Pic;              // this depth's Pi base, packed Kd(Kd+1)/2 per node
  double *Sst;              // per node: S (q*q), S^{-1} (q*q), spare (q)
  double *BT;               // per node: B, T_hi, T_lo (q*Kd each)
  double *node_ld;
  int *flags;
};

// Shared-memory footprint of one node (doubles), see tree_node().
__host__ __device__ __forceinline__ long long tree_smem_doubles(int q, int ldk) {
  return 5LL * q * q + 6LL * q + 4LL * q * ldk;
}

// Gauss-Jordan with partial pivoting on [S | I] (q <= QB rows, one row per lane, in registers), q <= 16.  Row
// interchanges are logical: every lane carries the current position `pos` of its row, so a swap is two position
// updates.  Pivot rule as the LU of the coupling system (row of max |.| among the not-yet-pivoted positions >= k,
// the smallest position on ties), hence the same pivots, U_kk and sign.  On exit the lane at position a writes row a
// of S^{-1} to Wout[a][q..2q); lane 0 writes |U_kk| to ukk[k]; returns sign and zero-pivot flag.
template <int QB>
__device__ void gj_regs(const double *W, double *Wout, int q, double *ukk, int &sign, int &zero) {
  const int lane = threadIdx.x & 31, q2 = 2 * q;
  double w[2 * QB];
#pragma unroll
  for (int j = 0; j < QB; j++) {
    w[j] = (lane < q && j < q) ? W[lane * q2 + j] : 0.0;
    w[QB + j] = (lane < q && j < q) ? W[lane * q2 + q + j] : 0.0;
  }
  int pos = lane;
  sign = 1; zero = 0;
#pragma unroll
  for (int k = 0; k < QB; k++) {
    if (k < q) {                                   // (warp-uniform; keeps the loop fully unrolled)
      double best = (lane < q && pos >= k) ? fabs(w[k]) : -1.0;
      int bp = pos, bl = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int p2 = __shfl_xor_sync(0xffffffffu, bp, o), l2 = __shfl_xor_sync(0xffffffffu, bl, o);
        if (b2 > best || (b2 == best && p2 < bp)) { best = b2; bp = p2; bl = l2; }
      }
      const int P = bl;                            // lane holding the pivot row (position bp >= k)
      if (bp != k) {                               // swap positions k and bp
        sign = -sign;
        if (pos == k) pos = bp;
        else if (lane == P) pos = k;
      }
      const double piv = __shfl_sync(0xffffffffu, w[k], P);
      if (piv < 0.0) sign = -sign;
      if (!(piv != 0.0)) zero = 1;
      if (lane == 0) ukk[k] = fabs(piv);
      const double ip = piv != 0.0 ? 1.0 / piv : 0.0;
      const double mlt = lane == P ? 0.0 : w[k] * ip;
#pragma unroll
      for (int j = 0; j < QB; j++) {               // (constant trip count: fully unrolled, w stays in registers)
        if (j > k && j < q) {
          const double prj = __shfl_sync(0xffffffffu, w[j], P);
          w[j] = lane == P ? w[j] * ip : fma(-mlt, prj, w[j]);
        }
      }
      w[k] = lane == P ? 1.0 : 0.0;
#pragma unroll
      for (int j = QB; j < 2 * QB; j++) {
        if (j - QB < q) {
          const double prj = __shfl_sync(0xffffffffu, w[j], P);
          w[j] = lane == P ? w[j] * ip : fma(-mlt, prj, w[j]);
        }
      }
    }
  }
  if (lane < q) {
#pragma unroll
    for (int j = 0; j < QB; j++) if (j < q) Wout[pos * q2 + q + j] = w[QB + j];
  }
}

// The same elimination with one COLUMN of [S | I] per lane (2q <= 32 columns, q <= QB rows in registers), for
// 8 < q <= 16: per step the pivot column's lane scans its own q entries for the pivot, and every lane updates its
// column with the multipliers broadcast from that lane -- q shuffles per step instead of the row layout's 2q, and
// no per-lane 2q-register rows.  Logical interchanges (every lane carries the same position table), the row layout's
// exact arithmetic (multiplier W[a][k] * (1 / piv), one FMA per entry, pivot row scaled), hence bitwise its result.
template <int QB>
__device__ void gj_cols(const double *W, double *Wout, int q, double *ukk, int &sign, int &zero) {
  const int lane = threadIdx.x & 31, q2 = 2 * q;
  const bool act = lane < q2;
  double cl[QB];
  int pos[QB];
#pragma unroll
  for (int a = 0; a < QB; a++) { cl[a] = (act && a < q) ? W[a * q2 + lane] : 0.0; pos[a] = a; }
  sign = 1; zero = 0;
  for (int k = 0; k < q; k++) {
    // pivot: physical row of max |W[., k]| among positions >= k, smallest position on ties (lane k's column)
    double best = -1.0; int bp = 1 << 30, P = 0;
#pragma unroll
    for (int a = 0; a < QB; a++)
      if (a < q && pos[a] >= k) {
        const double v = fabs(cl[a]);
        if (v > best || (v == best && pos[a] < bp)) { best = v; bp = pos[a]; P = a; }
      }
    P = __shfl_sync(0xffffffffu, P, k);
    double pj = 0.0;                               // this lane's entry of the pivot row
#pragma unroll
    for (int a = 0; a < QB; a++) if (a == P) pj = cl[a];
    const double piv = __shfl_sync(0xffffffffu, pj, k);
    int posP = 0;
#pragma unroll
    for (int a = 0; a < QB; a++) if (a == P) posP = pos[a];
    if (posP != k) {                               // swap positions k and posP
      sign = -sign;
#pragma unroll
      for (int a = 0; a < QB; a++) { if (pos[a] == k) pos[a] = posP; else if (a == P) pos[a] = k; }
    }
    if (piv < 0.0) sign = -sign;
    if (!(piv != 0.0)) zero = 1;
    if (lane == 0) ukk[k] = fabs(piv);
    const double ip = piv != 0.0 ? 1.0 / piv : 0.0;
#pragma unroll
    for (int a = 0; a < QB; a++) {
      if (a < q) {
        const double mlt = __shfl_sync(0xffffffffu, cl[a], k) * ip;     // (lane k's column: W[a][k])
        cl[a] = a == P ? cl[a] * ip : fma(-mlt, pj, cl[a]);
      }
    }
    if (lane == k) {
#pragma unroll
      for (int a = 0; a < QB; a++) cl[a] = a == P ? 1.0 : 0.0;
    }
  }
  if (act && lane >= q) {
#pragma unroll
    for (int a = 0; a < QB; a++) if (a < q) Wout[pos[a] * q2 + lane] = cl[a];
  }
}

// The same elimination for 8 < q <= 32 by one warp in shared memory, no CTA barrier.  [S | I] is first transposed
// from W (row-major, stride 2q) into Wt (column-major: element (a, j) at j q + a), so that the lanes (one row each)
// touch consecutive words and the pivot row is a broadcast -- a row-major layout with stride 2q puts 8 lanes on each
// bank group.  Logical interchanges as above, and no pivot-row scaling during the sweep (each non-pivot row
// subtracts (Wt[a][k] / Wt[P][k]) row_P, the pivot row is left as it is); at the end the lane of position a divides
// its right half by its pivot and writes row a of S^{-1} to Wout[a][q..2q) (row-major, stride 2q; Wout may be W).
// Same pivots and U_kk as the LU.
static __device__ void gj_warp(const double *W, double *Wt, double *Wout, int q, double *ukk, int &sign, int &zero) {
  const int lane = threadIdx.x & 31, q2 = 2 * q;
  for (int a = 0; a < q; a++)
    for (int j = lane; j < q2; j += 32) Wt[j * q + a] = W[a * q2 + j];
  __syncwarp();
  int pos = lane;
  sign = 1; zero = 0;
  for (int k = 0; k < q; k++) {
    double best = (lane < q && pos >= k) ? fabs(Wt[k * q + lane]) : -1.0;
    int bp = pos, bl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int p2 = __shfl_xor_sync(0xffffffffu, bp, o), l2 = __shfl_xor_sync(0xffffffffu, bl, o);
      if (b2 > best || (b2 == best && p2 < bp)) { best = b2; bp = p2; bl = l2; }
    }
    const int P = bl;
    if (bp != k) {
      sign = -sign;
      if (pos == k) pos = bp;
      else if (lane == P) pos = k;
    }
    const double piv = Wt[k * q + P];
    if (piv < 0.0) sign = -sign;
    if (!(piv != 0.0)) zero = 1;
    if (lane == 0) ukk[k] = fabs(piv);
    if (lane < q && lane != P) {
      const double mlt = piv != 0.0 ? Wt[k * q + lane] / piv : 0.0;
      // columns k+1 .. 2q-1 (column k becomes 0), 8 at a time: all loads of a batch before its stores
      for (int j0 = k + 1; j0 < q2; j0 += 8) {
        double pv[8], rv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int j = j0 + u < q2 ? j0 + u : q2 - 1;
          pv[u] = Wt[j * q + P]; rv[u] = Wt[j * q + lane];
        }
#pragma unroll
        for (int u = 0; u < 8; u++) if (j0 + u < q2) Wt[(j0 + u) * q + lane] = fma(-mlt, pv[u], rv[u]);
      }
      Wt[k * q + lane] = 0.0;
    }
    __syncwarp();
  }
  if (lane < q) {
    const double d = Wt[pos * q + lane];
    const double id = d != 0.0 ? 1.0 / d : 0.0;
    for (int j = 0; j < q; j++) Wout[pos * q2 + q + j] = Wt[(q + j) * q + lane] * id;
  }
  __syncwarp();
}

// One CTA per depth-d node c (heap index (2^d - 1) + i):
//   S_c = [[I, Pi_c2[s,s]], [Pi_c1[s,s], I]]; Gauss-Jordan with partial pivoting (row of max |.|, first
//   index on ties -- the same pivots and U_kk as the LU of the paper's coupling system) gives log|det S_c|,
//   its sign and S_c^{-1};
//   T_c = S_c^{-1} B_c, refined in compensated arithmetic (T = T_hi + T_lo);
//   Pi_c = Pi_c1[a,a] + Pi_c2[a,a] - sum_u B_c[(u+r) mod q, a] T_c[u, b], 4x2 register tiles per thread.
// Children's projected Gram matrices from global memory (packed, one per child at depth d+1).
struct GlobalPi {
  const double *P1, *P2;    // Pi_c1, Pi_c2 (packed lower triangles)
  int Kd;
  __device__ double s21(int a, int b) const { return P2[pk(Kd + a, Kd + b)]; }   // Pi_c2[s_a, s_b]
  __device__ double s12(int a, int b) const { return P1[pk(Kd + a, Kd + b)]; }   // Pi_c1[s_a, s_b]
  __device__ double b2(int a, int col) const { return P2[pk(Kd + a, col)]; }     // Pi_c2[s_a, col]
  __device__ double b1(int a, int col) const { return P1[pk(Kd + a, col)]; }     // Pi_c1[s_a, col]
  template <bool DD> __device__ void d(int a, int b, double &hs, double &ls) const {   // Pi_c1[a,b] + Pi_c2[a,b]
    const long long pp = (long long)a * (a + 1) / 2 + b;
    if (DD) two_sum(__ldg(P1 + pp), __ldg(P2 + pp), hs, ls); else { hs = __ldg(P1 + pp) + __ldg(P2 + pp); ls = 0.0; }
  }
};

#ifdef TREE_TRACE
#include <stdio.h>
#define TSTAMP(k) if (threadIdx.x == 0 && i == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tts[k])); }
#else
#define TSTAMP(k)
#endif
// Node-level dependencies inside k_tree_top (instead of a grid barrier per level): a parent starts as soon as its
// children have written the bottom rows of their Pi (the ones its S_c and B_c read) and runs its Gauss-Jordan,
// T and refinement while the children finish the rest of their Pi.
__device__ __forceinline__ void tree_wait(const int *f, int v) {
  int x;
  while (true) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(x) : "l"(f) : "memory");
    if (x >= v) break;
    __nanosleep(100);
  }
}
__device__ __forceinline__ void tree_signal(int *f, int v) {    // after a CTA barrier that follows the writes
  asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ void tree_wait_children(const TreeCtx &c, long long node, int v) {
  if (c.ready && c.wait) {
    if (threadIdx.x == 0) { tree_wait(c.ready + 2 * node + 1, v); tree_wait(c.ready + 2 * node + 2, v); }
    __syncthreads();
  }
}

template <bool DD, class Src, int QMAX = 32, bool PIDD = true>
__device__ void tree_node(const TreeCtx &c, long long i, double *sm, const Src &src) {
  const int t = threadIdx.x, NT = blockDim.x;
#ifdef TREE_TRACE
  unsigned long long tts[10] = {0};
#endif
  TSTAMP(0)
  const long long node = (1LL << c.d) - 1 + i;
  const int r = c.r, q = c.q, Kd = c.Kd, ldk = c.ldk, q2 = 2 * q;
  double *W = sm;                    // q x 2q  [S | I] -> [I | S^{-1}]
  double *S0 = W + q * q2;           // q x q
  double *rowk = S0 + q * q;         // 2q
  double *rowold = rowk + q2;        // 2q
  double *colk = rowold + q2;        // q: |U_kk|
  double *mult = colk + q;           // q: elimination multipliers of the current step
  double *W2 = mult + q;             // q x 2q: Gauss-Jordan ping-pong buffer
  double *B = W2 + q * q2;           // q x ldk
  double *Th = B + (long long)q * ldk;
  double *Tl = Th + (long long)q * ldk;
  double *R = Tl + (long long)q * ldk;
  __shared__ int s_zero, s_sign, s_nref;
  tree_wait_children(c, node, 1);              // (k_tree_top) the children's bottom rows of Pi
  for (int p = t; p < q * q2; p += NT) {
    const int a = p / q2, b = p - a * q2;
    double v;
    if (b >= q) v = (b - q == a) ? 1.0 : 0.0;
    else {
      v = a == b ? 1.0 : 0.0;
      if (a < r && b >= r) v = src.s21(a, b - r);
      if (a >= r && b < r) v = src.s12(a - r, b);
      S0[a * q + b] = v;
    }
    W[p] = v;
  }
  for (int p = t; p < q * ldk; p += NT) {
    const int a = p / ldk, b = p - a * ldk;
    double v = 0.0;
    if (b < Kd) v = a < r ? src.b2(a, b) : src.b1(a - r, b);
    B[p] = v; Tl[p] = 0.0;
  }
  __syncthreads();
  TSTAMP(1)
  // ---------------- Gauss-Jordan with partial pivoting ----------------
  // q <= TREE_GJ_WARP_MAX (8): warp 0 in registers (gj_regs); larger systems: the whole CTA, one barrier per step
  // (gj_cols / gj_warp, one warp for q <= 16 / 32, measured slower).  (S^{-1} goes to W2, row-major, or wherever the
  // last ping-pong step left it; gj_warp uses W2 as its transposed work area and then writes S^{-1} into W.)
  // One warp needs ~1000 cycles per elimination step at q = 8 and ~2700 at q = 26 (tools/micro/gj_bench.cu); a
  // two-warp column layout and a software-pipelined row sweep were no faster.
  if (q <= TREE_GJ_WARP_MAX) {
    if (t < 32) {
      int sign, zero;
      if (q <= 8) gj_regs<8>(W, W2, q, colk, sign, zero);
      else if (q <= TREE_GJ_REGS) gj_cols<16>(W, W2, q, colk, sign, zero);
      else if (QMAX > 16) gj_warp(W, W2, W, q, colk, sign, zero);
      if (t == 0) { s_sign = sign; s_zero = zero; }
    }
  } else {
    // ping-pong buffers (read Wa, write Wb), one barrier per step; every warp finds the pivot itself
    double *Wa = W, *Wb = W2;
    const int lane = t & 31;
    int sign = 1, zero = 0;
    for (int k = 0; k < q; k++) {
      int p = k; double best = -1.0;
      for (int a = k + lane; a < q; a += 32) { const double v = fabs(Wa[a * q2 + k]); if (v > best) { best = v; p = a; } }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {     // xor butterfly: every lane ends with the same (best, p)
        const double b2 = __shfl_xor_sync(0xffffffffu, best, o); const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
        if (b2 > best || (b2 == best && p2 < p)) { best = b2; p = p2; }
      }
      const double piv = Wa[p * q2 + k];
      if (t == 0) {
        colk[k] = best;                        // |U_kk| (log det below)
        if (p != k) sign = -sign;
        if (piv < 0.0) sign = -sign;
        if (!(piv != 0.0)) zero = 1;
      }
      const double ip = piv != 0.0 ? 1.0 / piv : 0.0;
      const double *prow = Wa + p * q2;
      if (q2 <= 64) {                          // thread = (column j, every NT/64-th row): no index division
        const int j = t & 63;
        if (j < q2) {
          const double pj = prow[j];
          for (int a = t >> 6; a < q; a += NT >> 6) {
            if (a == k) Wb[a * q2 + j] = pj * ip;
            else {
              const int sa = a == p ? k : a;   // rows k and p swap before the elimination
              Wb[a * q2 + j] = fma(-Wa[sa * q2 + k] * ip, pj, Wa[sa * q2 + j]);
            }
          }
        }
      } else {
        for (int e = t; e < q * q2; e += NT) {
          const int a = e / q2, j = e - a * q2;
          if (a == k) Wb[e] = prow[j] * ip;
          else {
            const int sa = a == p ? k : a;     // rows k and p swap before the elimination
            Wb[e] = fma(-Wa[sa * q2 + k] * ip, prow[j], Wa[sa * q2 + j]);
          }
        }
      }
      __syncthreads();
      double *tmp = Wa; Wa = Wb; Wb = tmp;
    }
    if (t == 0) { s_sign = sign; s_zero = zero; }
  }
  __syncthreads();
  TSTAMP(2)
  if (t < 32) {                                 // log|det S_c| = sum_k log|U_kk|, fixed-order warp reduction
    double la = 0.0, umax = 0.0, umin = 1e300;
    for (int k = t; k < q; k += 32) { const double u = colk[k]; la += log(u); umax = fmax(umax, u); umin = fmin(umin, u); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      la += __shfl_xor_sync(0xffffffffu, la, o);
      umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
      umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, o));
    }
    if (t == 0) {
      const bool zero = s_zero != 0;
      c.node_ld[node] = la;
      if (zero || (s_sign <= 0 && !c.nonspd)) { atomicAdd(&c.flags[1], 1); atomicMin(&c.flags[2], (int)node); }
      else if (s_sign < 0) atomicAdd(&c.flags[10], 1);          // det S_c < 0: allowed when not SPD (R20)
      // refinement steps: one when the pivot growth ratio is mild, two otherwise (cond(S_c) up to ~1e12)
      s_nref = (!zero && umax < 1e6 * umin) ? 1 : 2;
    }
  }
  __syncthreads();
  TSTAMP(3)
  const bool zero = s_zero != 0;
  // S^{-1}, row stride 2q: W2 (gj_regs), W (gj_warp), or wherever the last ping-pong step left it
  const double *Si = (q <= TREE_GJ_WARP_MAX ? (q <= TREE_GJ_REGS ? W2 : W) : ((q & 1) ? W2 : W)) + q;
  if (!zero && Kd > 0) {
    const int qK = q * ldk;
    for (int e = t; e < qK; e += NT) {                // T_hi = S^{-1} B
      const int a = e / ldk, col = e - a * ldk;
      double s = 0.0;
      for (int j = 0; j < q; j++) s = fma(Si[a * q2 + j], B[j * ldk + col], s);
      Th[e] = s;
    }
    __syncthreads();
    TSTAMP(4)
    const int nref = s_nref;
    for (int it = 0; it < nref; it++) {               // iterative refinement, residual compensated
      for (int e = t; e < qK; e += NT) {
        const int a = e / ldk, col = e - a * ldk;
        if (DD) {
          Acc2 A = acc2(B[e]);
          for (int k = 0; k < q; k++) acc_fma_dd(A, -S0[a * q + k], Th[k * ldk + col], Tl[k * ldk + col]);
          R[e] = acc_val(A);
        } else {
          double s = B[e];
          for (int k = 0; k < q; k++) s = fma(-S0[a * q + k], Th[k * ldk + col] + Tl[k * ldk + col], s);
          R[e] = s;
        }
      }
      __syncthreads();
      for (int e = t; e < qK; e += NT) {
        const int a = e / ldk, col = e - a * ldk;
        double s = 0.0;
        for (int j = 0; j < q; j++) s = fma(Si[a * q2 + j], R[j * ldk + col], s);
        Tl[e] += s;
      }
      __syncthreads();
    }
    TSTAMP(5)
    // ---------------- Pi_c, 4x2 register tiles over the packed lower triangle ----------------
    // Bands of 4 rows; band P (rows 4P .. 4P+3) holds column tiles J = 0 .. 2P+1 (columns 2J, 2J+1); tiles up to
    // band P: (P+1)(P+2).  Consecutive threads take consecutive column pairs of a band: their T reads are
    // consecutive 16-byte words (conflict-free double2 loads) and their B reads one broadcast -- a 2x4 tile with
    // 4-column strides per lane had made every T load an 8-way bank conflict (the deep levels' bottleneck).
    double *Pc = c.Pic + i * ((long long)Kd * (Kd + 1) / 2);
    const bool PDD = DD && PIDD && c.dd;   // compensated Pi update (all but the deepest levels)
    const int NB = (Kd + 3) >> 2;
    const int ntile = NB * (NB + 1);
    tree_wait_children(c, node, 2);            // (k_tree_top) the children's whole Pi
    auto pi_tile = [&](int tile) {
      int P = (int)((sqrt(4.0 * (double)tile + 1.0) - 1.0) * 0.5);
      while (P * (P + 1) > tile) P--;
      while ((P + 1) * (P + 2) <= tile) P++;
      const int a0 = 4 * P, b0 = 2 * (tile - P * (P + 1));
      double hs[4][2], ls[4][2];
#pragma unroll
      for (int ii = 0; ii < 4; ii++)
#pragma unroll
        for (int jj = 0; jj < 2; jj++) {
          const int a = a0 + ii, b = b0 + jj;
          double s = 0.0, e = 0.0;
          if (a < Kd && b <= a) {                                 // packed (a, b): same index in both children
            if (PDD) src.template d<true>(a, b, s, e); else src.template d<false>(a, b, s, e);
          }
          hs[ii][jj] = s; ls[ii][jj] = e;
        }
      for (int u = 0; u < q; u++) {
        const int ub = u < q - r ? u + r : u + r - q;
        const double *bu = B + (long long)ub * ldk + a0;
        const double2 th2 = *(const double2 *)(Th + (long long)u * ldk + b0);
        const double2 tl2 = *(const double2 *)(Tl + (long long)u * ldk + b0);
        const double th[2] = {th2.x, th2.y}, tl[2] = {tl2.x, tl2.y};
        double bv[4];
#pragma unroll
        for (int x = 0; x < 4; x++) bv[x] = -bu[x];
#pragma unroll
        for (int ii = 0; ii < 4; ii++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            if (PDD) {
              double pr, pe, s2, e2;
              two_prod(bv[ii], th[jj], pr, pe);
              two_sum(hs[ii][jj], pr, s2, e2);
              hs[ii][jj] = s2;
              ls[ii][jj] += e2 + fma(bv[ii], tl[jj], pe);
            } else {
              hs[ii][jj] = fma(bv[ii], th[jj] + tl[jj], hs[ii][jj]);
            }
          }
      }
#pragma unroll
      for (int ii = 0; ii < 4; ii++)
#pragma unroll
        for (int jj = 0; jj < 2; jj++) {
          const int a = a0 + ii, b = b0 + jj;
          if (a < Kd && b <= a) Pc[(long long)a * (a + 1) / 2 + b] = hs[ii][jj] + ls[ii][jj];
        }
    };
    // (k_tree_top) the bands holding the parent's rows first, then the flag, then the rest
    const int Pb = c.ready ? max(0, (Kd - c.r_up) >> 2) : 0, tb = Pb * (Pb + 1);
    for (int tile = tb + t; tile < ntile; tile += NT) pi_tile(tile);
    if (c.ready) {
      __threadfence();
      __syncthreads();
      if (t == 0) tree_signal(c.ready + node, 1);
    }
    for (int tile = t; tile < tb; tile += NT) pi_tile(tile);
  }
  TSTAMP(6)
  // persist S, S^{-1}, B, T_hi, T_lo for the solve
  double *Sg = c.Sst + i * (long long)(2 * q * q + q);
  for (int p = t; p < q * q; p += NT) {
    const int a = p / q, b = p - a * q;
    Sg[p] = S0[p];
    Sg[q * q + p] = Si[a * q2 + b];
  }
  const long long qKd = (long long)q * Kd;
  double *BTg = c.BT + i * 3LL * qKd;
  for (long long p = t; p < qKd; p += NT) {
    const int a = (int)(p / Kd), b = (int)(p - (long long)a * Kd);
    BTg[p] = B[a * ldk + b];
    BTg[qKd + p] = Th[a * ldk + b];
    BTg[2 * qKd + p] = Tl[a * ldk + b];
  }
  if (c.ready) __threadfence();
  __syncthreads();
  if (c.ready && t == 0) tree_signal(c.ready + node, 2);
  TSTAMP(7)
#ifdef TREE_TRACE
  if (threadIdx.x == 0 && i == 0)
    printf("[tree d=%d q=%d Kd=%d] load %.2f gj %.2f logdet %.2f T %.2f refine %.2f Pi %.2f store %.2f us\n", c.d, q, Kd,
           1e-3 * (tts[1] - tts[0]), 1e-3 * (tts[2] - tts[1]), 1e-3 * (tts[3] - tts[2]), 1e-3 * (tts[4] - tts[3]),
           1e-3 * (tts[5] - tts[4]), 1e-3 * (tts[6] - tts[5]), 1e-3 * (tts[7] - tts[6]));
#endif
}

