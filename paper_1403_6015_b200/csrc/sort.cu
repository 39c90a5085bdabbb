// sort.cu -- G1: stable ascending argsort of the FP64 points (the kd-tree
// ordering reduces to a sort in 1-D; ties keep the lower original index).
//
// LSD radix sort on order-preserving 64-bit keys, 8 passes of 8-bit digits.  Each pass:
//   hist    : per 4096-key tile digit counts             (HBM-bound, 8 B/key read)
//   scan    : per-digit exclusive scan over tiles (256 CTAs) + digit totals
//   scatter : stable tile-local ranks via __match_any_sync + per-warp counters, then scatter
//             (HBM-bound, 16 B/key read + 16 B/key write)
// Stability: tiles are ranked in order, warps within a tile in order, keys within a warp in order.
#include "hodlr_internal.cuh"
#include <mutex>
#include <vector>

namespace {

constexpr int TILE = 4096;
constexpr int STHREADS = 512;    // 16 warps x 256 keys

// Keys + the identity result (xs = x, perm = iota) + a sortedness flag: an already ascending x
// (ties included) has the identity as its stable argsort, and the radix passes are skipped.
__global__ void k_make_keys(const double *__restrict__ x, long long n, unsigned long long *__restrict__ key,
                            long long *__restrict__ idx, double *__restrict__ xs, long long *__restrict__ perm,
                            int *__restrict__ flags) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = x[i];
  if (!isfinite(v)) atomicOr(&flags[0], 1);
  if (v == 0.0) v = 0.0;                        // -0.0 -> +0.0 before sorting
  if (i + 1 < n && !(v <= x[i + 1])) atomicOr(&flags[7], 1);   // -0.0 <= +0.0 holds, so ties stay ties
  xs[i] = v;
  perm[i] = i;
  unsigned long long b = __double_as_longlong(v);
  b ^= (b >> 63) ? 0xffffffffffffffffULL : 0x8000000000000000ULL;
  key[i] = b;
  idx[i] = i;
}

__device__ __forceinline__ void hist_body(const unsigned long long *__restrict__ key, long long n, int shift,
                                          int ntiles, unsigned int *__restrict__ cnt) {
  __shared__ unsigned int c[256];
  for (int t = threadIdx.x; t < 256; t += STHREADS) c[t] = 0;
  __syncthreads();
  long long base = (long long)blockIdx.x * TILE;
  for (int t = threadIdx.x; t < TILE; t += STHREADS) {
    long long p = base + t;
    if (p < n) atomicAdd(&c[(key[p] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += STHREADS) cnt[(long long)t * ntiles + blockIdx.x] = c[t];
}

// per digit d (one CTA each): exclusive scan of cnt[d][0..ntiles) in place, digit total to tot[d]
__device__ __forceinline__ void scan_digit_body(unsigned int *__restrict__ cnt, int ntiles,
                                                unsigned int *__restrict__ tot) {
  __shared__ unsigned int part[256];
  unsigned int *a = cnt + (long long)blockIdx.x * ntiles;
  const int per = (ntiles + 255) / 256;
  const int b = threadIdx.x * per, e = min(b + per, ntiles);
  unsigned int v[16];
  unsigned int s = 0;
  for (int i = b, k = 0; i < e; i++, k++) { v[k] = a[i]; s += v[k]; }
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    unsigned int x = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += x;
    __syncthreads();
  }
  unsigned int run = part[threadIdx.x] - s;
  for (int i = b, k = 0; i < e; i++, k++) { a[i] = run; run += v[k]; }
  if (threadIdx.x == 255) tot[blockIdx.x] = part[255];
}

__device__ __forceinline__ void scatter_body(const unsigned long long *__restrict__ kin,
                                                      const long long *__restrict__ iin, long long n, int shift,
                                                      int ntiles, const unsigned int *__restrict__ gscan,
                                                      const unsigned int *__restrict__ tot,
                                                      unsigned long long *__restrict__ kout,
                                                      long long *__restrict__ iout) {
  __shared__ unsigned int wc[16][256];
  __shared__ unsigned int dbase[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < 16 * 256; t += STHREADS) (&wc[0][0])[t] = 0;
  __syncthreads();
  const long long base = (long long)blockIdx.x * TILE + warp * 256;
  unsigned long long k[8]; long long id[8]; unsigned int loc[8]; int dig[8];
  const unsigned int lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    long long p = base + r * 32 + lane;
    bool valid = p < n;
    k[r] = valid ? kin[p] : 0ull;
    id[r] = valid ? iin[p] : 0;
    int d = valid ? (int)((k[r] >> shift) & 255u) : 256;
    dig[r] = d;
    unsigned int peers = __match_any_sync(0xffffffffu, d);
    unsigned int before = 0;
    if (valid) before = wc[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wc[warp][d] = before + __popc(peers);
    __syncwarp();
    loc[r] = before + __popc(peers & lt);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += STHREADS) {
    unsigned int run = 0;
    for (int w = 0; w < 16; w++) { unsigned int t = wc[w][d]; wc[w][d] = run; run += t; }
  }
  if (threadIdx.x < 32) {          // exclusive scan of the 256 digit totals (8 per lane)
    const int l = threadIdx.x;
    unsigned int v[8], s = 0;
    for (int k = 0; k < 8; k++) { v[k] = tot[8 * l + k]; s += v[k]; }
    unsigned int inc = s;
    for (int o = 1; o < 32; o <<= 1) { unsigned int x = __shfl_up_sync(0xffffffffu, inc, o); if (l >= o) inc += x; }
    unsigned int run = inc - s;
    for (int k = 0; k < 8; k++) { dbase[8 * l + k] = run; run += v[k]; }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; r++) {
    if (dig[r] == 256) continue;
    long long dst = (long long)dbase[dig[r]] + gscan[(long long)dig[r] * ntiles + blockIdx.x] + wc[warp][dig[r]] + loc[r];
    kout[dst] = k[r];
    iout[dst] = id[r];
  }
}

__device__ __forceinline__ void finish_body(const unsigned long long *__restrict__ key, const long long *__restrict__ idx,
                                            long long n, double *__restrict__ xs, long long *__restrict__ perm) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long b = key[i];
  b ^= (b >> 63) ? 0x8000000000000000ULL : 0xffffffffffffffffULL;
  xs[i] = __longlong_as_double((long long)b);
  perm[i] = idx[i];
}

// The radix passes as one CUDA graph behind a conditional IF node set on the device from k_make_keys's flags:
// nothing runs for an ascending (or non-finite) x, and the build needs no host round trip to decide.  The graph's
// kernels read their buffers from a plan-owned context (rewritten per build), so the graph is instantiated once per
// (n, device).
struct SortCtx {
  unsigned long long *k0, *k1;
  long long *i0, *i1;
  unsigned int *cnt, *tot;
  long long n; int ntiles;
  double *xs; long long *perm;
  const int *flags;
};
__global__ void k_sort_cond(cudaGraphConditionalHandle hdl, const SortCtx *__restrict__ c) {
  cudaGraphSetConditional(hdl, (c->flags[7] && !c->flags[0]) ? 1u : 0u);   // unsorted and finite
}
__global__ void __launch_bounds__(STHREADS) k_hist(const SortCtx *__restrict__ c, int pass) {
  hist_body(pass & 1 ? c->k1 : c->k0, c->n, 8 * pass, c->ntiles, c->cnt);
}
__global__ void __launch_bounds__(256) k_scan_digit(const SortCtx *__restrict__ c) {
  scan_digit_body(c->cnt, c->ntiles, c->tot);
}
__global__ void __launch_bounds__(STHREADS) k_scatter(const SortCtx *__restrict__ c, int pass) {
  const bool odd = pass & 1;
  scatter_body(odd ? c->k1 : c->k0, odd ? c->i1 : c->i0, c->n, 8 * pass, c->ntiles, c->cnt, c->tot,
               odd ? c->k0 : c->k1, odd ? c->i0 : c->i1);
}
__global__ void k_finish(const SortCtx *__restrict__ c) {            // 8 passes: the result is back in k0 / i0
  finish_body(c->k0, c->i0, c->n, c->xs, c->perm);
}

struct SortPlan { long long n; int dev; SortCtx *d_ctx = nullptr; cudaGraphExec_t ge = nullptr; bool busy = false; };
static std::mutex g_sort_mu;
static std::vector<SortPlan *> g_sort_plans;

static cudaError_t sort_graph(SortPlan *P, int ntiles, int nb) {
  cudaError_t e = cudaMalloc((void **)&P->d_ctx, sizeof(SortCtx));
  cudaGraph_t g = nullptr;
  if (e == cudaSuccess) e = cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle hdl;
  if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hdl, g, 0, cudaGraphCondAssignDefault);
  const SortCtx *pc = P->d_ctx;
  void *acond[] = {(void *)&hdl, (void *)&pc};
  cudaGraphNode_t ncond = nullptr, nif = nullptr, prev = nullptr;
  if (e == cudaSuccess) {
    cudaKernelNodeParams k = {};
    k.func = (void *)k_sort_cond; k.gridDim = dim3(1); k.blockDim = dim3(1); k.kernelParams = acond;
    e = cudaGraphAddKernelNode(&ncond, g, nullptr, 0, &k);
  }
  cudaGraphNodeParams cpar = {};
  if (e == cudaSuccess) {
    cpar.type = cudaGraphNodeTypeConditional;
    cpar.conditional.handle = hdl; cpar.conditional.type = cudaGraphCondTypeIf; cpar.conditional.size = 1;
    e = cudaGraphAddNode(&nif, g, &ncond, 1, &cpar);
  }
  int passes[8];
  for (int p = 0; p < 8; p++) passes[p] = p;
  if (e == cudaSuccess) {
    cudaGraph_t body = cpar.conditional.phGraph_out[0];
    for (int p = 0; p < 8 && e == cudaSuccess; p++) {
      void *ap[] = {(void *)&pc, (void *)&passes[p]};
      void *as[] = {(void *)&pc};
      cudaKernelNodeParams k = {};
      cudaGraphNode_t n1, n2, n3;
      k.func = (void *)k_hist; k.gridDim = dim3(ntiles); k.blockDim = dim3(STHREADS); k.kernelParams = ap;
      e = cudaGraphAddKernelNode(&n1, body, prev ? &prev : nullptr, prev ? 1 : 0, &k);
      if (e != cudaSuccess) break;
      k.func = (void *)k_scan_digit; k.gridDim = dim3(256); k.blockDim = dim3(256); k.kernelParams = as;
      e = cudaGraphAddKernelNode(&n2, body, &n1, 1, &k);
      if (e != cudaSuccess) break;
      k.func = (void *)k_scatter; k.gridDim = dim3(ntiles); k.blockDim = dim3(STHREADS); k.kernelParams = ap;
      e = cudaGraphAddKernelNode(&n3, body, &n2, 1, &k);
      prev = n3;
    }
    if (e == cudaSuccess) {
      void *as[] = {(void *)&pc};
      cudaKernelNodeParams k = {};
      cudaGraphNode_t n4;
      k.func = (void *)k_finish; k.gridDim = dim3(nb); k.blockDim = dim3(256); k.kernelParams = as;
      e = cudaGraphAddKernelNode(&n4, body, &prev, 1, &k);
    }
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&P->ge, g, 0);
  if (g) cudaGraphDestroy(g);
  return e;
}

// ---------------------------------------------------------------------------------------------------------------
// NEXT-3: the kd ordering of d-dimensional points ("sorted recursively, one dimension at a time";
// DESIGN.md R19): for L = 0 .. max(kappa, 1) - 1, top down, every depth-L node sorts its points stably by
// coordinate L mod d, and the count-median split halves it.  One level is one stable LSD radix sort of the whole
// array by (node, coordinate): 8 digit passes on the coordinate's order-preserving key, then ceil(L / 8) passes on
// the depth-L node index -- equal nodes keep the coordinate order, equal coordinates the previous order, which is
// each node's stable sort -- then one gather of the coordinate rows and the permutation.
// ---------------------------------------------------------------------------------------------------------------
__global__ void k_kd_init(const double *__restrict__ x, long long n, int dim, double *__restrict__ xs,
                          long long *__restrict__ perm, int *__restrict__ flags) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int k = 0; k < dim; k++) {
    double v = x[i * dim + k];
    if (!isfinite(v)) atomicOr(&flags[0], 1);
    if (v == 0.0) v = 0.0;                      // -0.0 -> +0.0
    xs[k * n + i] = v;
  }
  perm[i] = i;
}
__global__ void k_kd_keys(const double *__restrict__ xa, long long n, unsigned long long *__restrict__ key,
                          long long *__restrict__ idx) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long b = __double_as_longlong(xa[i]);
  b ^= (b >> 63) ? 0xffffffffffffffffULL : 0x8000000000000000ULL;
  key[i] = b;
  idx[i] = i;
}
// node key of the element that came from position idx[i]: the depth-L node whose rows contain that position
__global__ void k_kd_nodekeys(const long long *__restrict__ idx, long long n, const long long *__restrict__ lo, int L,
                              unsigned long long *__restrict__ key) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long p = idx[i], base = (1LL << L) - 1;
  long long a = 0, b = (1LL << L) - 1;            // largest j in [a, b] with lo[base + j] <= p
  while (a < b) { const long long m = (a + b + 1) >> 1; if (lo[base + m] <= p) a = m; else b = m - 1; }
  key[i] = (unsigned long long)a;
}
__global__ void k_kd_gather(const long long *__restrict__ idx, long long n, int dim, const double *__restrict__ xin,
                            const long long *__restrict__ pin, double *__restrict__ xout, long long *__restrict__ pout) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long j = idx[i];
  for (int k = 0; k < dim; k++) xout[k * n + i] = xin[k * n + j];
  pout[i] = pin[j];
}
// The deep levels in one launch: CTA b takes the depth-L0 node b (m <= KD_LOCAL points) and runs levels L0 .. levels-1
// in shared memory.  At level L each depth-L sub-node is sorted by (coordinate key, position) with its own bitonic
// network over S = 2^ceil(log2(largest sub-node)) slots (padding slots sort last): the tuples are distinct, so the
// result is each sub-node's stable sort by that coordinate (the global passes' result).  Points are read through the
// running order cur[] (coordinate-major input, L1/L2-cached).
constexpr int KD_LOCAL = 4096, KD_LT = 512;
constexpr size_t KD_LOCAL_SMEM = 2 * KD_LOCAL * (8 + 4) + KD_LOCAL * (2 + 2);
__global__ void __launch_bounds__(KD_LT) k_kd_local(const double *__restrict__ xin, const long long *__restrict__ pin,
                                                    long long n, int dim, int L0, int levels,
                                                    const long long *__restrict__ lo, const long long *__restrict__ hi,
                                                    double *__restrict__ xout, long long *__restrict__ pout) {
  extern __shared__ unsigned long long kd_sm[];    // KD_LOCAL_SMEM bytes
  unsigned long long *key = kd_sm;                 // 2 KD_LOCAL slots
  unsigned int *tag = (unsigned int *)(key + 2 * KD_LOCAL);        // position in the node (padding: ~0)
  unsigned short *cur = (unsigned short *)(tag + 2 * KD_LOCAL), *nxt = cur + KD_LOCAL;
  const int t = threadIdx.x;
  const long long root = (1LL << L0) - 1 + blockIdx.x, base = lo[root];
  const int m = (int)(hi[root] - base);
  for (int i = t; i < m; i += KD_LT) cur[i] = (unsigned short)i;
  __syncthreads();
  for (int L = L0; L < levels; L++) {
    const int ax = L % dim;
    const long long first = ((root + 1) << (L - L0)) - 1;   // depth-L descendants of root: ids first .. first + nsub - 1
    const int nsub = 1 << (L - L0);
    int S = 1, sh = 0;                             // count-median: the first sub-node is the largest
    while (S < (int)(hi[first] - lo[first])) { S <<= 1; sh++; }
    const int V = nsub << sh;
    for (int v = t; v < V; v += KD_LT) {
      const int sb = v >> sh, li = v & (S - 1);
      const int p0 = (int)(lo[first + sb] - base), sz = (int)(hi[first + sb] - lo[first + sb]);
      if (li < sz) {
        unsigned long long b = __double_as_longlong(xin[(long long)ax * n + base + cur[p0 + li]]);
        b ^= (b >> 63) ? 0xffffffffffffffffULL : 0x8000000000000000ULL;
        key[v] = b; tag[v] = (unsigned)(p0 + li);
      } else { key[v] = ~0ULL; tag[v] = ~0u; }
    }
    __syncthreads();
    for (int k = 2; k <= S; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = t; i < V; i += KD_LT) {
          const int l = i ^ j;
          if (l > i) {
            const unsigned ta = tag[i], tb = tag[l];
            const unsigned long long ka = key[i], kb = key[l];
            const bool gt = ka != kb ? ka > kb : ta > tb;
            if (gt == (k == S || (i & k) == 0)) { key[i] = kb; key[l] = ka; tag[i] = tb; tag[l] = ta; }
          }
        }
        __syncthreads();
      }
    for (int v = t; v < V; v += KD_LT) {
      const int sb = v >> sh, li = v & (S - 1);
      const int p0 = (int)(lo[first + sb] - base), sz = (int)(hi[first + sb] - lo[first + sb]);
      if (li < sz) nxt[p0 + li] = cur[tag[v]];
    }
    __syncthreads();
    for (int i = t; i < m; i += KD_LT) cur[i] = nxt[i];
    __syncthreads();
  }
  for (int i = t; i < m; i += KD_LT) {
    const long long src = base + cur[i];
    for (int k = 0; k < dim; k++) xout[(long long)k * n + base + i] = xin[(long long)k * n + src];
    pout[base + i] = pin[src];
  }
}
__global__ void __launch_bounds__(STHREADS) k_hist_p(const unsigned long long *key, long long n, int shift, int ntiles,
                                                     unsigned int *cnt) {
  hist_body(key, n, shift, ntiles, cnt);
}
__global__ void __launch_bounds__(256) k_scan_p(unsigned int *cnt, int ntiles, unsigned int *tot) {
  scan_digit_body(cnt, ntiles, tot);
}
__global__ void __launch_bounds__(STHREADS) k_scatter_p(const unsigned long long *kin, const long long *iin, long long n,
                                                        int shift, int ntiles, const unsigned int *cnt,
                                                        const unsigned int *tot, unsigned long long *kout,
                                                        long long *iout) {
  scatter_body(kin, iin, n, shift, ntiles, cnt, tot, kout, iout);
}

}  // namespace

hodlr_status hodlr_kd_sort(hodlr_s *h, const double *x, long long n, int dim) {
  const int ntiles = (int)((n + TILE - 1) / TILE);
  if (ntiles > 256 * 16) return hodlr_set_error(HODLR_EINVAL, "sort: n too large for the radix tile table");
  unsigned long long *k[2] = {(unsigned long long *)hodlr_dalloc_tmp(h, sizeof(unsigned long long) * n),
                              (unsigned long long *)hodlr_dalloc_tmp(h, sizeof(unsigned long long) * n)};
  long long *id[2] = {(long long *)hodlr_dalloc_tmp(h, sizeof(long long) * n),
                      (long long *)hodlr_dalloc_tmp(h, sizeof(long long) * n)};
  unsigned int *cnt = (unsigned int *)hodlr_dalloc_tmp(h, sizeof(unsigned int) * (256 * (size_t)ntiles + 256));
  double *xs2 = (double *)hodlr_dalloc_tmp(h, sizeof(double) * (size_t)n * dim);
  long long *perm2 = (long long *)hodlr_dalloc_tmp(h, sizeof(long long) * n);
  if (!k[0] || !k[1] || !id[0] || !id[1] || !cnt || !xs2 || !perm2)
    return hodlr_set_error(HODLR_ENOMEM, "sort: device allocation failed");
  unsigned int *tot = cnt + 256 * (size_t)ntiles;
  const int nb = (int)((n + 255) / 256);
  double *xa[2] = {h->xs, xs2};
  long long *pa[2] = {h->perm, perm2};
  int cur = 0;                 // xa[cur], pa[cur]: the current order
  ph_begin(h, PH_SORT);
  k_kd_init<<<nb, 256, 0, h->st>>>(x, n, dim, h->xs, h->perm, h->dflags);
  HLAUNCH(h, "k_kd_init");
  const int levels = h->kappa > 0 ? h->kappa : 1;
  int L0 = 0;                  // first level whose nodes all fit one CTA's shared memory (count-median: sizes differ by <= 1)
  while (L0 < levels && (n + (1LL << L0) - 1) >> L0 > KD_LOCAL) L0++;
  for (int L = 0; L < L0; L++) {
    k_kd_keys<<<nb, 256, 0, h->st>>>(xa[cur] + (size_t)(L % dim) * n, n, k[0], id[0]);
    HLAUNCH(h, "k_kd_keys");
    int b = 0;                 // k[b], id[b]: the pass input
    auto pass = [&](int shift) -> hodlr_status {
      k_hist_p<<<ntiles, STHREADS, 0, h->st>>>(k[b], n, shift, ntiles, cnt);
      HLAUNCH(h, "k_hist_p");
      k_scan_p<<<256, 256, 0, h->st>>>(cnt, ntiles, tot);
      HLAUNCH(h, "k_scan_p");
      k_scatter_p<<<ntiles, STHREADS, 0, h->st>>>(k[b], id[b], n, shift, ntiles, cnt, tot, k[b ^ 1], id[b ^ 1]);
      HLAUNCH(h, "k_scatter_p");
      b ^= 1;
      return HODLR_OK;
    };
    for (int p = 0; p < 8; p++) { hodlr_status s = pass(8 * p); if (s != HODLR_OK) return s; }
    if (L > 0) {
      k_kd_nodekeys<<<nb, 256, 0, h->st>>>(id[b], n, h->lo, L, k[b]);
      HLAUNCH(h, "k_kd_nodekeys");
      for (int p = 0; p < (L + 7) / 8; p++) { hodlr_status s = pass(8 * p); if (s != HODLR_OK) return s; }
    }
    k_kd_gather<<<nb, 256, 0, h->st>>>(id[b], n, dim, xa[cur], pa[cur], xa[cur ^ 1], pa[cur ^ 1]);
    HLAUNCH(h, "k_kd_gather");
    cur ^= 1;
  }
  if (L0 < levels) {
    HCUDA(hodlr_allow_smem((const void *)k_kd_local, h->dev));
    k_kd_local<<<(int)(1LL << L0), KD_LT, KD_LOCAL_SMEM, h->st>>>(xa[cur], pa[cur], n, dim, L0, levels, h->lo, h->hi, xa[cur ^ 1],
                                                       pa[cur ^ 1]);
    HLAUNCH(h, "k_kd_local");
    cur ^= 1;
  }
  if (cur) {
    HCUDA(cudaMemcpyAsync(h->xs, xs2, sizeof(double) * (size_t)n * dim, cudaMemcpyDeviceToDevice, h->st));
    HCUDA(cudaMemcpyAsync(h->perm, perm2, sizeof(long long) * n, cudaMemcpyDeviceToDevice, h->st));
  }
  ph_end(h, PH_SORT);
  return HODLR_OK;
}

hodlr_status hodlr_sort_and_tree(hodlr_s *h, const double *x, long long n) {
  const int ntiles = (int)((n + TILE - 1) / TILE);
  unsigned long long *k0 = (unsigned long long *)hodlr_dalloc_tmp(h, sizeof(unsigned long long) * n);
  unsigned long long *k1 = (unsigned long long *)hodlr_dalloc_tmp(h, sizeof(unsigned long long) * n);
  long long *i0 = (long long *)hodlr_dalloc_tmp(h, sizeof(long long) * n);
  long long *i1 = (long long *)hodlr_dalloc_tmp(h, sizeof(long long) * n);
  unsigned int *cnt = (unsigned int *)hodlr_dalloc_tmp(h, sizeof(unsigned int) * (256 * (size_t)ntiles + 256));
  unsigned int *tot = cnt + 256 * (size_t)ntiles;
  if (ntiles > 256 * 16) return hodlr_set_error(HODLR_EINVAL, "sort: n too large for the radix tile table");
  if (!k0 || !k1 || !i0 || !i1 || !cnt) return hodlr_set_error(HODLR_ENOMEM, "sort: device allocation failed");
  int nb = (int)((n + 255) / 256);
  SortPlan *P = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_sort_mu);
    for (SortPlan *Q : g_sort_plans) if (!Q->busy && Q->n == n && Q->dev == h->dev) { P = Q; P->busy = true; break; }
  }
  if (!P) {
    P = new SortPlan(); P->n = n; P->dev = h->dev; P->busy = true;
    cudaError_t e = sort_graph(P, ntiles, nb);
    if (e != cudaSuccess) return hodlr_cuda_check(e, "sort graph");   // (plan leaked on error)
    std::lock_guard<std::mutex> lk(g_sort_mu);
    g_sort_plans.push_back(P);
  }
  struct Rel { SortPlan *p; ~Rel() { std::lock_guard<std::mutex> lk(g_sort_mu); p->busy = false; } } rel{P};
  SortCtx cx;
  cx.k0 = k0; cx.k1 = k1; cx.i0 = i0; cx.i1 = i1; cx.cnt = cnt; cx.tot = tot; cx.n = n; cx.ntiles = ntiles;
  cx.xs = h->xs; cx.perm = h->perm; cx.flags = h->dflags;
  ph_begin(h, PH_SORT);
  HCUDA(cudaMemsetAsync(h->dflags + 7, 0, sizeof(int), h->st));
  HCUDA(cudaMemcpyAsync(P->d_ctx, &cx, sizeof(cx), cudaMemcpyHostToDevice, h->st));
  k_make_keys<<<nb, 256, 0, h->st>>>(x, n, k0, i0, h->xs, h->perm, h->dflags);
  HLAUNCH(h, "k_make_keys");
  // radix passes only for an unsorted finite x, decided on the device (no host round trip); a non-finite x is
  // reported from the flags the build reads back at its end
  HCUDA(cudaGraphLaunch(P->ge, h->st));
  h->launches++; hodlr_global_launches++;      // (k_sort_cond; the passes only run for an unsorted x)
  ph_end(h, PH_SORT);
  return HODLR_OK;
}
