// api.cu -- the C-ABI of include/hodlr.h: validation, host plan, memory, phase orchestration.
#include "hodlr_internal.cuh"
#include <stdio.h>
#include <stdlib.h>
#include <stdarg.h>
#include <string.h>
#include <limits.h>
#include <new>
#include <mutex>
#include <vector>
#include <algorithm>

#include <chrono>
static thread_local char g_err[1024] = "";

int hodlr_trace_on() {
  static int on = -1;
  if (on < 0) { const char *ev = getenv("HODLR_TRACE"); on = ev && atoi(ev) ? 1 : 0; }
  return on;
}

void hodlr_trace(const char *what) {
  if (!hodlr_trace_on()) return;
  static auto t0 = std::chrono::steady_clock::now();
  static auto tl = t0;
  auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[hodlr %9.3f ms +%7.3f] %s\n", std::chrono::duration<double, std::milli>(now - t0).count(),
          std::chrono::duration<double, std::milli>(now - tl).count(), what);
  tl = now;
}
long long hodlr_global_launches = 0;

hodlr_status hodlr_set_error(hodlr_status code, const char *fmt, ...) {
  va_list ap; va_start(ap, fmt); vsnprintf(g_err, sizeof g_err, fmt, ap); va_end(ap);
  return code;
}

hodlr_status hodlr_cuda_check(cudaError_t e, const char *what) {
  if (e == cudaErrorMemoryAllocation) return hodlr_set_error(HODLR_ENOMEM, "%s: %s", what, cudaGetErrorString(e));
  return hodlr_set_error(HODLR_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Device blocks of freed handles are kept (per device, exact size) and handed to the next handle asking for the
// same size: a repeated build of one shape then makes no allocation or free calls (hodlr_free synchronizes the
// handle's streams before caching, so a reused block has no pending work).  Bounded at 16 GB per process (or
// HODLR_CACHE_MAX_MB); when an allocation fails the device's cached blocks are returned to the pool and the
// allocation is retried once; hodlr_cache_trim() empties the cache on request.
namespace {
struct CachedBlock { int dev; size_t bytes; void *p; };
std::mutex g_blk_mu;
std::vector<CachedBlock> g_blk_cache;
size_t g_blk_cached = 0;
size_t blk_cache_max() {
  static size_t mx = 0;
  if (!mx) { const char *ev = getenv("HODLR_CACHE_MAX_MB"); mx = ev ? (size_t)atoll(ev) << 20 : (size_t)16 << 30; }
  return mx;
}
// Free every cached block of `dev` (all devices if dev < 0); the caller holds g_blk_mu.
void blk_cache_drain_locked(int dev) {
  for (size_t i = g_blk_cache.size(); i-- > 0;) {
    if (dev >= 0 && g_blk_cache[i].dev != dev) continue;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g_blk_cache[i].dev) cudaSetDevice(g_blk_cache[i].dev);
    cudaFree(g_blk_cache[i].p);            // synchronous: the block has no pending work (see hodlr_free)
    if (cur >= 0 && cur != g_blk_cache[i].dev) cudaSetDevice(cur);
    g_blk_cached -= g_blk_cache[i].bytes;
    g_blk_cache.erase(g_blk_cache.begin() + (long)i);
  }
}
}

static void *dalloc_impl(hodlr_s *h, size_t bytes, bool transient) {
  void *p = nullptr;
  if (bytes == 0) bytes = 8;
  if (h->nallocs >= (int)(sizeof(h->allocs) / sizeof(h->allocs[0]))) return nullptr;
  {
    std::lock_guard<std::mutex> lk(g_blk_mu);
    for (size_t i = g_blk_cache.size(); i-- > 0;)
      if (g_blk_cache[i].dev == h->dev && g_blk_cache[i].bytes == bytes) {
        p = g_blk_cache[i].p; g_blk_cached -= bytes;
        g_blk_cache.erase(g_blk_cache.begin() + (long)i);
        break;
      }
  }
  if (!p) {
    char msg[96];
    snprintf(msg, sizeof msg, "dalloc: cache miss, cudaMallocAsync %.1f MB", bytes / 1048576.0);
    hodlr_trace(msg);
  }
  if (!p && cudaMallocAsync(&p, bytes, h->st) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
    hodlr_trace("dalloc: allocation failed: draining the cache and trimming the pool");
    {   // flush this device's idle cached blocks back to the driver and retry once
      std::lock_guard<std::mutex> lk(g_blk_mu);
      blk_cache_drain_locked(h->dev);
    }
    cudaStreamSynchronize(h->st);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    if (cudaMallocAsync(&p, bytes, h->st) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  }
  h->alloc_bytes[h->nallocs] = bytes;
  h->alloc_tmp[h->nallocs] = transient ? 1 : 0;
  h->allocs[h->nallocs++] = p;
  h->bytes += (long long)bytes;
  return p;
}

void *hodlr_dalloc(hodlr_s *h, size_t bytes) { return dalloc_impl(h, bytes, false); }

cudaError_t hodlr_allow_smem(const void *func, int dev) {
  int maxsm = 0;
  cudaError_t e = cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, func);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm - (int)fa.sharedSizeBytes);
}
void *hodlr_dalloc_tmp(hodlr_s *h, size_t bytes) { return dalloc_impl(h, bytes, true); }

// Hand the handle's transient blocks (radix-sort keys, ACA records / state) to the block cache.  Only called when
// the handle's streams are idle.
static void release_transient(hodlr_s *h) {
  std::lock_guard<std::mutex> lk(g_blk_mu);
  int w = 0;
  for (int i = 0; i < h->nallocs; i++) {
    if (!h->alloc_tmp[i]) {
      h->allocs[w] = h->allocs[i]; h->alloc_bytes[w] = h->alloc_bytes[i]; h->alloc_tmp[w] = 0; w++;
      continue;
    }
    h->bytes -= (long long)h->alloc_bytes[i];
    if (g_blk_cached + h->alloc_bytes[i] <= blk_cache_max()) {
      g_blk_cache.push_back({h->dev, h->alloc_bytes[i], h->allocs[i]});
      g_blk_cached += h->alloc_bytes[i];
    } else {
      cudaFreeAsync(h->allocs[i], h->st);
    }
  }
  h->nallocs = w;
  h->used = nullptr; h->ast = nullptr; h->d_forced = nullptr;     // (ACA state: transient)
}

static void setup_pool(int dev) {
  static int done_dev = -1;
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ULL;    // keep freed blocks in the pool: repeated builds reuse them
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

// sigma_i^2 = s2 + noise[perm[i]] in sorted order (heteroscedastic noise); flags[8] marks a negative / non-finite entry
__global__ void k_noise_gather(const double *__restrict__ noise, const long long *__restrict__ perm, long long n,
                               double s2, double *__restrict__ dn, int *flags) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = noise[perm[i]];
  if (!(v >= 0.0) || !isfinite(v)) atomicOr(&flags[8], 1);
  dn[i] = s2 + v;
}

static hodlr_status finish(hodlr_s *h, hodlr_status st, double *tsec) {
  cudaError_t e1 = cudaEventRecord(h->ev1, h->st);
  cudaError_t e2 = cudaStreamSynchronize(h->st);
  if (st != HODLR_OK) return st;
  if (e1 != cudaSuccess) return hodlr_cuda_check(e1, "event record");
  if (e2 != cudaSuccess) return hodlr_cuda_check(e2, "stream synchronize");
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, h->ev0, h->ev1) == cudaSuccess && tsec) *tsec = ms * 1e-3;
  for (int p = 0; p < PH_N; p++) {
    if (!h->ph_pending[p]) continue;
    float pm = 0.f;   // side-stream phases may still be running: keep them pending until they complete
    if (cudaEventElapsedTime(&pm, h->ph_ev[p][0], h->ph_ev[p][1]) == cudaSuccess) {
      h->ph_ms[p] += pm; h->ph_calls[p]++; h->ph_pending[p] = 0;
    } else {
      cudaGetLastError();
    }
  }
  return HODLR_OK;
}

extern "C" {

const char *hodlr_last_error(void) { return g_err; }

void hodlr_cache_trim(void) {
  std::lock_guard<std::mutex> lk(g_blk_mu);
  blk_cache_drain_locked(-1);
}
const char *hodlr_version(void) { return "hodlr_b200 0.1 sm_100a fp64"; }
int64_t hodlr_launch_count(void) { return hodlr_global_launches; }

// Streams and events are pooled per device across handles (creating and destroying them per handle costs
// more host time than a small factorization).
struct HRes {
  int dev;
  cudaStream_t st2, st3, sthi, st2b;
  cudaEvent_t ev_join2;
  cudaEvent_t ev0, ev1, ev_fork, ev_join, ev_chol, ev_hi;
  cudaEvent_t ph_ev[PH_N][2];
  void *pin;                 // pinned host staging for the handle's device-to-host reads (HODLR_PIN_BYTES)
};
static std::mutex g_res_mu;
static std::vector<HRes> g_res_pool;

static void res_acquire(hodlr_s *h) {
  HRes r;
  bool got = false;
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    for (size_t i = 0; i < g_res_pool.size(); i++)
      if (g_res_pool[i].dev == h->dev) { r = g_res_pool[i]; g_res_pool.erase(g_res_pool.begin() + i); got = true; break; }
  }
  if (!got) {
    r.dev = h->dev;
    cudaEventCreate(&r.ev0); cudaEventCreate(&r.ev1);
    cudaEventCreateWithFlags(&r.ev_fork, cudaEventDisableTiming); cudaEventCreateWithFlags(&r.ev_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&r.ev_chol, cudaEventDisableTiming);
    int lo_pri = 0, hi_pri = 0;
    cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
    // Stream priorities (measured): the step loop highest; the fused small-block ACA just below it (ahead
    // of the leaf Cholesky's CTAs, behind the passes: ACA phase 2.82 -> 2.43 ms); the leaf Cholesky lowest
    const int pf = std::min(lo_pri, hi_pri + 1), pc = lo_pri;
    cudaStreamCreateWithPriority(&r.st2, cudaStreamNonBlocking, pf);
    cudaStreamCreateWithPriority(&r.st2b, cudaStreamNonBlocking, pf);
    cudaEventCreateWithFlags(&r.ev_join2, cudaEventDisableTiming);
    cudaStreamCreateWithPriority(&r.st3, cudaStreamNonBlocking, pc);
    cudaStreamCreateWithPriority(&r.sthi, cudaStreamNonBlocking, hi_pri);
    cudaEventCreateWithFlags(&r.ev_hi, cudaEventDisableTiming);
    for (int p = 0; p < PH_N; p++) for (int j = 0; j < 2; j++) cudaEventCreate(&r.ph_ev[p][j]);
    if (cudaHostAlloc(&r.pin, HODLR_PIN_BYTES, cudaHostAllocDefault) != cudaSuccess) { cudaGetLastError(); r.pin = nullptr; }
  }
  h->st2b = r.st2b; h->ev_join2 = r.ev_join2;
  h->st2 = r.st2; h->st3 = r.st3; h->ev0 = r.ev0; h->ev1 = r.ev1; h->ev_fork = r.ev_fork; h->ev_join = r.ev_join;
  h->ev_chol = r.ev_chol; h->sthi = r.sthi; h->ev_hi = r.ev_hi;
  for (int p = 0; p < PH_N; p++) for (int j = 0; j < 2; j++) h->ph_ev[p][j] = r.ph_ev[p][j];
  h->pin = r.pin;
}

static void res_release(hodlr_s *h) {
  if (!h->st2) return;
  HRes r;
  r.st2b = h->st2b; r.ev_join2 = h->ev_join2;
  r.dev = h->dev; r.st2 = h->st2; r.st3 = h->st3; r.ev0 = h->ev0; r.ev1 = h->ev1; r.ev_fork = h->ev_fork;
  r.ev_join = h->ev_join; r.ev_chol = h->ev_chol; r.sthi = h->sthi; r.ev_hi = h->ev_hi;
  for (int p = 0; p < PH_N; p++) for (int j = 0; j < 2; j++) r.ph_ev[p][j] = h->ph_ev[p][j];
  r.pin = h->pin;
  std::lock_guard<std::mutex> lk(g_res_mu);
  g_res_pool.push_back(r);
}

void hodlr_free(hodlr_t h) {
  if (!h) return;
  if (h->st3) cudaStreamSynchronize(h->st3);
  if (h->st2) cudaStreamSynchronize(h->st2);
  if (h->st2b) cudaStreamSynchronize(h->st2b);
  if (h->sthi) cudaStreamSynchronize(h->sthi);
  cudaStreamSynchronize(h->st);
  {
    std::lock_guard<std::mutex> lk(g_blk_mu);
    for (int i = h->nallocs - 1; i >= 0; i--) {
      if (g_blk_cached + h->alloc_bytes[i] <= blk_cache_max()) {
        g_blk_cache.push_back({h->dev, h->alloc_bytes[i], h->allocs[i]});
        g_blk_cached += h->alloc_bytes[i];
      } else {
        cudaFreeAsync(h->allocs[i], h->st);
      }
    }
  }
  res_release(h);
  hodlr_dist_fini(h);
  delete[] h->h_lo; delete[] h->h_hi; delete[] h->h_rank;
  delete h;
}

// Validate one setting's parameters (theta = {a, ell[, alpha]})
static hodlr_status check_setting(hodlr_kernel kernel, const double *theta, double sigma2, int b) {
  if (!(sigma2 >= 0.0) || !isfinite(sigma2)) return hodlr_set_error(HODLR_EINVAL, "build: setting %d: sigma2 = %g", b, sigma2);
  if (!(theta[1] > 0.0) || !isfinite(theta[1])) return hodlr_set_error(HODLR_EINVAL, "build: setting %d: ell = %g <= 0", b, theta[1]);
  if (!(theta[0] >= 0.0) || !isfinite(theta[0])) return hodlr_set_error(HODLR_EINVAL, "build: setting %d: a = %g < 0", b, theta[0]);
  if (kernel == HODLR_RQ && (!(theta[2] > 0.0) || !isfinite(theta[2])))
    return hodlr_set_error(HODLR_EINVAL, "build: setting %d: rational quadratic alpha = %g <= 0", b, theta[2]);
  return HODLR_OK;
}

// Covariance parameters of one setting (Table I)
static KParams make_kp(hodlr_kernel kernel, const double *theta, double sigma2) {
  KParams kp;
  memset(&kp, 0, sizeof(kp));
  kp.kern = (int)kernel; kp.a2 = theta[0] * theta[0]; kp.s2 = sigma2;
  kp.c = kernel == HODLR_SE ? 1.0 / (2.0 * theta[1] * theta[1])
       : kernel == HODLR_MATERN32 ? sqrt(3.0) / theta[1]
       : kernel == HODLR_MATERN52 ? sqrt(5.0) / theta[1]
       : (kernel == HODLR_EXP || kernel == HODLR_BIHARM) ? 1.0 / theta[1] : 1.0 / (theta[1] * theta[1]);
  kp.alpha = kernel == HODLR_RQ ? theta[2] : 0.5;
  kp.ell = theta[1];
  kp.c2 = (2.0 * theta[1]) * theta[1];            // the oracle's 2.0 * ell * ell (left to right)
  kp.sq = kernel == HODLR_MATERN32 ? sqrt(3.0) : sqrt(5.0);
  int ex;   // exact reciprocals (powers of two) let kval_o multiply instead of divide, bit for bit the same
  kp.rc2 = frexp(kp.c2, &ex) == 0.5 ? 1.0 / kp.c2 : 0.0;
  kp.rell = frexp(theta[1], &ex) == 0.5 ? 1.0 / theta[1] : 0.0;
  kp.dn = nullptr;
  return kp;
}

// Problem s of a batched handle: sorted rows and permutation of problem 0 shifted by s * nseg
__global__ void k_replicate_order(double *xs, long long *perm, long long nseg, int B) {
  const long long N = nseg * B;
  for (long long i = nseg + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const long long s = i / nseg, j = i - s * nseg;
    xs[i] = xs[j];
    perm[i] = perm[j] + s * nseg;
  }
}

// hodlr_build (B = 1) and hodlr_build_batch (B = 2^t problems on the same points): one implementation.
static hodlr_status build_impl(const double *x, int64_t nseg, int32_t dim, int32_t B, hodlr_kernel kernel, const double *thetas,
                               int tstride, const double *sigma2s, int32_t leaf, double eps, const hodlr_dist *dist,
                               const hodlr_opts *opts, void *cuda_stream, hodlr_t *out) {
  if (!out) return hodlr_set_error(HODLR_EINVAL, "build: out is NULL");
  *out = nullptr;
  if (!x || !thetas || !sigma2s) return hodlr_set_error(HODLR_EINVAL, "build: NULL x or theta");
  if (nseg < 1) return hodlr_set_error(HODLR_EINVAL, "build: n = %lld < 1", (long long)nseg);
  if (leaf < 1) return hodlr_set_error(HODLR_EINVAL, "build: leaf = %d < 1", leaf);
  if (!(eps > 0.0 && eps < 1.0)) return hodlr_set_error(HODLR_EINVAL, "build: eps = %g not in (0, 1)", eps);
  if ((int)kernel < 0 || (int)kernel > 7) return hodlr_set_error(HODLR_EINVAL, "build: unknown kernel %d", (int)kernel);
  const bool nonspd = kernel == HODLR_MQ || kernel == HODLR_BIHARM;     // DESIGN.md R20
  if (nonspd && (B > 1 || (dist && dist->nranks > 1)))
    return hodlr_set_error(HODLR_EINVAL, "build: MQ / BIHARM (not positive definite) run on one GPU, unbatched");
  if (B < 1 || (B & (B - 1))) return hodlr_set_error(HODLR_EINVAL, "build_batch: B = %d is not a power of two", B);
  if (dim < 1 || dim > 64) return hodlr_set_error(HODLR_EINVAL, "build_nd: dim = %d not in [1, 64]", dim);
  if (dim > 1 && (B > 1 || (dist && dist->nranks > 1)))
    return hodlr_set_error(HODLR_EINVAL, "build_nd: d-dimensional points run on one GPU, unbatched (NEXT-3)");
  if (B > 1 && nseg < leaf) return hodlr_set_error(HODLR_EINVAL, "build_batch: n = %lld < leaf = %d", (long long)nseg, leaf);
  if (B > 1 && ((dist && dist->nranks > 1) || (opts && opts->noise)))
    return hodlr_set_error(HODLR_EINVAL, "build_batch: no dist or noise on batched handles");
  for (int b = 0; b < B; b++) {
    hodlr_status cs = check_setting(kernel, thetas + (size_t)b * tstride, sigma2s[b], b);
    if (cs != HODLR_OK) return cs;
  }
  const long long n = nseg * (long long)B;
  const double *theta = thetas;
  const double sigma2 = sigma2s[0];
  if (opts && opts->flags != 0) return hodlr_set_error(HODLR_EINVAL, "build: opts.flags must be 0");
  int cap = (opts && opts->rank_cap > 0) ? opts->rank_cap : 48;
  if (cap > ACA_MAXCAP) return hodlr_set_error(HODLR_EINVAL, "build: rank_cap %d > %d", cap, ACA_MAXCAP);
  hodlr_s *h = new (std::nothrow) hodlr_s();
  if (!h) return hodlr_set_error(HODLR_ENOMEM, "build: host allocation failed");
  memset((void *)h, 0, sizeof(*h));
  h->st = (cudaStream_t)cuda_stream;
  hodlr_status st = HODLR_OK;
  cudaError_t ce = cudaGetDevice(&h->dev);
  if (ce != cudaSuccess) { delete h; return hodlr_cuda_check(ce, "cudaGetDevice"); }
  setup_pool(h->dev);
  res_acquire(h);
  cudaEventRecord(h->ev0, h->st);
  h->launches = 0;
  h->n = n; h->leaf = leaf; h->eps = eps; h->cap = cap; h->theta[0] = theta[0]; h->theta[1] = theta[1];
  h->kp = make_kp(kernel, theta, sigma2);
  h->kp.dim = dim; h->kp.ldp = n;             // coordinate-major points (NEXT-3; 1-D: one row)
  h->dim = dim;
  h->nonspd = nonspd ? 1 : 0;
  h->nbatch = B; h->nseg = nseg;
  h->tbatch = 0;
  while ((1 << h->tbatch) < B) h->tbatch++;
  // O2-equivalent tree: kappa = largest integer with leaf * 2^kappa <= n
  int kappa = 0;
  while (((long long)leaf << (kappa + 1)) <= n && kappa < HODLR_MAXDEPTH - 2) kappa++;
  h->kappa = kappa;
  h->nnodes = (1LL << (kappa + 1)) - 1; h->ninternal = (1LL << kappa) - 1; h->nleaves = 1LL << kappa;
  h->h_lo = new long long[h->nnodes]; h->h_hi = new long long[h->nnodes];
  h->h_rank = new int[h->ninternal > 0 ? h->ninternal : 1]();
  h->h_lo[0] = 0; h->h_hi[0] = n;
  for (long long c = 0; c < h->ninternal; c++) {          // count-median split, left = ceil(m/2)
    long long m = h->h_hi[c] - h->h_lo[c], half = (m + 1) / 2;
    h->h_lo[2 * c + 1] = h->h_lo[c]; h->h_hi[2 * c + 1] = h->h_lo[c] + half;
    h->h_lo[2 * c + 2] = h->h_lo[c] + half; h->h_hi[2 * c + 2] = h->h_hi[c];
  }
  h->leaf_min = INT_MAX; h->leaf_max = 0;
  for (long long l = 0; l < h->nleaves; l++) {
    long long m = h->h_hi[h->ninternal + l] - h->h_lo[h->ninternal + l];
    if (m < h->leaf_min) h->leaf_min = (int)m;
    if (m > h->leaf_max) h->leaf_max = (int)m;
  }
  st = hodlr_dist_init(h, dist);                       // subtree sharding
  if (st != HODLR_OK) { hodlr_free(h); return st; }
  // panel slots: depth e holds min(cap, max node size at depth e) columns
  long long cols = 0;
  for (int e = 1; e <= kappa; e++) {
    long long mmax = 0;
    for (long long id = (1LL << e) - 1; id < (2LL << e) - 1; id++) mmax = std::max(mmax, h->h_hi[id] - h->h_lo[id]);
    h->dt.capd[e] = e <= h->tbatch ? 0 : (int)std::min<long long>(cap, mmax);   // (batched: top blocks are zero)
    h->dt.colbase[e] = cols;
    cols += h->dt.capd[e];
  }
  h->xh_cols = cols;
  h->xs = (double *)hodlr_dalloc(h, sizeof(double) * n * dim);
  h->perm = (long long *)hodlr_dalloc(h, sizeof(long long) * n);
  h->lo = (long long *)hodlr_dalloc(h, sizeof(long long) * h->nnodes);
  h->hi = (long long *)hodlr_dalloc(h, sizeof(long long) * h->nnodes);
  h->dflags = (int *)hodlr_dalloc(h, sizeof(int) * 16);
  h->d_dt = (DepthTab *)hodlr_dalloc(h, sizeof(DepthTab));
  h->ldx = ((n + 31) / 32) * 32 + 32;
  h->Xh = (double *)hodlr_dalloc(h, sizeof(double) * (size_t)h->ldx * (size_t)(cols > 0 ? cols : 1));
  if (!h->xs || !h->perm || !h->lo || !h->hi || !h->dflags || !h->d_dt || !h->Xh) {
    hodlr_free(h);
    return hodlr_set_error(HODLR_ENOMEM, "build: device allocation of %.2f GB failed",
                           1e-9 * (double)(8.0 * n * (cols + 4)));
  }
  if (h->nranks > 1) {          // row ranges of every rank's subtree (the solution allgather slices)
    h->d_rowlo = (long long *)hodlr_dalloc(h, sizeof(long long) * h->nranks);
    if (!h->d_rowlo) { hodlr_free(h); return hodlr_set_error(HODLR_ENOMEM, "build: device allocation failed"); }
    std::vector<long long> rl(h->nranks);
    h->rows_max = 0;
    for (int r = 0; r < h->nranks; r++) {
      const long long id = (1LL << h->tsplit) - 1 + r;
      rl[r] = h->h_lo[id];
      h->rows_max = std::max(h->rows_max, h->h_hi[id] - h->h_lo[id]);
    }
    if (cudaMemcpy(h->d_rowlo, rl.data(), sizeof(long long) * h->nranks, cudaMemcpyHostToDevice) != cudaSuccess) {
      hodlr_free(h); return hodlr_set_error(HODLR_ECUDA, "build: copy failed");
    }
  }
  int fl[16] = {0}; fl[2] = INT_MAX;
#define CK(call) do { cudaError_t _e = (call); if (_e != cudaSuccess) { st = hodlr_cuda_check(_e, #call); goto fail; } } while (0)
  CK(cudaMemcpyAsync(h->dflags, fl, sizeof(fl), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->lo, h->h_lo, sizeof(long long) * h->nnodes, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->hi, h->h_hi, sizeof(long long) * h->nnodes, cudaMemcpyHostToDevice, h->st));
  CK(cudaMemcpyAsync(h->d_dt, &h->dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));
  hodlr_trace("build: enter");
  st = dim > 1 ? hodlr_kd_sort(h, x, nseg, dim) : hodlr_sort_and_tree(h, x, nseg);
  hodlr_trace("build: sort issued");
  if (st != HODLR_OK) goto fail;
  if (B > 1) {     // batched: every problem has problem 0's order; per-problem parameters on the device
    k_replicate_order<<<592, 256, 0, h->st>>>(h->xs, h->perm, nseg, B);
    {
      cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) { st = hodlr_cuda_check(le, "launch k_replicate_order"); goto fail; }
    }
    h->launches++; hodlr_global_launches++;
    std::vector<KParams> kps(B);
    for (int b = 0; b < B; b++) {
      kps[b] = make_kp(kernel, thetas + (size_t)b * tstride, sigma2s[b]);
      kps[b].dim = 1; kps[b].ldp = n;
    }
    h->d_kps = (KParams *)hodlr_dalloc(h, sizeof(KParams) * B);
    if (!h->d_kps) { st = hodlr_set_error(HODLR_ENOMEM, "build: device allocation failed"); goto fail; }
    CK(cudaMemcpyAsync(h->d_kps, kps.data(), sizeof(KParams) * B, cudaMemcpyHostToDevice, h->st));
    CK(cudaStreamSynchronize(h->st));      // (kps is a host temporary)
  }
  if (opts && opts->noise) {     // heteroscedastic diagonal, carried with its point into sorted order
    h->d_noise = (double *)hodlr_dalloc(h, sizeof(double) * (size_t)n);
    if (!h->d_noise) { st = hodlr_set_error(HODLR_ENOMEM, "build: device allocation failed"); goto fail; }
    k_noise_gather<<<(int)((n + 255) / 256), 256, 0, h->st>>>(opts->noise, h->perm, n, sigma2, h->d_noise, h->dflags);
    {
      cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) { st = hodlr_cuda_check(le, "launch k_noise_gather"); goto fail; }
    }
    h->launches++; hodlr_global_launches++;
    h->kp.dn = h->d_noise;
  }
  // The leaf Cholesky factors (part of "Factor", Fig. 6 line 7) do not depend on the compression: they are
  // issued now on a side stream and overlap the ACA; hodlr_factor waits for them.
  st = hodlr_leaf_alloc(h);
  if (st != HODLR_OK) goto fail;
  if (opts && opts->forced_ranks && h->ninternal > 0) {    // parity test hook (hodlr.h)
    h->d_forced = (int *)hodlr_dalloc_tmp(h, sizeof(int) * (size_t)h->ninternal);
    if (!h->d_forced) { st = hodlr_set_error(HODLR_ENOMEM, "build: device allocation failed"); goto fail; }
    CK(cudaMemcpyAsync(h->d_forced, opts->forced_ranks, sizeof(int) * (size_t)h->ninternal, cudaMemcpyHostToDevice, h->st));
  }
  static int chol_after = -1;     // HODLR_CHOL_AFTER_ACA=1: run the leaf Cholesky after the ACA (experiments)
  if (chol_after < 0) { const char *ev = getenv("HODLR_CHOL_AFTER_ACA"); chol_after = ev && atoi(ev) ? 1 : 0; }
  if (h->nonspd) {
    h->chol_done = 0;              // LU leaves in hodlr_factor (factor.cu)
  } else if (!chol_after) {
    bool launched = false;
    CK(cudaEventRecord(h->ev_fork, h->st));
    CK(cudaStreamWaitEvent(h->st3, h->ev_fork, 0));
    ph_begin(h, PH_CHOL, h->st3);
    st = hodlr_leaf_chol_mma(h, h->st3, &launched);
    if (st != HODLR_OK) goto fail;
    ph_end(h, PH_CHOL, h->st3);
    CK(cudaEventRecord(h->ev_chol, h->st3));
    h->chol_done = launched ? 1 : 0;
  }
  hodlr_trace("build: chol launched");
  st = hodlr_aca(h);
  hodlr_trace("build: aca returned");
  if (st != HODLR_OK) goto fail;
  if (chol_after && !h->nonspd) {
    bool launched = false;
    ph_begin(h, PH_CHOL);
    st = hodlr_leaf_chol_mma(h, h->st, &launched);
    if (st != HODLR_OK) goto fail;
    ph_end(h, PH_CHOL);
    CK(cudaEventRecord(h->ev_chol, h->st));
    h->chol_done = launched ? 1 : 0;
  }
  {
    // one round trip: the flags and the per-block ranks through the pinned staging buffer (pageable
    // destinations would each block the host on their own)
    int *pf = (int *)h->pin;
    const bool pin_ranks = pf && sizeof(int) * (16 + (size_t)h->ninternal) <= HODLR_PIN_BYTES;
    if (pf) CK(cudaMemcpyAsync(pf, h->dflags, sizeof(int) * 16, cudaMemcpyDeviceToHost, h->st));
    if (h->ninternal > 0)
      CK(cudaMemcpyAsync(pin_ranks ? pf + 16 : h->h_rank, h->rank, sizeof(int) * h->ninternal, cudaMemcpyDeviceToHost, h->st));
    int fl16[16];
    if (!pf) CK(cudaMemcpyAsync(fl16, h->dflags, sizeof(fl16), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (pf) memcpy(fl16, pf, sizeof(fl16));
    if (pin_ranks && h->ninternal > 0) memcpy(h->h_rank, pf + 16, sizeof(int) * h->ninternal);
    int f5 = fl16[5], f8 = fl16[8];
    if (h->aca_steps < 0) {                             // the graph's step counter (hodlr_aca): 3 launches per step
      h->aca_steps = fl16[6];
      h->launches += 3 * fl16[6]; hodlr_global_launches += 3 * fl16[6];
    }
    if (fl16[0]) { st = hodlr_set_error(HODLR_EINVAL, "build: x contains NaN or Inf"); goto fail; }   // (k_make_keys)
    if (f8) { st = hodlr_set_error(HODLR_EINVAL, "build: noise contains a negative or non-finite entry"); goto fail; }
    // per-depth max ranks (the panel layout K_e must agree on every rank) and the rank-cap hits
    std::vector<double> loc(kappa + 2, 0.0);
    for (int e = 1; e <= kappa; e++) {
      int r = 0;
      for (long long b = (1LL << (e - 1)) - 1; b < (1LL << e) - 1; b++) r = std::max(r, h->h_rank[b]);
      loc[e] = r;
    }
    loc[0] = f5;
    if (h->nranks > 1) {
      const size_t per = kappa + 2;
      double *dbuf = (double *)hodlr_dalloc_tmp(h, sizeof(double) * per * (h->nranks + 1));
      if (!dbuf) { st = hodlr_set_error(HODLR_ENOMEM, "build: device allocation failed"); goto fail; }
      std::vector<double> all(per * h->nranks);
      CK(cudaMemcpyAsync(dbuf, loc.data(), sizeof(double) * per, cudaMemcpyHostToDevice, h->st));
      st = hodlr_allgather(h, dbuf, dbuf + per, sizeof(double) * per);
      if (st != HODLR_OK) goto fail;
      CK(cudaMemcpyAsync(all.data(), dbuf + per, sizeof(double) * per * h->nranks, cudaMemcpyDeviceToHost, h->st));
      CK(cudaStreamSynchronize(h->st));
      for (size_t j = 0; j < per; j++) {
        double v = 0.0;
        for (int r = 0; r < h->nranks; r++) v = j == 0 ? v + all[r * per] : std::max(v, all[r * per + j]);
        loc[j] = v;
      }
    }
    f5 = (int)loc[0];
    h->rank_cap_hits = f5;
    if (f5) { st = hodlr_set_error(HODLR_ERANKCAP, "build: %d block(s) reached the rank cap %d without meeting eps", f5, cap); goto fail; }
    h->dt.Kdim[0] = 0;
    for (int e = 1; e <= kappa; e++) {
      h->dt.rdep[e] = (int)loc[e];
      h->dt.Kdim[e] = h->dt.Kdim[e - 1] + h->dt.rdep[e];
    }
  }
  CK(cudaMemcpyAsync(h->d_dt, &h->dt, sizeof(DepthTab), cudaMemcpyHostToDevice, h->st));
  st = finish(h, HODLR_OK, &h->t_build);
  hodlr_trace("build: finished");
  if (st != HODLR_OK) goto fail;
  release_transient(h);        // h->st is idle here; the leaf Cholesky (st3) uses no transient block
  h->state = 1;
  *out = h;
  return HODLR_OK;
fail:
  cudaStreamSynchronize(h->st);
  hodlr_free(h);
  return st;
#undef CK
}

hodlr_status hodlr_build(const double *x, int64_t n, hodlr_kernel kernel, const double *theta, double sigma2,
                         int32_t leaf, double eps, const hodlr_dist *dist, const hodlr_opts *opts, void *cuda_stream,
                         hodlr_t *out) {
  return build_impl(x, n, 1, 1, kernel, theta, 0, &sigma2, leaf, eps, dist, opts, cuda_stream, out);
}

hodlr_status hodlr_build_nd(const double *x, int64_t n, int32_t dim, hodlr_kernel kernel, const double *theta,
                            double sigma2, int32_t leaf, double eps, const hodlr_opts *opts, void *cuda_stream,
                            hodlr_t *out) {
  return build_impl(x, n, dim, 1, kernel, theta, 0, &sigma2, leaf, eps, nullptr, opts, cuda_stream, out);
}

hodlr_status hodlr_build_batch(const double *x, int64_t n, hodlr_kernel kernel, const double *thetas,
                               const double *sigma2s, int32_t B, int32_t leaf, double eps, const hodlr_opts *opts,
                               void *cuda_stream, hodlr_t *out) {
  return build_impl(x, n, 1, B, kernel, thetas, kernel == HODLR_RQ ? 3 : 2, sigma2s, leaf, eps, nullptr, opts,
                    cuda_stream, out);
}

hodlr_status hodlr_batch_results(hodlr_t h, double *logdet_host, double *quad_host) {
  if (!h || !logdet_host) return hodlr_set_error(HODLR_EINVAL, "batch_results: NULL argument");
  if (h->state == -1) return hodlr_set_error(HODLR_ENOTPD, "batch_results: factorization failed");
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "batch_results: not factored");
  if (quad_host && !h->aug) return hodlr_set_error(HODLR_ESTATE, "batch_results: no right-hand side was fused (hodlr_factor_solve)");
  if (h->nranks > 1) return hodlr_set_error(HODLR_EINVAL, "batch_results: sharded handle");
  const int B = h->nbatch;
  double *d = (double *)hodlr_dalloc_tmp(h, sizeof(double) * 2 * B);
  if (!d) return hodlr_set_error(HODLR_ENOMEM, "batch_results: device allocation failed");
  hodlr_status st = hodlr_batch_parts(h, d);
  std::vector<double> v(2 * (size_t)B);
  cudaError_t e = cudaSuccess;
  if (st == HODLR_OK) e = cudaMemcpyAsync(v.data(), d, sizeof(double) * 2 * B, cudaMemcpyDeviceToHost, h->st);
  if (st == HODLR_OK && e == cudaSuccess) e = cudaStreamSynchronize(h->st);
  release_transient(h);
  if (st != HODLR_OK) return st;
  if (e != cudaSuccess) return hodlr_cuda_check(e, "batch_results");
  for (int b = 0; b < B; b++) {
    logdet_host[b] = v[b];
    if (quad_host) quad_host[b] = v[B + b];
  }
  return HODLR_OK;
}

hodlr_status hodlr_factor(hodlr_t h) {
  if (!h) return hodlr_set_error(HODLR_EINVAL, "factor: NULL handle");
  if (h->state != 1) return hodlr_set_error(HODLR_ESTATE, "factor: handle is not in the built state");
  h->aug = 0; h->y_aug = nullptr;
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  hodlr_trace("factor: enter");
  hodlr_status st = hodlr_factor_impl(h);
  hodlr_trace("factor: launched");
  st = finish(h, st, &h->t_factor);
  hodlr_trace("factor: finished");
  if (st != HODLR_OK) { h->state = -1; h->logdet = -INFINITY; return st; }
  int f[11];
  cudaError_t e = cudaMemcpy(f, h->dflags, sizeof(f), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return hodlr_cuda_check(e, "factor flags");
  h->det_sign = (f[10] & 1) ? -1 : 1;
  if (f[1]) {
    h->state = -1; h->logdet = -INFINITY;
    return hodlr_set_error(HODLR_ENOTPD, "factor: node %d is not positive definite (%d failures)", f[2], f[1]);
  }
  e = cudaMemcpy(&h->logdet, h->d_logdet, sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return hodlr_cuda_check(e, "factor logdet");
  h->state = 2;
  return HODLR_OK;
}

hodlr_status hodlr_factor_solve(hodlr_t h, const double *y, double *x, double *quad_host) {
  if (!h || !y) return hodlr_set_error(HODLR_EINVAL, "factor_solve: NULL argument");
  if (h->state != 1) return hodlr_set_error(HODLR_ESTATE, "factor_solve: handle is not in the built state");
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  if (x) {                                   // device or page-locked host memory (written by the solve kernel)
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, x) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered || !pa.devicePointer) {
      cudaGetLastError();
      return hodlr_set_error(HODLR_EINVAL, "factor_solve: x is neither device nor page-locked host memory");
    }
    x = (double *)pa.devicePointer;
  }
  h->aug = 1; h->y_aug = y;                  // y is column 0 of every leaf panel (leaf_mma.cu, factor.cu)
  hodlr_status st = HODLR_OK;
  cudaError_t ce = cudaMemsetAsync(h->dflags + 3, 0, sizeof(int), h->st);
  if (ce != cudaSuccess) st = hodlr_cuda_check(ce, "factor_solve flags");
  if (st == HODLR_OK) st = hodlr_factor_impl(h);
  if (st == HODLR_OK && x) st = hodlr_solve_impl(h, y, x, 1, h->n, false, true);   // down passes only
  int f[11] = {0};
  double quad = 0.0;
  // results through the pinned staging buffer: [0, 2) log det, y^T C^{-1} y; then the flags (one round trip)
  double *pd = (double *)h->pin;
  if (st == HODLR_OK) {
    if (pd) {
      ce = cudaMemcpyAsync(pd, h->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, h->st);
      // Pi at the root with the fused right-hand side is the 1 x 1 matrix y^T C^{-1} y
      if (ce == cudaSuccess) ce = cudaMemcpyAsync(pd + 1, h->Pipool + h->dt.piOff[0], sizeof(double), cudaMemcpyDeviceToHost, h->st);
      if (ce == cudaSuccess) ce = cudaMemcpyAsync(pd + 2, h->dflags, sizeof(f), cudaMemcpyDeviceToHost, h->st);
    } else {
      ce = cudaMemcpyAsync(f, h->dflags, sizeof(f), cudaMemcpyDeviceToHost, h->st);
      if (ce == cudaSuccess) ce = cudaMemcpyAsync(&h->logdet, h->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, h->st);
      if (ce == cudaSuccess) ce = cudaMemcpyAsync(&quad, h->Pipool + h->dt.piOff[0], sizeof(double), cudaMemcpyDeviceToHost, h->st);
    }
    if (ce != cudaSuccess) st = hodlr_cuda_check(ce, "factor_solve results");
  }
  st = finish(h, st, &h->t_factor);
  if (st == HODLR_OK && pd) { h->logdet = pd[0]; quad = pd[1]; memcpy(f, pd + 2, sizeof(f)); }
  h->y_aug = nullptr;
  if (st != HODLR_OK) { h->state = -1; h->logdet = -INFINITY; return st; }
  if (f[1]) {
    h->state = -1; h->logdet = -INFINITY;
    if (quad_host) *quad_host = NAN;
    return hodlr_set_error(HODLR_ENOTPD, "factor_solve: node %d is not positive definite (%d failures)", f[2], f[1]);
  }
  h->det_sign = (f[10] & 1) ? -1 : 1;
  h->state = 2;                              // factored: logdet / solve / gp_loglik for other right-hand sides work
  if (f[3]) {
    int z = 0;
    cudaMemcpy(h->dflags + 3, &z, sizeof(int), cudaMemcpyHostToDevice);
    return hodlr_set_error(HODLR_EINVAL, "factor_solve: y contains NaN or Inf (the factorization itself is valid)");
  }
  if (quad_host) *quad_host = quad;
  return HODLR_OK;
}

hodlr_status hodlr_logdet(hodlr_t h, double *logdet_host) {
  if (!h || !logdet_host) return hodlr_set_error(HODLR_EINVAL, "logdet: NULL argument");
  if (h->state == -1) { *logdet_host = -INFINITY; return hodlr_set_error(HODLR_ENOTPD, "logdet: factorization failed"); }
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "logdet: not factored");
  *logdet_host = h->logdet;
  h->t_logdet = 0.0;
  return HODLR_OK;
}

hodlr_status hodlr_logdet_sign(hodlr_t h, double *logabs_host, int32_t *sign_host) {
  if (!h || !logabs_host || !sign_host) return hodlr_set_error(HODLR_EINVAL, "logdet_sign: NULL argument");
  if (h->state == -1) {
    *logabs_host = -INFINITY; *sign_host = 0;
    return hodlr_set_error(HODLR_ENOTPD, "logdet_sign: factorization failed");
  }
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "logdet_sign: not factored");
  *logabs_host = h->logdet; *sign_host = h->det_sign;
  return HODLR_OK;
}

static hodlr_status check_y_flag(hodlr_t h) {
  int f3 = 0;
  cudaError_t e = cudaMemcpy(&f3, h->dflags + 3, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return hodlr_cuda_check(e, "solve flags");
  if (f3) {
    int z = 0;
    cudaMemcpy(h->dflags + 3, &z, sizeof(int), cudaMemcpyHostToDevice);
    return hodlr_set_error(HODLR_EINVAL, "y contains NaN or Inf");
  }
  return HODLR_OK;
}

hodlr_status hodlr_apply(hodlr_t h, const double *x, double *y, int64_t nrhs, int64_t ld) {
  if (!h || !x || !y) return hodlr_set_error(HODLR_EINVAL, "apply: NULL argument");
  if (h->state == 0) return hodlr_set_error(HODLR_ESTATE, "apply: not built");
  if (nrhs < 1 || ld < h->n) return hodlr_set_error(HODLR_EINVAL, "apply: nrhs = %lld, ld = %lld", (long long)nrhs, (long long)ld);
  if (h->nranks > 1) return hodlr_set_error(HODLR_EINVAL, "apply: sharded handles are not supported (each rank holds its subtree's factors only)");
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  hodlr_status st = HODLR_OK;
  for (int64_t j = 0; j < nrhs && st == HODLR_OK; j++) st = hodlr_apply_impl(h, x + j * ld, y + j * ld);
  return finish(h, st, nullptr);
}

hodlr_status gp_predict(hodlr_t h, const double *y, const double *xt, int64_t m, double *mean, double *var) {
  if (!h || !y || m < 0 || (m > 0 && (!xt || !mean))) return hodlr_set_error(HODLR_EINVAL, "predict: NULL argument or m < 0");
  if (h->state == -1) return hodlr_set_error(HODLR_ENOTPD, "predict: factorization failed");
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "predict: not factored");
  if (h->nranks > 1) return hodlr_set_error(HODLR_EINVAL, "predict: sharded handles are not supported");
  if (h->nonspd && var) return hodlr_set_error(HODLR_EINVAL, "predict: no variance for a kernel that is not positive definite");
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  hodlr_status st = hodlr_predict_impl(h, y, xt, m, mean, var);
  st = finish(h, st, nullptr);
  if (st != HODLR_OK) return st;
  return check_y_flag(h);
}

hodlr_status hodlr_solve(hodlr_t h, const double *y, double *x, int64_t nrhs, int64_t ld) {
  if (!h || !y || !x) return hodlr_set_error(HODLR_EINVAL, "solve: NULL argument");
  if (h->state == -1) return hodlr_set_error(HODLR_ENOTPD, "solve: factorization failed");
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "solve: not factored");
  if (nrhs < 1 || ld < h->n) return hodlr_set_error(HODLR_EINVAL, "solve: nrhs = %lld, ld = %lld", (long long)nrhs, (long long)ld);
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  hodlr_status st = HODLR_OK;
  st = hodlr_solve_impl(h, y, x, nrhs, ld, false);       // up to SOLVE_RMAX columns per launch
  st = finish(h, st, &h->t_solve);
  if (st != HODLR_OK) return st;
  return check_y_flag(h);
}

hodlr_status gp_loglik(hodlr_t h, const double *y, double *out_host) {
  if (!h || !y || !out_host) return hodlr_set_error(HODLR_EINVAL, "gp_loglik: NULL argument");
  if (h->state == -1) { *out_host = -INFINITY; return hodlr_set_error(HODLR_ENOTPD, "gp_loglik: factorization failed"); }
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "gp_loglik: not factored");
  if (h->nonspd) return hodlr_set_error(HODLR_EINVAL, "gp_loglik: the kernel is not positive definite (not a covariance)");
  h->launches = 0;
  cudaEventRecord(h->ev0, h->st);
  hodlr_status st = hodlr_solve_impl(h, y, nullptr, 1, h->n, true);
  double yCy = 0.0;
  if (st == HODLR_OK) {   // h at the root = y^T C^{-1} y
    double hh[2] = {0.0, 0.0};
    cudaError_t e = cudaMemcpyAsync(hh, h->hvec, sizeof(hh), cudaMemcpyDeviceToHost, h->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
    yCy = hh[0] + hh[1];
    if (e != cudaSuccess) st = hodlr_cuda_check(e, "gp_loglik copy");
  }
  double tdummy = 0;
  st = finish(h, st, &tdummy);
  if (st != HODLR_OK) return st;
  st = check_y_flag(h);
  if (st != HODLR_OK) return st;
  // -1/2 y^T C^{-1} y - 1/2 log det C - (n/2) log(2 pi)   (eq. 1)
  *out_host = -0.5 * yCy - 0.5 * h->logdet - 0.5 * (double)h->n * log(2.0 * M_PI);
  return HODLR_OK;
}

hodlr_status hodlr_info(hodlr_t h, hodlr_info_t *info) {
  if (!h || !info) return hodlr_set_error(HODLR_EINVAL, "info: NULL argument");
  memset(info, 0, sizeof(*info));
  info->kappa = h->kappa; info->leaf_min = h->leaf_min; info->leaf_max = h->leaf_max;
  info->K = h->dt.Kdim[h->kappa];
  for (int e = 1; e <= h->kappa && e < 64; e++) {
    info->max_rank_by_depth[e] = h->dt.rdep[e];
    double s = 0; long long c = 0;
    for (long long b = (1LL << (e - 1)) - 1; b < (1LL << e) - 1; b++)
      if (hodlr_owns_block(h, b)) { s += h->h_rank[b]; c++; }
    info->mean_rank_by_depth[e] = c ? s / c : 0.0;
  }
  info->factor_bytes = h->bytes;
  info->t_build = h->t_build; info->t_factor = h->t_factor; info->t_logdet = h->t_logdet; info->t_solve = h->t_solve;
  info->rank_cap_hits = h->rank_cap_hits;
  info->aca_steps = h->aca_steps;
  info->rank = h->grank; info->nranks = h->nranks; info->split_depth = h->tsplit;
  info->gpu_launches_last = h->launches;
  for (int p = 0; p < PH_N && p < 16; p++) { info->kernel_ms[p] = h->ph_ms[p]; info->kernel_calls[p] = h->ph_calls[p]; }
  return HODLR_OK;
}

hodlr_status hodlr_get_order(hodlr_t h, double *xs_dev, int64_t *perm_dev) {
  if (!h) return hodlr_set_error(HODLR_EINVAL, "get_order: NULL handle");
  if (xs_dev) { cudaError_t e = cudaMemcpyAsync(xs_dev, h->xs, sizeof(double) * h->n * h->dim, cudaMemcpyDeviceToDevice, h->st); if (e) return hodlr_cuda_check(e, "get_order"); }
  if (perm_dev) { cudaError_t e = cudaMemcpyAsync(perm_dev, h->perm, sizeof(long long) * h->n, cudaMemcpyDeviceToDevice, h->st); if (e) return hodlr_cuda_check(e, "get_order"); }
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? HODLR_OK : hodlr_cuda_check(e, "get_order");
}

hodlr_status hodlr_get_tree(hodlr_t h, int64_t *lo_host, int64_t *hi_host, int32_t *ranks_host) {
  if (!h) return hodlr_set_error(HODLR_EINVAL, "get_tree: NULL handle");
  if (lo_host) memcpy(lo_host, h->h_lo, sizeof(long long) * h->nnodes);
  if (hi_host) memcpy(hi_host, h->h_hi, sizeof(long long) * h->nnodes);
  if (ranks_host && h->ninternal) memcpy(ranks_host, h->h_rank, sizeof(int) * h->ninternal);
  return HODLR_OK;
}

hodlr_status hodlr_get_logdet_parts(hodlr_t h, double *leaf_parts_host, double *node_parts_host) {
  if (!h) return hodlr_set_error(HODLR_EINVAL, "get_logdet_parts: NULL handle");
  if (h->state != 2) return hodlr_set_error(HODLR_ESTATE, "get_logdet_parts: not factored");
  cudaError_t e = cudaSuccess;
  if (leaf_parts_host) e = cudaMemcpy(leaf_parts_host, h->leaf_ld, sizeof(double) * h->nleaves, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && node_parts_host && h->ninternal)
    e = cudaMemcpy(node_parts_host, h->node_ld, sizeof(double) * h->ninternal, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? HODLR_OK : hodlr_cuda_check(e, "get_logdet_parts");
}

}  // extern "C"
