// dist.cu -- multi-GPU subtree sharding support (north_star): the shard plan and the
// allgather transport used at the exchange points of build, factor and solve.
//
// Transport: NCCL (loaded with dlopen at run time, one GPU per rank, ncclAllGather on the handle's stream),
// or an in-process group of virtual ranks (host threads sharing one device: barrier + device-to-device
// copies), which runs the sharded path on a single GPU.
#include "hodlr_internal.cuh"
#include <dlfcn.h>
#include <string.h>
#include <mutex>
#include <condition_variable>
#include <chrono>
#include <stdlib.h>
#include <vector>

// ---------------------------------------------------------------------------------------------
// NCCL through dlopen (no link-time dependency; reuses the process's libnccl.so.2 when torch loaded it)
// ---------------------------------------------------------------------------------------------
typedef int ncclResult_t_;
typedef struct { char internal[128]; } ncclUniqueId_;
struct NcclApi {
  bool ok = false;
  ncclResult_t_ (*getUniqueId)(ncclUniqueId_ *);
  ncclResult_t_ (*commInitRank)(void **, int, ncclUniqueId_, int);
  ncclResult_t_ (*allGather)(const void *, void *, size_t, int, void *, cudaStream_t);
  ncclResult_t_ (*commDestroy)(void *);
  const char *(*getErrorString)(ncclResult_t_);
};
static NcclApi g_nccl;
static std::mutex g_nccl_mu;
struct CommEntry { char id[128]; int rank, nranks, dev; void *comm; };
static std::vector<CommEntry> g_comms;

static std::mutex g_load_mu;
static bool nccl_load() {
  std::lock_guard<std::mutex> lk(g_load_mu);
  if (g_nccl.ok) return true;
  void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return false;
  g_nccl.getUniqueId = (ncclResult_t_(*)(ncclUniqueId_ *))dlsym(lib, "ncclGetUniqueId");
  g_nccl.commInitRank = (ncclResult_t_(*)(void **, int, ncclUniqueId_, int))dlsym(lib, "ncclCommInitRank");
  g_nccl.allGather = (ncclResult_t_(*)(const void *, void *, size_t, int, void *, cudaStream_t))dlsym(lib, "ncclAllGather");
  g_nccl.commDestroy = (ncclResult_t_(*)(void *))dlsym(lib, "ncclCommDestroy");
  g_nccl.getErrorString = (const char *(*)(ncclResult_t_))dlsym(lib, "ncclGetErrorString");
  g_nccl.ok = g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.allGather && g_nccl.commDestroy && g_nccl.getErrorString;
  return g_nccl.ok;
}
static const int NCCL_FLOAT64 = 8;    // ncclDouble / ncclFloat64 in nccl.h

// ---------------------------------------------------------------------------------------------
// In-process group: every virtual rank posts its send/recv pointers, waits for the others, copies all send
// buffers into its own receive buffer (device-to-device, its own stream), and waits again so that no send
// buffer is reused before every rank has copied it.
// ---------------------------------------------------------------------------------------------
struct HodlrGroup {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  const void *send[256];
  // scaling projection (hodlr_group_mode): 1 = record every gathered buffer (rank 0's view, device copies);
  // 2 = solo replay: only rank 0 runs, each exchange copies the recorded buffer and overwrites rank 0's slot with
  // its live send (the other ranks' parts are what they computed in the recorded run: same inputs, deterministic
  // kernels), so rank 0's critical path is timed without the other ranks' work on the same GPU
  int mode = 0;
  size_t replay_next = 0;
  std::vector<void *> rec;
  std::vector<size_t> rec_bytes;
};

// Returns false when the other ranks do not arrive within HODLR_GROUP_TIMEOUT_S seconds (default 300): a rank that
// failed before an exchange then makes the waiting ranks fail instead of blocking forever.
static bool group_barrier(HodlrGroup *g) {
  static int tmo = -1;
  if (tmo < 0) { const char *ev = getenv("HODLR_GROUP_TIMEOUT_S"); tmo = ev ? atoi(ev) : 300; }
  std::unique_lock<std::mutex> lk(g->mu);
  const long long my = g->gen;
  if (++g->arrived == g->n) { g->arrived = 0; g->gen++; g->cv.notify_all(); return true; }
  if (g->cv.wait_for(lk, std::chrono::seconds(tmo), [&] { return g->gen != my; })) return true;
  g->arrived--;                              // withdraw: this rank gives up on the exchange
  return false;
}

hodlr_status hodlr_allgather(hodlr_s *h, const void *send, void *recv, size_t bytes) {
  if (h->nranks <= 1) {
    if (send != recv) HCUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, h->st));
    return HODLR_OK;
  }
  hodlr_trace("allgather");
  if (h->comm) {
    const int r = g_nccl.allGather(send, recv, bytes / 8, NCCL_FLOAT64, h->comm, h->st);
    if (r != 0) return hodlr_set_error(HODLR_ENCCL, "ncclAllGather: %s", g_nccl.getErrorString(r));
    return HODLR_OK;
  }
  HodlrGroup *g = (HodlrGroup *)h->group;
  if (g->mode == 2) {                       // solo replay (rank 0 only)
    if (g->replay_next >= g->rec.size() || g->rec_bytes[g->replay_next] != bytes * g->n)
      return hodlr_set_error(HODLR_EINVAL, "group replay: exchange %zu does not match the recorded run", g->replay_next);
    HCUDA(cudaMemcpyAsync(recv, g->rec[g->replay_next++], bytes * g->n, cudaMemcpyDeviceToDevice, h->st));
    HCUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, h->st));
    return HODLR_OK;
  }
  HCUDA(cudaStreamSynchronize(h->st));
  { std::lock_guard<std::mutex> lk(g->mu); g->send[h->grank] = send; }
  if (!group_barrier(g)) return hodlr_set_error(HODLR_ECUDA, "group exchange: the other ranks did not arrive (failed?)");
  for (int j = 0; j < g->n; j++)
    HCUDA(cudaMemcpyAsync((char *)recv + (size_t)j * bytes, g->send[j], bytes, cudaMemcpyDeviceToDevice, h->st));
  if (g->mode == 1 && h->grank == 0) {      // record rank 0's gathered buffer
    void *p = nullptr;
    HCUDA(cudaMalloc(&p, bytes * g->n));
    HCUDA(cudaMemcpyAsync(p, recv, bytes * g->n, cudaMemcpyDeviceToDevice, h->st));
    std::lock_guard<std::mutex> lk(g->mu);
    g->rec.push_back(p); g->rec_bytes.push_back(bytes * g->n);
  }
  HCUDA(cudaStreamSynchronize(h->st));
  if (!group_barrier(g)) return hodlr_set_error(HODLR_ECUDA, "group exchange: the other ranks did not arrive (failed?)");
  return HODLR_OK;
}

hodlr_status hodlr_dist_init(hodlr_s *h, const hodlr_dist *d) {
  h->grank = 0; h->nranks = 1; h->tsplit = 0; h->comm = nullptr; h->group = nullptr;
  if (!d || d->nranks <= 1) return HODLR_OK;
  const int P = d->nranks;
  if ((P & (P - 1)) != 0 || P > 256) return hodlr_set_error(HODLR_EINVAL, "dist: nranks = %d is not a power of two <= 256", P);
  if (d->rank < 0 || d->rank >= P) return hodlr_set_error(HODLR_EINVAL, "dist: rank %d not in [0, %d)", d->rank, P);
  if ((d->nccl_unique_id != nullptr) == (d->group != nullptr))
    return hodlr_set_error(HODLR_EINVAL, "dist: exactly one of nccl_unique_id and group must be set");
  int t = 0;
  while ((1 << t) < P) t++;
  if (t > h->kappa) return hodlr_set_error(HODLR_EINVAL, "dist: %d ranks need kappa >= %d (kappa = %d)", P, t, h->kappa);
  h->grank = d->rank; h->nranks = P; h->tsplit = t;
  if (d->group) {
    if (((HodlrGroup *)d->group)->n != P) return hodlr_set_error(HODLR_EINVAL, "dist: group size differs from nranks");
    h->group = d->group;
    return HODLR_OK;
  }
  if (!nccl_load()) return hodlr_set_error(HODLR_ENCCL, "dist: libnccl.so.2 could not be loaded");
  // communicators are cached per (unique id, rank, device) for the life of the process: repeated builds with
  // the same id reuse theirs (ncclCommInitRank costs far more than a factorization)
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  for (const CommEntry &ce : g_comms)
    if (ce.rank == d->rank && ce.nranks == P && ce.dev == h->dev && memcmp(ce.id, d->nccl_unique_id, 128) == 0) {
      h->comm = ce.comm;
      return HODLR_OK;
    }
  ncclUniqueId_ id;
  memcpy(&id, d->nccl_unique_id, sizeof(id));
  void *comm = nullptr;
  const int r = g_nccl.commInitRank(&comm, P, id, d->rank);
  if (r != 0) return hodlr_set_error(HODLR_ENCCL, "ncclCommInitRank: %s", g_nccl.getErrorString(r));
  CommEntry ce;
  memcpy(ce.id, d->nccl_unique_id, 128); ce.rank = d->rank; ce.nranks = P; ce.dev = h->dev; ce.comm = comm;
  g_comms.push_back(ce);
  h->comm = comm;
  return HODLR_OK;
}

void hodlr_dist_fini(hodlr_s *h) { h->comm = nullptr; }   // communicators stay cached (see hodlr_dist_init)

extern "C" {

hodlr_status hodlr_nccl_unique_id(void *out128) {
  if (!out128) return hodlr_set_error(HODLR_EINVAL, "nccl_unique_id: NULL");
  if (!nccl_load()) return hodlr_set_error(HODLR_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId_ id;
  const int r = g_nccl.getUniqueId(&id);
  if (r != 0) return hodlr_set_error(HODLR_ENCCL, "ncclGetUniqueId: %s", g_nccl.getErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return HODLR_OK;
}

hodlr_status hodlr_group_create(int32_t nranks, void **group) {
  if (!group || nranks < 1 || nranks > 256) return hodlr_set_error(HODLR_EINVAL, "group_create: bad arguments");
  HodlrGroup *g = new HodlrGroup();
  g->n = nranks;
  *group = g;
  return HODLR_OK;
}

void hodlr_group_destroy(void *group) {
  HodlrGroup *g = (HodlrGroup *)group;
  if (!g) return;
  for (void *p : g->rec) cudaFree(p);
  delete g;
}

hodlr_status hodlr_group_mode(void *group, int32_t mode) {
  HodlrGroup *g = (HodlrGroup *)group;
  if (!g || mode < 0 || mode > 2) return hodlr_set_error(HODLR_EINVAL, "group_mode: bad arguments");
  if (mode == 2 && g->rec.empty()) return hodlr_set_error(HODLR_ESTATE, "group_mode: nothing recorded");
  if (mode == 1) { for (void *p : g->rec) cudaFree(p); g->rec.clear(); g->rec_bytes.clear(); }
  g->mode = mode; g->replay_next = 0;
  return HODLR_OK;
}

hodlr_status hodlr_dist_plan(int64_t n, int32_t leaf, int32_t rank, int32_t nranks, int32_t *kappa, int32_t *t,
                             int64_t *row_lo, int64_t *row_hi, int64_t *leaf_lo, int64_t *leaf_hi) {
  if (n < 1 || leaf < 1 || nranks < 1 || rank < 0 || rank >= nranks || (nranks & (nranks - 1)) != 0)
    return hodlr_set_error(HODLR_EINVAL, "dist_plan: bad arguments");
  int k = 0;
  while (((long long)leaf << (k + 1)) <= n && k < HODLR_MAXDEPTH - 2) k++;
  int tt = 0;
  while ((1 << tt) < nranks) tt++;
  if (tt > k) return hodlr_set_error(HODLR_EINVAL, "dist_plan: %d ranks need kappa >= %d", nranks, tt);
  // walk the count-median splits (left = ceil(m / 2)) from the root to the depth-t node `rank`
  long long lo = 0, hi = n;
  for (int d = 0; d < tt; d++) {
    const long long half = (hi - lo + 1) / 2;
    if ((rank >> (tt - 1 - d)) & 1) lo += half; else hi = lo + half;
  }
  if (kappa) *kappa = k;
  if (t) *t = tt;
  if (row_lo) *row_lo = lo;
  if (row_hi) *row_hi = hi;
  const long long per = 1LL << (k - tt);
  if (leaf_lo) *leaf_lo = (long long)rank * per;
  if (leaf_hi) *leaf_hi = (long long)(rank + 1) * per;
  return HODLR_OK;
}

}  // extern "C"
