// sweep.cu -- config 4 (BASELINE.json): GP log-likelihood (eq. 1) of B hyper-parameter
// settings (a, ell, sigma2) on the same points and observations.  The settings are independent problems; they are
// factored in batches (hodlr_build_batch: every kernel launch of the path covers a whole batch), and a batch that
// fails is redone setting by setting (up to `workers` concurrently: host threads, one stream each) so that each
// setting reports its own status.  With dist (nranks > 1) rank g takes settings g, g + P, ... and the values are
// allgathered ("replicas only").
#include "hodlr_internal.cuh"
#include <thread>
#include <vector>
#include <atomic>
#include <string.h>
#include <string>

#ifndef SWEEP_MAX_POINTS
#define SWEEP_MAX_POINTS (1LL << 23)   // points (B n) per batched handle
#endif

namespace {
__global__ void k_tile_rhs(const double *y, long long n, int B, double *yb) {
  const long long N = n * B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    yb[i] = y[i % n];
}
}  // namespace

extern "C" hodlr_status gp_loglik_sweep(const double *x, const double *y, int64_t n, hodlr_kernel kernel,
                                        const double *thetas, const double *sigma2s, int32_t B, int32_t leaf,
                                        double eps, const hodlr_dist *dist, void *cuda_stream, int32_t workers,
                                        double *out_host) {
  if (kernel == HODLR_RQ) return hodlr_set_error(HODLR_EINVAL, "sweep: the rational quadratic (3 parameters) is not supported");
  if (kernel == HODLR_MQ || kernel == HODLR_BIHARM)
    return hodlr_set_error(HODLR_EINVAL, "sweep: the kernel is not positive definite (no log-likelihood)");
  if (!x || !y || !thetas || !sigma2s || !out_host || B < 1 || n < 1)
    return hodlr_set_error(HODLR_EINVAL, "gp_loglik_sweep: bad arguments");
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return hodlr_cuda_check(ce, "cudaGetDevice");
  const int P = (dist && dist->nranks > 1) ? dist->nranks : 1;
  const int g = P > 1 ? dist->rank : 0;
  std::vector<int> mine;
  for (int b = g; b < B; b += P) mine.push_back(b);
  std::vector<double> val(B, 0.0);
  std::vector<hodlr_status> stat(B, HODLR_OK);
  std::vector<std::string> msg(B);
  // the caller's stream orders our reads of x and y after its prior work
  ce = cudaStreamSynchronize((cudaStream_t)cuda_stream);
  if (ce != cudaSuccess) return hodlr_cuda_check(ce, "gp_loglik_sweep: stream");
  const double half_log2pi_n = 0.5 * (double)n * log(2.0 * M_PI);
  // ---- batches: the largest powers of two of this rank's settings that fit ----
  std::vector<int> redo;
  {
    const int tw = 2;                              // (the rational quadratic is refused above)
    long long bmax = 1;
    while (bmax * 2 * n <= SWEEP_MAX_POINTS) bmax *= 2;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    size_t k0 = 0;
    double *yb = nullptr; long long yb_n = 0;
    while (k0 < mine.size()) {
      long long nb = 1;
      while (nb * 2 <= bmax && k0 + nb * 2 <= mine.size()) nb *= 2;
      if (nb == 1 || n < leaf) {                   // single settings: the per-setting path below
        for (size_t k = k0; k < k0 + nb; k++) redo.push_back(mine[k]);
        k0 += nb; continue;
      }
      std::vector<double> th((size_t)nb * tw), s2((size_t)nb);
      for (long long j = 0; j < nb; j++) {
        const int b = mine[k0 + j];
        for (int q = 0; q < 2; q++) th[j * tw + q] = thetas[2 * b + q];
        s2[j] = sigma2s[b];
      }
      hodlr_status st = HODLR_OK;
      if (yb_n < nb * n) {                          // (stream-ordered pool allocations: no device-wide sync)
        if (yb) cudaFreeAsync(yb, s);
        yb = nullptr; yb_n = 0;
        if (cudaMallocAsync(&yb, sizeof(double) * nb * n, s) != cudaSuccess) { cudaGetLastError(); st = hodlr_set_error(HODLR_ENOMEM, "sweep: rhs"); }
        else yb_n = nb * n;
      }
      hodlr_t h = nullptr;
      if (st == HODLR_OK) {
        k_tile_rhs<<<592, 256, 0, s>>>(y, n, (int)nb, yb);
        hodlr_global_launches++;
        st = hodlr_build_batch(x, n, kernel, th.data(), s2.data(), (int)nb, leaf, eps, nullptr, s, &h);
      }
      double qtot = 0.0;
      std::vector<double> ld(nb), qd(nb);
      // y fused into the factorization: y^T C_s^{-1} y is problem s's root Pi, no solve pass
      if (st == HODLR_OK) st = hodlr_factor_solve(h, yb, nullptr, &qtot);
      if (st == HODLR_OK) st = hodlr_batch_results(h, ld.data(), qd.data());
      hodlr_free(h);
      if (st == HODLR_OK) {
        // eq. 1: -1/2 y^T C^{-1} y - 1/2 log det C - (n/2) log(2 pi)
        for (long long j = 0; j < nb; j++) val[mine[k0 + j]] = -0.5 * qd[j] - 0.5 * ld[j] - half_log2pi_n;
      } else {
        for (long long j = 0; j < nb; j++) redo.push_back(mine[k0 + j]);   // find the failing setting(s)
      }
      k0 += nb;
    }
    if (yb) { cudaFreeAsync(yb, s); cudaStreamSynchronize(s); }
  }
  std::atomic<int> next(0);
  const int W = std::max(1, std::min<int>(workers > 0 ? workers : 8, (int)redo.size()));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int coop = W > 1 ? std::max(16, 2 * nsm / W) : 0;
  auto work = [&]() {
    cudaSetDevice(dev);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (;;) {
      const int k = next.fetch_add(1);
      if (k >= (int)redo.size()) break;
      const int b = redo[k];
      hodlr_t h = nullptr;
      double ll = -INFINITY;
      hodlr_status st = hodlr_build(x, n, kernel, thetas + 2 * b, sigma2s[b], leaf, eps, nullptr, nullptr, s, &h);
      if (st == HODLR_OK) h->coop_ctas = coop;  // W problems in flight: each upper-tree launch takes ~1/W of the GPU
      double quad = 0.0, ld = 0.0;
      // y fused into the factorization: y^T C^{-1} y is the root's Pi, no solve pass at all
      if (st == HODLR_OK) st = hodlr_factor_solve(h, y, nullptr, &quad);
      if (st == HODLR_OK) st = hodlr_logdet(h, &ld);
      // eq. 1: -1/2 y^T C^{-1} y - 1/2 log det C - (n/2) log(2 pi)
      if (st == HODLR_OK) ll = -0.5 * quad - 0.5 * ld - half_log2pi_n;
      if (st != HODLR_OK) msg[b] = hodlr_last_error();
      hodlr_free(h);
      val[b] = st == HODLR_OK ? ll : -INFINITY;
      stat[b] = st;
    }
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  };
  std::vector<std::thread> th;
  if (!redo.empty())
    for (int w = 0; w < W; w++) th.emplace_back(work);
  for (auto &t : th) t.join();
  if (P > 1) {     // allgather (value, status) of every rank's settings (slot k of rank r = setting r + k P)
    hodlr_s ex;
    memset((void *)&ex, 0, sizeof(ex));
    ex.kappa = 1 << 20; ex.dev = dev; ex.st = (cudaStream_t)cuda_stream;
    hodlr_status st = hodlr_dist_init(&ex, dist);
    if (st != HODLR_OK) return st;
    const int per = (B + P - 1) / P;
    std::vector<double> send(2 * per, 0.0), all(2 * (size_t)per * P, 0.0);
    for (int k = 0; k < (int)mine.size(); k++) { send[2 * k] = val[mine[k]]; send[2 * k + 1] = (double)stat[mine[k]]; }
    double *dbuf = nullptr;
    if (cudaMalloc(&dbuf, sizeof(double) * 2 * per * (P + 1)) != cudaSuccess) return hodlr_set_error(HODLR_ENOMEM, "sweep");
    cudaMemcpy(dbuf, send.data(), sizeof(double) * 2 * per, cudaMemcpyHostToDevice);
    st = hodlr_allgather(&ex, dbuf, dbuf + 2 * per, sizeof(double) * 2 * per);
    if (st == HODLR_OK) {
      cudaStreamSynchronize(ex.st);
      cudaMemcpy(all.data(), dbuf + 2 * per, sizeof(double) * 2 * per * P, cudaMemcpyDeviceToHost);
    }
    cudaFree(dbuf);
    hodlr_dist_fini(&ex);
    if (st != HODLR_OK) return st;
    for (int r = 0; r < P; r++)
      for (int k = 0; r + k * P < B; k++) {
        val[r + k * P] = all[2 * ((size_t)r * per + k)];
        stat[r + k * P] = (hodlr_status)(int)all[2 * ((size_t)r * per + k) + 1];
      }
  }
  hodlr_status first = HODLR_OK;
  for (int b = 0; b < B; b++) {
    out_host[b] = val[b];
    if (first == HODLR_OK && stat[b] != HODLR_OK) {
      first = stat[b];
      hodlr_set_error(first, "gp_loglik_sweep: setting %d: %s", b, msg[b].empty() ? "(on another rank)" : msg[b].c_str());
    }
  }
  return first;
}
