// predict.cu -- GP prediction at test points (NEXT-1 of SURVEY 8(f); eq_reg1 / eq_reg2):
//   mean_j = k(xt_j, x) alpha,                alpha = C^{-1} y          (hodlr_solve)
//   var_j  = k(xt_j, xt_j) - k(xt_j, x) C^{-1} k(x, xt_j)               (latent f; sigma^2 not added)
// The cross-covariance columns k(x, xt_j) are evaluated on the fly (Table I); the variance
// solves them in batches of PB test points with the HODLR solve.  Fixed-order reductions: deterministic.
#include "hodlr_internal.cuh"
#include <algorithm>

namespace {

constexpr int PB = 32;           // test points per variance batch

// mean_j = sum_i k(xt_j - xs_i) alpha[perm[i]]: a CTA takes MT test points; the sorted points and their alpha are
// staged in shared memory in chunks and reused by all MT test points (thread (test point, lane) over the chunk),
// fixed-order warp reductions.
constexpr int MT = 8;            // test points per CTA (one warp each)
constexpr int MCH = 2048;        // points per staged chunk
__global__ void __launch_bounds__(MT * 32) k_predict_mean(KParams kp, const double *xs, const long long *perm,
                                                          long long n, const double *alpha, const double *xt,
                                                          long long m, double *mean) {
  __shared__ double sx[MCH], sa[MCH];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long j = (long long)blockIdx.x * MT + w;
  const double x0 = j < m ? xt[j] : 0.0;
  double s = 0.0;
  for (long long c0 = 0; c0 < n; c0 += MCH) {
    const int len = (int)(n - c0 < MCH ? n - c0 : MCH);
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += MT * 32) { sx[i] = xs[c0 + i]; sa[i] = alpha[perm[c0 + i]]; }
    __syncthreads();
    for (int i = lane; i < len; i += 32) s = fma(kval(kp, x0 - sx[i]), sa[i], s);
  }
  s = warp_sum(s);
  if (lane == 0 && j < m) mean[j] = s;
}

// Kx[:, b] = k(x - xt_{j0 + b}) in the caller's original order (column-major, leading dimension n).
__global__ void k_cross_cols(KParams kp, const double *xs, const long long *perm, long long n,
                             const double *xt, long long j0, int nb, double *Kx) {
  const long long tot = n * nb;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < tot; p += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(p / n); const long long i = p - (long long)b * n;
    Kx[(long long)b * n + perm[i]] = kval(kp, xs[i] - xt[j0 + b]);
  }
}

// var_{j0+b} = k(0) - Kx[:, b] . Z[:, b]: one CTA per column, fixed-order block reduction.
__global__ void __launch_bounds__(256) k_predict_var(KParams kp, long long n, const double *Kx, const double *Z,
                                                     long long j0, double *var) {
  __shared__ double red[8];
  const int b = blockIdx.x, t = threadIdx.x;
  const double *kc = Kx + (long long)b * n, *zc = Z + (long long)b * n;
  double s = 0.0;
  for (long long i = t; i < n; i += 256) s = fma(kc[i], zc[i], s);
  s = warp_sum(s);
  if ((t & 31) == 0) red[t >> 5] = s;
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; w++) tot += red[w];
    var[j0 + b] = kval(kp, 0.0) - tot;
  }
}

}  // namespace

hodlr_status hodlr_predict_impl(hodlr_s *h, const double *y, const double *xt, long long m, double *mean, double *var) {
  const long long n = h->n;
  const size_t need = (size_t)n * (1 + 2 * PB);
  if (h->pred_ws_n < need) {
    h->pred_ws = (double *)hodlr_dalloc(h, sizeof(double) * need);
    if (!h->pred_ws) return hodlr_set_error(HODLR_ENOMEM, "predict: workspace");
    h->pred_ws_n = need;
  }
  double *alpha = h->pred_ws, *Kx = alpha + n, *Z = Kx + n * PB;
  hodlr_status st = hodlr_solve_impl(h, y, alpha, false);
  if (st != HODLR_OK) return st;
  if (m > 0) {
    k_predict_mean<<<(unsigned)((m + MT - 1) / MT), MT * 32, 0, h->st>>>(h->kp, h->xs, h->perm, n, alpha, xt, m, mean);
    HLAUNCH(h, "k_predict_mean");
  }
  if (var) {
    for (long long j0 = 0; j0 < m; j0 += PB) {
      const int nb = (int)std::min<long long>(PB, m - j0);
      const long long tot = n * nb;
      k_cross_cols<<<(unsigned)std::min<long long>((tot + 255) / 256, 8192), 256, 0, h->st>>>(h->kp, h->xs, h->perm, n,
                                                                                          xt, j0, nb, Kx);
      HLAUNCH(h, "k_cross_cols");
      for (int b = 0; b < nb && st == HODLR_OK; b++) st = hodlr_solve_impl(h, Kx + (long long)b * n, Z + (long long)b * n, false);
      if (st != HODLR_OK) return st;
      k_predict_var<<<nb, 256, 0, h->st>>>(h->kp, n, Kx, Z, j0, var);
      HLAUNCH(h, "k_predict_var");
    }
  }
  return HODLR_OK;
}
