// predict.cu -- GP prediction at test points (NEXT-1 of SURVEY 8(f); eq_reg1 / eq_reg2):
//   mean_j = k(xt_j, x) alpha,                alpha = C^{-1} y          (hodlr_solve)
//   var_j  = k(xt_j, xt_j) - k(xt_j, x) C^{-1} k(x, xt_j)               (latent f; sigma^2 not added)
// The cross-covariance columns k(x, xt_j) are evaluated on the fly (Table I); the variance needs
// only the quadratic forms k_j^T C^{-1} k_j: the solve's up pass (h at the root) for PB columns in one batched
// launch.  Fixed-order reductions: deterministic.
#include "hodlr_internal.cuh"
#include <algorithm>

namespace {

// d-dimensional handles (NEXT-3): k(xt_j, x_i) of sorted point i (coordinate-major xs) and test point j (row-major xt)
__device__ __forceinline__ double kval_xt(const KParams &kp, const double *xs, long long i, const double *xt, long long j) {
  double r2 = 0.0;
  for (int k = 0; k < kp.dim; k++) { const double d = xs[k * kp.ldp + i] - xt[j * kp.dim + k]; r2 = fma(d, d, r2); }
  if (kp.kern == HODLR_SE) return kp.a2 * exp(-r2 * kp.c);
  return kval(kp, sqrt(r2));
}

constexpr int PB = 32;           // test points per variance batch

// mean_j = sum_i k(xt_j - xs_i) alpha[perm[i]]: CTA (b, y) takes MT test points and the y-th slice of MSL points;
// the slice's sorted points and their alpha are staged in shared memory in chunks and reused by all MT test points
// (thread (test point, lane) over the chunk), fixed-order warp reductions into partial[j][y]; k_predict_mean_sum adds
// the slices in order (deterministic).  Slicing the points keeps the whole GPU busy for few test points.
constexpr int MT = 8;            // test points per CTA (one warp each)
constexpr int MCH = 2048;        // points per staged chunk
constexpr long long MSL = 16384; // points per slice (grid.y)
__global__ void __launch_bounds__(MT * 32) k_predict_mean(KParams kp, const double *xs, const long long *perm,
                                                          long long n, const double *alpha, const double *xt,
                                                          long long m, double *partial, int nsl) {
  __shared__ double sx[MCH], sa[MCH];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long j = (long long)blockIdx.x * MT + w;
  const long long s0 = blockIdx.y * MSL, s1 = s0 + MSL < n ? s0 + MSL : n;
  double s = 0.0;
  if (kp.dim > 1) {                              // d-dimensional: coordinate rows read directly (coalesced by lane)
    const long long jj = j < m ? j : 0;
    for (long long i = s0 + lane; i < s1; i += 32) s = fma(kval_xt(kp, xs, i, xt, jj), alpha[perm[i]], s);
    s = warp_sum(s);
    if (lane == 0 && j < m) partial[j * nsl + blockIdx.y] = s;
    return;
  }
  const double x0 = j < m ? xt[j] : 0.0;
  for (long long c0 = s0; c0 < s1; c0 += MCH) {
    const int len = (int)(s1 - c0 < MCH ? s1 - c0 : MCH);
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += MT * 32) { sx[i] = xs[c0 + i]; sa[i] = alpha[perm[c0 + i]]; }
    __syncthreads();
    for (int i = lane; i < len; i += 32) s = fma(kval(kp, x0 - sx[i]), sa[i], s);
  }
  s = warp_sum(s);
  if (lane == 0 && j < m) partial[j * nsl + blockIdx.y] = s;
}

__global__ void k_predict_mean_sum(const double *partial, int nsl, long long m, double *mean) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int y = 0; y < nsl; y++) s += partial[j * nsl + y];
  mean[j] = s;
}

// Kx[:, b] = k(x - xt_{j0 + b}) in the caller's original order (column-major, leading dimension n).
__global__ void k_cross_cols(KParams kp, const double *xs, const long long *perm, long long n,
                             const double *xt, long long j0, int nb, double *Kx) {
  const long long tot = n * nb;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < tot; p += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(p / n); const long long i = p - (long long)b * n;
    Kx[(long long)b * n + perm[i]] = kp.dim > 1 ? kval_xt(kp, xs, i, xt, j0 + b) : kval(kp, xs[i] - xt[j0 + b]);
  }
}

// var_{j0+b} = k(0) - k_b^T C^{-1} k_b, the quadratic form being the root's h of the batched up pass (a compensated
// pair, column b at hv + b hcol)
__global__ void k_predict_var_h(KParams kp, const double *hv, long long hcol, int nb, long long j0, double *var) {
  const int b = threadIdx.x;
  if (b < nb) var[j0 + b] = kval(kp, 0.0) - (hv[b * hcol] + hv[b * hcol + 1]);
}

}  // namespace

hodlr_status hodlr_predict_impl(hodlr_s *h, const double *y, const double *xt, long long m, double *mean, double *var) {
  if (h->nbatch > 1) return hodlr_set_error(HODLR_EINVAL, "predict: not supported on batched handles");
  const long long n = h->n;
  const int nsl = (int)((n + MSL - 1) / MSL);
  const size_t need = (size_t)n * (1 + PB) + (size_t)(m > 0 ? m : 1) * nsl;
  if (h->pred_ws_n < need) {
    h->pred_ws = (double *)hodlr_dalloc(h, sizeof(double) * need);
    if (!h->pred_ws) return hodlr_set_error(HODLR_ENOMEM, "predict: workspace");
    h->pred_ws_n = need;
  }
  double *alpha = h->pred_ws, *Kx = alpha + n, *partial = Kx + n * PB;
  hodlr_status st = hodlr_solve_impl(h, y, alpha, 1, n, false);
  if (st != HODLR_OK) return st;
  if (m > 0) {
    k_predict_mean<<<dim3((unsigned)((m + MT - 1) / MT), (unsigned)nsl), MT * 32, 0, h->st>>>(h->kp, h->xs, h->perm,
                                                                                           n, alpha, xt, m, partial, nsl);
    HLAUNCH(h, "k_predict_mean");
    k_predict_mean_sum<<<(unsigned)((m + 255) / 256), 256, 0, h->st>>>(partial, nsl, m, mean);
    HLAUNCH(h, "k_predict_mean");
  }
  if (var) {
    for (long long j0 = 0; j0 < m; j0 += PB) {
      const int nb = (int)std::min<long long>(PB, m - j0);
      const long long tot = n * nb;
      k_cross_cols<<<(unsigned)std::min<long long>((tot + 255) / 256, 8192), 256, 0, h->st>>>(h->kp, h->xs, h->perm, n,
                                                                                          xt, j0, nb, Kx);
      HLAUNCH(h, "k_cross_cols");
      // k_j^T C^{-1} k_j for all nb columns at once: the batched up pass alone (h at the root), no down pass
      st = hodlr_solve_impl(h, Kx, nullptr, nb, n, true);
      if (st != HODLR_OK) return st;
      k_predict_var_h<<<1, PB, 0, h->st>>>(h->kp, h->hvec, h->hcol, nb, j0, var);
      HLAUNCH(h, "k_predict_var");
    }
  }
  return HODLR_OK;
}
