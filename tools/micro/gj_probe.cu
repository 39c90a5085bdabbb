// Development probe: cost breakdown of one-warp register Gauss-Jordan steps (argmax / broadcast / update).
#include <cstdio>
#include <cmath>
template <int QB, int MODE>   // MODE 0 full, 1 no argmax (pivot = k), 2 no argmax + reciprocal multiply, 3 update only
__global__ void __launch_bounds__(32, 1) k(const double *W0, double *out, int q, long long *cyc) {
  const int lane = threadIdx.x;
  double w[2 * QB];
#pragma unroll
  for (int j = 0; j < 2 * QB; j++) w[j] = (lane < q && j < 2 * q) ? W0[lane * 2 * q + j] : 0.0;
  long long t0 = clock64();
  int pos = lane;
#pragma unroll
  for (int kk = 0; kk < QB; kk++) {
    if (kk < q) {
      int P = kk;
      if (MODE == 0 || MODE == 6) {
        double best = (lane < q && pos >= kk) ? fabs(w[kk]) : -1.0;
        int bp = pos, bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
          const int p2 = __shfl_xor_sync(0xffffffffu, bp, o), l2 = __shfl_xor_sync(0xffffffffu, bl, o);
          if (b2 > best || (b2 == best && p2 < bp)) { best = b2; bp = p2; bl = l2; }
        }
        P = bl;
        if (bp != kk) { if (pos == kk) pos = bp; else if (lane == P) pos = kk; }
      }
      const double piv = (MODE == 3 || MODE == 4) ? 1.0 : __shfl_sync(0xffffffffu, w[kk], P);
      const double ip = (MODE >= 2 && MODE != 6) ? piv : 1.0 / piv;
      const double mlt = lane == P ? 0.0 : w[kk] * ip;
      if (MODE < 4) {
#pragma unroll
      for (int j = 0; j < 2 * QB; j++) {
        if (j > kk && (j < q || (j >= QB && j - QB < q))) {
          const double prj = __shfl_sync(0xffffffffu, w[j], P);
          w[j] = lane == P ? w[j] * ip : fma(-mlt, prj, w[j]);
        }
      }
      } else {  // MODE 4: update only, batched; MODE 6: full step, batched
        const double sc = lane == P ? ip : 1.0, ml = lane == P ? 0.0 : mlt;
#pragma unroll
        for (int j0 = 0; j0 < 2 * QB; j0 += 8) {
          double pr[8];
#pragma unroll
          for (int u = 0; u < 8; u++) { const int j = j0 + u; if (j > kk && (j < q || (j >= QB && j - QB < q))) pr[u] = __shfl_sync(0xffffffffu, w[j], P); }
#pragma unroll
          for (int u = 0; u < 8; u++) { const int j = j0 + u; if (j > kk && (j < q || (j >= QB && j - QB < q))) w[j] = fma(-ml, pr[u], w[j] * sc); }
        }
      }
    }
  }
  long long t1 = clock64();
  for (int j = 0; j < 2 * QB; j++) if (lane < q) out[lane * 2 * QB + j] = w[j];
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  double *W, *o; long long *c;
  cudaMalloc(&W, 64 * 64 * 8); cudaMalloc(&o, 64 * 64 * 8); cudaMalloc(&c, 8);
  double h[64 * 64];
  for (int i = 0; i < 64 * 64; i++) h[i] = (i % 7) * 0.1 + (i % 65 == 0 ? 2.0 : 0.0);
  cudaMemcpy(W, h, sizeof(h), cudaMemcpyHostToDevice);
  long long cy;
#define RUN(QB, M, q) for (int r = 0; r < 3; r++) { k<QB, M><<<1, 32>>>(W, o, q, c); } cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("QB=%d mode=%d q=%d: %lld cycles (%.0f per step)\n", QB, M, q, cy, (double)cy / q);
  RUN(32, 0, 26) RUN(32, 1, 26) RUN(32, 2, 26) RUN(32, 3, 26) RUN(32, 4, 26) RUN(32, 6, 26)
  RUN(16, 0, 16) RUN(16, 1, 16) RUN(16, 2, 16) RUN(16, 3, 16)
  RUN(8, 0, 8) RUN(8, 1, 8) RUN(8, 3, 8) RUN(8, 4, 8) RUN(16, 4, 16)
  return 0;
}
