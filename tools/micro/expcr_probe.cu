// Development probe: exp_cr (hodlr_internal.cuh) vs the host libm exp and a long-double reference.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
#include "hodlr_internal.cuh"
__global__ void k(const double *x, double *y, double *z, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { y[i] = exp_cr(x[i]); z[i] = exp(x[i]); }
}
int main() {
  const int n = 1 << 22;
  std::vector<double> x(n), y(n), z(n);
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> u(0.0, 60.0), u2(0.0, 700.0), u3(0.0, 1e-3);
  for (int i = 0; i < n; i++) x[i] = -(i % 3 == 0 ? u(g) : (i % 3 == 1 ? u2(g) : u3(g)));
  double *dx, *dy, *dz; cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dz, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dx, dy, dz, n);
  cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(z.data(), dz, n * 8, cudaMemcpyDeviceToHost);
  long d_cr = 0, d_cuda = 0, d_crl = 0, bad = 0;
  for (int i = 0; i < n; i++) {
    const double h = std::exp(x[i]);
    const double l = (double)std::exp((long double)x[i]);
    if (y[i] != h) d_cr++;
    if (z[i] != h) d_cuda++;
    if (y[i] != l) d_crl++;
    if (std::fabs(y[i] - h) > 2.5e-16 * h) bad++;
  }
  printf("exp_cr vs libm: %.5f%% differ (vs long double %.5f%%, > 1 ulp: %ld); CUDA exp vs libm: %.4f%%\n",
         100.0 * d_cr / n, 100.0 * d_crl / n, bad, 100.0 * d_cuda / n);
  return 0;
}
