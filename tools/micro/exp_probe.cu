// Development probe: how often CUDA's exp(double) differs from the host libm exp on ACA-like arguments.
#include <cstdio>
#include <cmath>
#include <vector>
#include <random>
__global__ void k(const double *x, double *y, int n) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) y[i] = exp(x[i]); }
int main() {
  const int n = 1 << 20;
  std::vector<double> x(n), y(n);
  std::mt19937_64 g(1); std::uniform_real_distribution<double> u(0.0, 60.0);
  for (auto &v : x) v = -u(g);
  double *dx, *dy; cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dx, dy, n);
  cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost);
  long diff = 0, diffl = 0;
  for (int i = 0; i < n; i++) {
    if (y[i] != std::exp(x[i])) diff++;
    if (y[i] != (double)std::exp((long double)x[i])) diffl++;
  }
  printf("CUDA exp vs host libm exp: %.4f%% differ; vs long-double rounded: %.4f%%\n", 100.0 * diff / n, 100.0 * diffl / n);
  return 0;
}
