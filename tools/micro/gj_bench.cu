// Microbenchmark (development tool): Gauss-Jordan with partial pivoting of one q x q coupling system in one warp,
// register (fully unrolled) vs shared-memory (transposed) variants.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -I../../paper_1403_6015_b200/csrc gj_bench.cu -o gj_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "tree_node.cuh"

template <int QB>
__global__ void __launch_bounds__(32, 1) k_regs(const double *W0, double *out, int q, long long *cyc) {
  __shared__ double W[32 * 64], W2[32 * 64], ukk[64];
  for (int p = threadIdx.x; p < q * 2 * q; p += 32) W[p] = W0[p];
  __syncwarp();
  long long t0 = clock64();
  int sign, zero;
  gj_regs<QB>(W, W2, q, ukk, sign, zero);
  __syncwarp();
  long long t1 = clock64();
  for (int p = threadIdx.x; p < q * 2 * q; p += 32) out[p] = W2[p];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void __launch_bounds__(32, 1) k_warp(const double *W0, double *out, int q, long long *cyc) {
  __shared__ double W[32 * 64], W2[32 * 64], ukk[64];
  for (int p = threadIdx.x; p < q * 2 * q; p += 32) W[p] = W0[p];
  __syncwarp();
  long long t0 = clock64();
  int sign, zero;
  gj_warp(W, W2, W, q, ukk, sign, zero);
  __syncwarp();
  long long t1 = clock64();
  for (int p = threadIdx.x; p < q * 2 * q; p += 32) out[p] = W[p];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  for (int q : {8, 16, 26, 32}) {
    std::vector<double> W(q * 2 * q);
    srand(1);
    for (int a = 0; a < q; a++)
      for (int j = 0; j < 2 * q; j++)
        W[a * 2 * q + j] = j < q ? (a == j ? 1.0 : 0.0) + 0.5 * ((rand() % 2001) / 1000.0 - 1.0) : (j - q == a ? 1.0 : 0.0);
    double *dW, *o1, *o2; long long *c;
    cudaMalloc(&dW, sizeof(double) * W.size()); cudaMalloc(&o1, sizeof(double) * W.size()); cudaMalloc(&o2, sizeof(double) * W.size());
    cudaMalloc(&c, 16);
    cudaMemcpy(dW, W.data(), sizeof(double) * W.size(), cudaMemcpyHostToDevice);
    long long cr = 0, cw = 0;
    for (int rep = 0; rep < 3; rep++) {
      if (q <= 8) k_regs<8><<<1, 32>>>(dW, o1, q, c);
      else if (q <= 16) k_regs<16><<<1, 32>>>(dW, o1, q, c);
      else k_regs<32><<<1, 32>>>(dW, o1, q, c);
      cudaMemcpy(&cr, c, 8, cudaMemcpyDeviceToHost);
      k_warp<<<1, 32>>>(dW, o2, q, c);
      cudaMemcpy(&cw, c, 8, cudaMemcpyDeviceToHost);
    }
    std::vector<double> a(W.size()), b(W.size());
    cudaMemcpy(a.data(), o1, sizeof(double) * W.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), o2, sizeof(double) * W.size(), cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (int r = 0; r < q; r++) for (int j = 0; j < q; j++) {
      md = fmax(md, fabs(a[r * 2 * q + q + j] - b[r * 2 * q + q + j])); mx = fmax(mx, fabs(a[r * 2 * q + q + j]));
    }
    printf("q=%2d  regs %7lld cycles  warp-smem %7lld cycles  max|diff| %.2e (max %.2e)  err=%s\n", q, cr, cw, md, mx,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
