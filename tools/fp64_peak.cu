// fp64_peak.cu -- measured FP64 peak on this B200 (DFMA pipe and DMMA mma.sync), for the roofline
// denominator (MEASURED_PEAKS.json has no FP64 figure).  Prints one JSON line.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma884(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_dmma1688(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0, b1 = 0.5;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double *out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best[3] = {1e30f, 1e30f, 1e30f};
  const int iters = 20000;
  const int blocks = sms * 4, threads = 256;
  for (int rep = 0; rep < 5; rep++) {
    float ms;
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[0]) best[0] = ms;
    cudaEventRecord(e0); k_dmma884<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[1]) best[1] = ms;
    cudaEventRecord(e0); k_dmma1688<<<blocks, threads>>>(out, iters / 2); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best[2]) best[2] = ms;
  }
  double thr = (double)blocks * threads;
  double f_dfma = thr * iters * 16 * 2 / (best[0] * 1e-3) / 1e12;
  double f_884 = (double)blocks * (threads / 32) * iters * 8 * (8 * 8 * 4 * 2) / (best[1] * 1e-3) / 1e12;
  double f_1688 = (double)blocks * (threads / 32) * (iters / 2) * 4 * (16 * 8 * 8 * 2) / (best[2] * 1e-3) / 1e12;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_m8n8k4_tflops\": %.3f, \"fp64_dmma_m16n8k8_tflops\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n",
         f_dfma, f_884, f_1688, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
