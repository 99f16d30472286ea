// FP64 throughput probe: DMMA m8n8k4 vs DFMA, all SMs, register-resident.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[8] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = fma(a, b, d[k]);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    k_dmma<<<sms, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    k_dmma<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)sms * warps * iters * 8 * 256;
    printf("DMMA warps/SM=%2d: %.2f TFLOP/s\n", warps, 2 * fma / (ms * 1e-3) / 1e12);
    k_dfma<<<sms, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    k_dfma<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fma = (double)sms * warps * 32 * iters * 8;
    printf("DFMA warps/SM=%2d: %.2f TFLOP/s\n", warps, 2 * fma / (ms * 1e-3) / 1e12);
  }
  return 0;
}
