// Micro-benchmarks of dependent-latency on B200: DFMA chain, rcp64, shfl.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void rcp_chain(double* out, int n, long long* cyc) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); r = fma(r, e, r);
    x = r + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void div_chain(double* out, int n, long long* cyc) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = 1.0 / x + 1.0; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void shfl_chain(double* out, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1) + 1.0; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void dfma_tput(double* out, double a, double b, int n, long long* cyc) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7; if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMallocManaged(&cyc, 8);
  int n = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    dfma_chain<<<1, 32>>>(out, 0.999, 0.001, n, cyc); cudaDeviceSynchronize();
    if (rep) printf("DFMA dependent latency: %.2f cycles\n", (double)*cyc / (4.0 * n));
    rcp_chain<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize();
    if (rep) printf("rcp64 (approx+2 Newton)+add chain: %.2f cycles\n", (double)*cyc / n);
    div_chain<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize();
    if (rep) printf("1.0/x + 1 chain: %.2f cycles\n", (double)*cyc / n);
    shfl_chain<<<1, 32>>>(out, n, cyc); cudaDeviceSynchronize();
    if (rep) printf("shfl_up(f64)+DADD chain: %.2f cycles\n", (double)*cyc / n);
    for (int w = 1; w <= 8; w *= 2) {
      dfma_tput<<<1, 32 * w>>>(out, 0.999, 0.001, n, cyc); cudaDeviceSynchronize();
      if (rep) printf("DFMA throughput, %d warps/SM: %.2f cycles per warp-instr per warp (8 indep chains)\n", w, (double)*cyc / (8.0 * n));
    }
  }
  return 0;
}
