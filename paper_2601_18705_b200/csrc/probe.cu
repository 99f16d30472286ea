// FP64 tensor-core throughput probe (bench.py's DMMA roofline denominator):
// every warp issues independent chains of mma.sync m8n8k4 f64 (SASS
// DMMA.8x8x4) on register operands, no memory traffic.  FLOPs per launch =
// 2 * 256 * 8 * iters * warps (one m8n8k4 = 256 FMA).
#include "common.cuh"

namespace dlrsn {
__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void dmma_probe_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double d[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma_acc(d[k][0], d[k][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.0) out[0] = s;  // keeps the chains live
}
}  // namespace dlrsn

using namespace dlrsn;

extern "C" int dlrsn_dmma_probe(int blocks, int warps_per_block, int iters, double* sink,
                                dlrsn_stream_t stream) {
  DLRSN_REQUIRE(blocks > 0 && warps_per_block > 0 && warps_per_block <= 32 && iters > 0,
                "bad probe shape");
  dmma_probe_kernel<<<blocks, 32 * warps_per_block, 0, as_stream(stream)>>>(sink, iters);
  DLRSN_CHECK_LAUNCH("dmma_probe_kernel");
  return DLRSN_OK;
}
