// Shared helpers for the sm_100a DLR-SN kernels: error plumbing, the
// sweep-native "SK" addressing (see include/dlrsn.h) and small fp64 utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>

#include "../../include/dlrsn.h"

namespace dlrsn {

void set_error(const char* fmt, ...);

// kernels launched by this library since load (dlrsn_launch_count)
inline std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

#define DLRSN_TRY_CUDA(expr)                                                        \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ::dlrsn::set_error("%s failed: %s", #expr, cudaGetErrorString(e_));           \
      return DLRSN_ECUDA;                                                           \
    }                                                                               \
  } while (0)

#define DLRSN_CHECK_LAUNCH(name)                                                    \
  do {                                                                              \
    ::dlrsn::launch_counter().fetch_add(1, std::memory_order_relaxed);              \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) {                                                        \
      ::dlrsn::set_error("launch of %s failed: %s", name, cudaGetErrorString(e_));  \
      return DLRSN_ECUDA;                                                           \
    }                                                                               \
  } while (0)

#define DLRSN_REQUIRE(cond, ...)                                                    \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      ::dlrsn::set_error(__VA_ARGS__);                                              \
      return DLRSN_EINVAL;                                                          \
    }                                                                               \
  } while (0)

inline cudaStream_t as_stream(dlrsn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Zero fill as a kernel, not cudaMemsetAsync: a memset can be queued on a
// copy engine behind unrelated bulk host<->device copies of other streams
// (measured: 256-byte memsets stretched to 75-135 us while bench.py's e2e
// copies ran), while a kernel stays on the compute pipe.
static __global__ void zero_words_kernel(uint32_t* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0u;
}
static inline cudaError_t zero_async(void* p, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  const int64_t n = (int64_t)((bytes + 3) / 4);  // callers pass 4-byte multiples
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 1184);
  zero_words_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<uint32_t*>(p), n);
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

constexpr double kFourPi = 12.566370614359172;  // 4*np.pi
constexpr double kPi = 3.141592653589793;
constexpr unsigned kFull = 0xffffffffu;

// ---- SK layout -------------------------------------------------------------
__host__ __device__ inline int sk_strips(int ny) { return (ny + 31) >> 5; }
__host__ __device__ inline int sk_steps(int nx) { return nx + 31; }
__host__ __device__ inline int64_t sk_vec_len(int nx, int ny) {
  return (int64_t)sk_strips(ny) * sk_steps(nx) * 128;
}
__host__ __device__ inline int64_t sk_scalar_len(int nx, int ny) {
  return (int64_t)sk_strips(ny) * sk_steps(nx) * 32;
}
// offset (in doubles) of the double2 holding oriented dofs (2h, 2h+1)
__host__ __device__ inline int64_t sk_vec_off(int T, int s, int t, int h, int lane) {
  return ((((int64_t)s * T + t) * 2 + h) * 32 + lane) * 2;
}
__host__ __device__ inline int64_t sk_sc_off(int T, int s, int t, int lane) {
  return ((int64_t)s * T + t) * 32 + lane;
}
// canonical cell (i,j) -> (strip, step, lane) in quadrant `quad`
__host__ __device__ inline void sk_locate(int i, int j, int quad, int nx, int ny, int& s, int& t,
                                          int& lane) {
  const int ip = (quad & 1) ? nx - 1 - i : i;
  const int jp = (quad & 2) ? ny - 1 - j : j;
  s = jp >> 5;
  lane = jp & 31;
  t = ip + lane;
}
// oriented local dof <-> canonical local dof (an involution)
__host__ __device__ inline int sk_flip(int quad) { return (quad & 1) | (quad & 2); }

// ---- memory-model helpers ---------------------------------------------------
__device__ inline int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ inline void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ inline int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a) ---------------------------
__device__ inline uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ inline void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ inline void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ inline void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion signalled on `bar`
__device__ inline void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ inline bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// warp-converged variant: every lane leaves the loop in the same iteration
__device__ inline void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try_wait(bar, parity))) {
  }
}

// deterministic block sum of NV doubles (fixed tree order); result in lane 0
// of warp 0.  blockDim.x must be a multiple of 32 and <= 1024.
template <int NV>
__device__ inline void block_sum(double (&v)[NV], double* smem /* 32*NV */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(kFull, v[k], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[w * NV + k] = v[k];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      v[k] = lane < nw ? smem[lane * NV + k] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(kFull, v[k], o);
    }
  }
}

}  // namespace dlrsn
