// K1 (latency-optimised): warp-specialised sweep for single-direction groups.
//
// Same math and data layout as sweep.cu (transport_sn.py:142-163,303-322),
// split so that only the upwind-dependent part sits on the critical path:
//
//   psi = A^-1 (rhs + scat + Cx x_in + Cy y_in) = z + Kx x_in + Ky y_in,
//   z = A^-1 (rhs + scat),  Kx = A^-1 Cx (4x2),  Ky = A^-1 Cy (4x2).
//
// A CTA owns one (group, 32-row strip) work item at a time:
//   * warps 1..3 ("producers") take the TMA-staged sigma_t / scattering
//     source / rhs of each chunk of C skewed steps, form and LU-factor the
//     4x4 local operator of every lane and write (z, Kx, Ky) -- 20 doubles per
//     lane-step -- into a double-buffered shared-memory ring;
//   * warp 0 ("consumer") walks the strip: per step 16 FMAs, the closure
//     accumulation, two stores and one shuffle, so the dependent chain is
//     ~3 FMAs + a shuffle instead of a full 4x4 factorisation.
// mbarriers (one arrive per chunk) order producers and consumer; the strip
// handoff is the self-flagging L2 column of sweep.cu.
#include <cmath>

#include "sweep_common.cuh"

namespace dlrsn {

__device__ __forceinline__ double ld_volatile_shared_f64(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}

__device__ __forceinline__ unsigned long long ws_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define WS_TRACE(k)                                                                   \
  do {                                                                                \
    if (a.trace && (threadIdx.x & 31) == 0 && m < a.trace_chunks)                     \
      a.trace[((int64_t)item * a.trace_chunks + m) * 8 + (k)] = ws_timer();           \
  } while (0)

constexpr int kWsC = 6;      // skewed steps per chunk (= 2 x producers)
constexpr int kWsProd = 3;   // producer warps 1-3; warp 7 polls the strip handoff;
                             // warps 4-6 stay idle so that the consumer (warp 0)
                             // has its SM sub-partition to itself
constexpr int kWsThreads = 256;
constexpr int kWsStages = 3;  // ring depth (also keeps the CTA alone on its SM)
constexpr int kWsHRing = 8;   // chunks of strip-handoff values staged in shared memory
constexpr int kWsPairs = 10; // z (2 pairs), Kx (4 pairs), Ky (4 pairs)
constexpr int kWsInD = kWsC * (32 + 128 + 128);  // sigma | scat | rhs doubles per stage
constexpr int kWsFacD = kWsC * kWsPairs * 64;    // factor doubles per stage
constexpr size_t kWsSmem = (kWsStages * (size_t)kWsInD + kWsStages * (size_t)kWsFacD) * sizeof(double);

__device__ __forceinline__ void named_bar_producers() {
  asm volatile("bar.sync 1, %0;" ::"r"(kWsProd * 32) : "memory");
}

// Factor one lane-step: (z, Kx, Ky) of the local operator at skewed step tt
// of the staged chunk.  Straight-line code (no early exit) so that two calls
// in a row are interleaved by the scheduler (two independent FP64 chains).
__device__ __forceinline__ void ws_factor_step(const SweepArgs& a, const double* s_S,
                                               const double* buf, double* fac, int tt, int lane,
                                               bool scat, double ox, double oy) {
  const double sigma = buf[tt * 32 + lane];
  const double2 r0 = reinterpret_cast<const double2*>(buf + kWsC * 160 + tt * 128)[lane];
  const double2 r1 = reinterpret_cast<const double2*>(buf + kWsC * 160 + tt * 128 + 64)[lane];
  double b[4] = {r0.x, r0.y, r1.x, r1.y};
  if (scat) {
    const double2 u0 = reinterpret_cast<const double2*>(buf + kWsC * 32 + tt * 128)[lane];
    const double2 u1 = reinterpret_cast<const double2*>(buf + kWsC * 32 + tt * 128 + 64)[lane];
    b[0] += u0.x; b[1] += u0.y; b[2] += u1.x; b[3] += u1.y;
  }
  double A[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) A[q] = fma(sigma, a.mass[q], s_S[q]);
  // LU without pivoting (positive-definite symmetric part, see solve4)
  const double p0 = rcp64(A[0]);
  const double l1 = A[4] * p0, l2 = A[8] * p0, l3 = A[12] * p0;
  A[5] -= l1 * A[1]; A[6] -= l1 * A[2]; A[7] -= l1 * A[3];
  A[9] -= l2 * A[1]; A[10] -= l2 * A[2]; A[11] -= l2 * A[3];
  A[13] -= l3 * A[1]; A[14] -= l3 * A[2]; A[15] -= l3 * A[3];
  const double p1 = rcp64(A[5]);
  const double m2 = A[9] * p1, m3 = A[13] * p1;
  A[10] -= m2 * A[6]; A[11] -= m2 * A[7];
  A[14] -= m3 * A[6]; A[15] -= m3 * A[7];
  const double p2 = rcp64(A[10]);
  const double n3 = A[14] * p2;
  A[15] -= n3 * A[11];
  const double p3 = rcp64(A[15]);
  auto solve = [&](double v0, double v1, double v2, double v3, double* x) {
    const double y1 = v1 - l1 * v0;
    const double y2 = v2 - l2 * v0 - m2 * y1;
    const double y3 = v3 - l3 * v0 - m3 * y1 - n3 * y2;
    x[3] = y3 * p3;
    x[2] = (y2 - A[11] * x[3]) * p2;
    x[1] = (y1 - A[6] * x[2] - A[7] * x[3]) * p1;
    x[0] = (v0 - A[1] * x[1] - A[2] * x[2] - A[3] * x[3]) * p0;
  };
  double z[4], c0[4], c1[4], c2[4];
  solve(b[0], b[1], b[2], b[3], z);
  solve(1.0, 0.0, 0.0, 0.0, c0);
  solve(0.0, 1.0, 0.0, 0.0, c1);
  solve(0.0, 0.0, 1.0, 0.0, c2);
  double2* out = reinterpret_cast<double2*>(fac + (int64_t)tt * kWsPairs * 64) + lane;
  out[0] = make_double2(z[0], z[1]);
  out[32] = make_double2(z[2], z[3]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // pair 2+i: row i of Kx = ox A^-1[:, {0,2}] e2x ; pair 6+i: Ky = oy A^-1[:, {0,1}] e2y
    out[32 * (2 + i)] = make_double2(ox * (c0[i] * a.ex[0] + c2[i] * a.ex[2]),
                                     ox * (c0[i] * a.ex[1] + c2[i] * a.ex[3]));
    out[32 * (6 + i)] = make_double2(oy * (c0[i] * a.ey[0] + c1[i] * a.ey[2]),
                                     oy * (c0[i] * a.ey[1] + c1[i] * a.ey[3]));
  }
}

__global__ void __launch_bounds__(kWsThreads) sweep_ws_kernel(const SweepArgs a) {
  // iterations past convergence take no work item (an early return would
  // cost the compiler its proof that warps stay converged at the shuffles)
  const bool skip = a.skip != nullptr && *a.skip != 0;
  extern __shared__ __align__(128) double sm[];
  double* in_ring = sm;                 // 2 x kWsInD
  double* fac_ring = sm + kWsStages * kWsInD;   // kWsStages x kWsFacD
  __shared__ __align__(8) uint64_t in_full[kWsStages], fac_full[kWsStages], fac_empty[kWsStages];
  __shared__ double s_S[16];
  __shared__ int s_item;
  // inflow from the strip below, staged by the poller warp (warp 7):
  // slot (m % kWsHRing) holds chunk m's kWsC values; kEmpty marks a free slot
  __shared__ __align__(16) double2 s_hin[kWsHRing * kWsC];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nx = a.nx, ny = a.ny, G = a.G;
  const int T = nx + 31;
  const int ns = (ny + 31) >> 5;
  const int items = ns * G;
  const int nchunks = (T + kWsC - 1) / kWsC;
  const int hchunks = (nx + kWsC - 1) / kWsC;
  const double empty = __longlong_as_double((long long)kEmpty);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsStages; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&fac_full[i], 1);
      mbar_init(&fac_empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // per-stage use counters (identical in every thread that tracks them)
  uint32_t uses[kWsStages] = {};

  for (;;) {
    if (threadIdx.x == 0) {
      s_item = skip ? items : atomicAdd(a.ticket, 1);
      // one draw past the end per CTA; the last one re-arms the counter
      if (!skip && s_item == items + (int)gridDim.x - 1) atomicExch(a.ticket, 0);
    }
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= items) break;
    const int s = item / G;
    const int g = item - s * G;
    const dlrsn_group* grp = a.groups + g;
    const int quad = grp->quad;
    const int slot = grp->slot[0];
    const double ox = grp->ox[0], oy = grp->oy[0];
    if (threadIdx.x < 16) s_S[threadIdx.x] = ox * a.gxp[threadIdx.x] + oy * a.gyp[threadIdx.x];
    __syncthreads();
    for (int e = threadIdx.x; e < kWsHRing * kWsC; e += blockDim.x)
      s_hin[e] = make_double2(empty, empty);
    __syncthreads();
    const int64_t strip_vec = (int64_t)s * T * 128;
    const double* sig = a.sigma_sk4 + (int64_t)quad * a.slen + (int64_t)s * T * 32;
    const double* scat = a.scat_sk4 ? a.scat_sk4 + (int64_t)quad * a.vlen + strip_vec : nullptr;
    const double* rhs = a.rhs_sk + (int64_t)slot * a.vlen + strip_vec;
    const bool row_ok = (s << 5) + lane < ny;

    auto issue = [&](int m) {  // thread 32 only
      const int st = m % kWsStages, t0 = m * kWsC;
      const uint32_t n = (uint32_t)min(kWsC, T - t0);
      double* buf = in_ring + st * kWsInD;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&in_full[st], n * (256u + (scat ? 1024u : 0u) + 1024u));
      tma_load_1d(buf, sig + t0 * 32, n * 256u, &in_full[st]);
      if (scat) tma_load_1d(buf + kWsC * 32, scat + t0 * 128, n * 1024u, &in_full[st]);
      tma_load_1d(buf + kWsC * 160, rhs + t0 * 128, n * 1024u, &in_full[st]);
    };

    if (warp == 7) {
      // ------------------------------ handoff poller -----------------------
      // Polls the L2 handoff column of the strip below for the next chunks
      // (kWsHRing - 1 chunks of lookahead, one L2 round trip per sweep of
      // polls) and stages arrived values in s_hin, so the consumer never
      // waits on an L2 round trip itself.  It re-arms the L2 slots it read.
      if (s > 0) {
        double2* hin = reinterpret_cast<double2*>(a.handoff) + ((int64_t)(s - 1) * G + g) * nx;
        // lane -> (chunk offset, position): kWsC positions x 5 chunks in flight
        const int off = lane / kWsC, pos = lane - off * kWsC;
        const bool poll_lane = off < 5;
        int base = 0;  // oldest chunk not yet staged
        double2 v = make_double2(empty, empty);
        int vm = -1;  // chunk the pending value belongs to
        long long spins = 0;
        while (base < hchunks) {
          const int m = base + off;
          const int col = m * kWsC + pos;
          const bool want = poll_lane && m < hchunks && col < nx;
          if (want && m != vm) {
            v = make_double2(empty, empty);
            vm = m;
          }
          if (want && (is_empty(v.x) || is_empty(v.y))) v = __ldcv(hin + col);
          // stage chunk `base` once all its values arrived and its slot is free
          const bool mine = want && off == 0;
          const bool ready = !mine || (!is_empty(v.x) && !is_empty(v.y));
          double2* slot = s_hin + (base % kWsHRing) * kWsC + pos;
          const bool slot_free = !mine || is_empty(ld_volatile_shared_f64(&slot->x));
          if (__all_sync(kFull, ready && slot_free)) {
            if (mine) {
              *reinterpret_cast<volatile double*>(&slot->y) = v.y;
              __threadfence_block();
              *reinterpret_cast<volatile double*>(&slot->x) = v.x;
              __stcg(hin + col, make_double2(empty, empty));  // re-arm for the next sweep
            }
            // shift the in-flight values down one chunk
            const double vx = __shfl_down_sync(kFull, v.x, kWsC);
            const double vy = __shfl_down_sync(kFull, v.y, kWsC);
            const int vmn = __shfl_down_sync(kFull, vm, kWsC);
            v = off < 4 ? make_double2(vx, vy) : make_double2(empty, empty);
            vm = off < 4 ? vmn : -1;
            ++base;
            spins = 0;
          } else {
            __nanosleep(20);
            if (++spins > (1ll << 28)) {  // upstream never arrived: flag and unblock
              if (lane == 0) atomicOr(a.status, 2);
              break;
            }
          }
        }
      }
    } else if (warp >= 4) {
      // idle
    } else if (warp > 0) {
      // ------------------------------ producers ----------------------------
      const int pw = warp - 1;
      if (threadIdx.x == 32) {
        for (int m0 = 0; m0 < kWsStages && m0 < nchunks; ++m0) issue(m0);
      }
      for (int m = 0; m < nchunks; ++m) {
        const int st = m % kWsStages;
        const uint32_t u = uses[st];
        if (warp == 1) WS_TRACE(3);
        mbar_wait_warp(&in_full[st], u & 1u);
        if (u > 0) mbar_wait_warp(&fac_empty[st], (u - 1) & 1u);
        if (warp == 1) WS_TRACE(4);
        const double* buf = in_ring + st * kWsInD;
        double* fac = fac_ring + st * kWsFacD;
        // kWsC = 2 kWsProd: each producer warp factors steps pw and pw + kWsProd
        // together (inactive lanes compute harmless garbage the consumer skips)
        ws_factor_step(a, s_S, buf, fac, pw, lane, scat != nullptr, ox, oy);
        ws_factor_step(a, s_S, buf, fac, pw + kWsProd, lane, scat != nullptr, ox, oy);
        if (warp == 1) WS_TRACE(5);
        named_bar_producers();  // stage st fully read (inputs) and written (factors)
        if (warp == 1) WS_TRACE(6);
        if (threadIdx.x == 32) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fac_full[st])) : "memory");
          if (m + kWsStages < nchunks) issue(m + kWsStages);
        }
        uses[st] = u + 1;
      }
    } else {
      // ------------------------------ consumer ------------------------------
      double* psi_p = a.psi_sk + (int64_t)slot * a.vlen + strip_vec + 2 * lane;
      double2* hin = s > 0 ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)(s - 1) * G + g) * nx
                           : nullptr;
      double2* hout = (s + 1 < ns) ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)s * G + g) * nx
                                   : nullptr;
      const bool hlane = hin != nullptr && lane < kWsC;
      double x0 = 0.0, x1 = 0.0;
      double u0 = 0.0, u1 = 0.0;  // the lane below's top edge, one step back
      for (int m = 0; m < nchunks; ++m) {
        const int st = m % kWsStages;
        const uint32_t u = uses[st];
        // inflow of lane 0 for this chunk's columns (staged by the poller);
        // lane 0 keeps all kWsC values in registers
        double2 hv[kWsC];
#pragma unroll
        for (int tt = 0; tt < kWsC; ++tt) hv[tt] = make_double2(0.0, 0.0);
        if (hin != nullptr) {
          const bool need = hlane && m < hchunks && m * kWsC + lane < nx;
          double2* hs = s_hin + (m % kWsHRing) * kWsC + lane;
          long long spins = 0;
          bool got = !need;
          while (!__all_sync(kFull, got)) {
            if (!got) {
              const double hx = ld_volatile_shared_f64(&hs->x);
              const double hy = ld_volatile_shared_f64(&hs->y);
              got = !is_empty(hx) && !is_empty(hy);
            }
            if (++spins > (1ll << 30)) {
              if (need && !got) {
                atomicOr(a.status, 2);
                hs->x = 0.0;
                hs->y = 0.0;
              }
              got = true;
            }
          }
          if (lane == 0) {
            const double2* h = s_hin + (m % kWsHRing) * kWsC;
#pragma unroll
            for (int tt = 0; tt < kWsC; ++tt)
              if (m < hchunks && m * kWsC + tt < nx) {
                hv[tt].x = ld_volatile_shared_f64(&h[tt].x);
                hv[tt].y = ld_volatile_shared_f64(&h[tt].y);
              }
          }
          __syncwarp();
          if (need) {  // free the slot: y first, x last (the poller tests x)
            *reinterpret_cast<volatile double*>(&hs->y) = empty;
            __threadfence_block();
            *reinterpret_cast<volatile double*>(&hs->x) = empty;
          }
        }
        // full-warp vote: lets the compiler prove convergence for the step
        // loop's shuffles (without it every shuffle gets a collective path)
        (void)__any_sync(kFull, true);
        WS_TRACE(0);
        mbar_wait_warp(&fac_full[st], u & 1u);
        WS_TRACE(1);
        const double2* fac = reinterpret_cast<const double2*>(fac_ring + st * kWsFacD) + lane;
        // Branch-free steps with the factors of step tt+1 loaded while step tt
        // computes.  Inactive lanes (skew padding / rows beyond ny) compute on
        // padding and store into the SK padding slots; their values never reach
        // an active lane (an inactive (lane, step) only feeds inactive ones)
        // and the x carry only advances on active steps.
        double2 fz[2], fk[8];
        auto load = [&](int tt, double2* z, double2* k) {
          const double2* f = fac + tt * kWsPairs * 32;  // double2 units
          z[0] = f[0]; z[1] = f[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) k[i] = f[64 + 32 * i];
        };
        load(0, fz, fk);
#pragma unroll
        for (int tt = 0; tt < kWsC; ++tt) {
          const int t = m * kWsC + tt;
          const int ip = t - lane;
          const bool act = row_ok && ip >= 0 && ip < nx;
          double2 nz[2], nk[8];
          if (tt + 1 < kWsC) load(tt + 1, nz, nk);
          // y-inflow: the strip below for lane 0, the lane below otherwise
          const double y0 = lane == 0 ? hv[tt].x : u0;
          const double y1 = lane == 0 ? hv[tt].y : u1;
          const double q0 = fma(fk[4].y, y1, fma(fk[4].x, y0, fma(fk[0].y, x1, fma(fk[0].x, x0, fz[0].x))));
          const double q1 = fma(fk[5].y, y1, fma(fk[5].x, y0, fma(fk[1].y, x1, fma(fk[1].x, x0, fz[0].y))));
          const double q2 = fma(fk[6].y, y1, fma(fk[6].x, y0, fma(fk[2].y, x1, fma(fk[2].x, x0, fz[1].x))));
          const double q3 = fma(fk[7].y, y1, fma(fk[7].x, y0, fma(fk[3].y, x1, fma(fk[3].x, x0, fz[1].y))));
          u0 = __shfl_up_sync(kFull, q2, 1);
          u1 = __shfl_up_sync(kFull, q3, 1);
          if (t < T) {  // steps past the slab's end would land in the next strip / slot
            double2* po = reinterpret_cast<double2*>(psi_p + (int64_t)t * 128);
            po[0] = make_double2(q0, q1);
            po[32] = make_double2(q2, q3);
          }
          if (lane == 31 && act && hout) __stcg(hout + ip, make_double2(q2, q3));
          x0 = act ? q1 : x0;
          x1 = act ? q3 : x1;
          if (tt + 1 < kWsC) {
            fz[0] = nz[0]; fz[1] = nz[1];
#pragma unroll
            for (int i = 0; i < 8; ++i) fk[i] = nk[i];
          }
        }
        __syncwarp();
        WS_TRACE(2);
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fac_empty[st])) : "memory");
        uses[st] = u + 1;
      }
    }
    __syncthreads();  // item done: every warp leaves the stage counters in step
    // producers and consumer advanced uses[] by the same amounts; nothing else
  }
}

int launch_sweep_ws(const SweepArgs& a, int max_ctas, cudaStream_t st) {
  int dev = 0, sms = 0, occ = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(sweep_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kWsSmem));
  DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_ws_kernel, kWsThreads,
                                                               kWsSmem));
  const int items = ((a.ny + 31) >> 5) * a.G;
  int ctas = items;
  const int cap = sms * (occ > 0 ? occ : 1);
  if (ctas > cap) ctas = cap;
  if (max_ctas > 0 && ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  sweep_ws_kernel<<<ctas, kWsThreads, kWsSmem, st>>>(a);
  DLRSN_CHECK_LAUNCH("sweep_ws_kernel");
  return DLRSN_OK;
}

}  // namespace dlrsn
