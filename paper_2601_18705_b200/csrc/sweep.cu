// K1: the upwind DG(Q1) transport sweep and its data movement.
//
// Restates transport_sn.py:142-163 (local operator), :303-322 (wavefront
// sweep), :403-407 (rhs), :419-438 (sweep_all + phi closure) for all swept
// directions at once.  Design:
//   * one warp = (direction group, 32-row strip); lane = row; the warp marches
//     the quadrant-oriented x axis with a one-column skew per lane, so the
//     x-upwind value stays in registers and the y-upwind value arrives by
//     __shfl_up_sync from the lane below one step earlier;
//   * data are stored in the sweep-native SK layout, so each warp-wide access
//     is one contiguous 512 B (double2 per lane) transaction;
//   * the strip above is fed through an L2 "handoff" column of self-flagging
//     slots (sNaN = empty); warps take work tickets in strip-major order, so
//     every wait targets a smaller, already-running ticket (deadlock-free
//     without co-residency assumptions);
//   * the 4x4 local operator A = sigma_t M + |wx| Gx' + |wy| Gy' is formed and
//     solved in registers per cell-angle (no stored inverses: the reference's
//     128 B/cell-angle cache is not materialised);
//   * the closure phi_g = sum_d cw_d psi_d of the warp's directions is
//     accumulated in registers (deterministic, no atomics).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sweep_common.cuh"

namespace dlrsn {

// Debug timeline (dlrsn_debug_trace): per (item, chunk) globaltimer before
// and after the handoff wait; null in production.
__device__ unsigned long long* g_trace = nullptr;
__device__ int g_trace_chunks = 0;
__device__ int g_flags = 0;  // debug: bit0 = no speculative handoff prefetch


// Steps per TMA chunk, pipeline depth and warps per CTA for a group width.
// (C steps per stage, P stages, WPC warps per CTA): measured on the config-2
// full-SN sweep (1024 directions, 280x280): double buffering with 4-warp CTAs
// keeps enough warps resident per SM; wider chunks or deeper rings lose
// occupancy to shared memory (scripts/full_sn.py).
// V selects a variant of the single-direction kernel (DLRSN_SWEEP1_CFG, tuning).
template <int DW, int V = 0> struct SweepCfg;
// DW = 1 (DLR steps, many strips): a 3-deep ring in 2-warp CTAs measured
// best on 1024^2 / 64 directions (1.48 vs 1.58 ms for 4-warp CTAs with a
// 2-deep ring; scripts/sweep_bench.py); variant 1 is the previous default
template <> struct SweepCfg<1, 0> { static constexpr int C = 4, P = 3, WPC = 2; };
template <> struct SweepCfg<1, 1> { static constexpr int C = 4, P = 2, WPC = 4; };
template <> struct SweepCfg<1, 2> { static constexpr int C = 8, P = 2, WPC = 2; };
template <> struct SweepCfg<1, 3> { static constexpr int C = 4, P = 4, WPC = 2; };
template <> struct SweepCfg<1, 4> { static constexpr int C = 4, P = 2, WPC = 2; };
template <> struct SweepCfg<1, 5> { static constexpr int C = 2, P = 6, WPC = 2; };
// smaller rings for more resident warps (16 / 12 per SM): measured slower on
// C4 (1.92-2.67 vs 1.58 ms): the prefetch depth matters more than occupancy
template <> struct SweepCfg<1, 6> { static constexpr int C = 2, P = 3, WPC = 2; };
template <> struct SweepCfg<1, 7> { static constexpr int C = 2, P = 4, WPC = 2; };
template <> struct SweepCfg<2, 0> { static constexpr int C = 4, P = 2, WPC = 4; };
template <> struct SweepCfg<4, 0> { static constexpr int C = 2, P = 2, WPC = 4; };
template <> struct SweepCfg<8, 0> { static constexpr int C = 1, P = 3, WPC = 2; };

template <int DW, int V = 0>
__host__ __device__ constexpr int stage_doubles() {
  return SweepCfg<DW, V>::C * (32 + 128 + 128 * DW);  // sigma | scat | rhs[DW]
}
template <int DW, int V = 0>
__host__ __device__ constexpr size_t sweep_smem_bytes() {
  return (size_t)SweepCfg<DW, V>::WPC * SweepCfg<DW, V>::P * stage_doubles<DW, V>() * sizeof(double);
}

// One persistent launch; see the file header.  Per warp, a P-deep ring of
// shared-memory stages is filled by TMA bulk copies (one elected lane, one
// mbarrier per stage): each stage holds C consecutive skewed steps of sigma_t,
// the scattering source and the DW direction rhs, all contiguous in the SK
// layout.  The y-inflow of lane 0 comes from the strip below through an L2
// handoff column whose slots start "empty" (sNaN sentinel): the producer
// stores, the consumer spins on the slot itself (no fences, no counters) and
// re-arms it after reading, so the buffer is clean for the next launch.
template <int DW, int V = 0>
__global__ void __launch_bounds__(SweepCfg<DW, V>::WPC * 32)
sweep_kernel(const SweepArgs a) {
  // iterations past convergence take no work item (no early return: that
  // would cost the compiler its proof that the warps stay converged)
  const bool skip = a.skip != nullptr && *a.skip != 0;
  constexpr int C = SweepCfg<DW, V>::C, P = SweepCfg<DW, V>::P, WPC = SweepCfg<DW, V>::WPC;
  constexpr int SD = stage_doubles<DW, V>();
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[WPC][P];
  __shared__ double s_S[WPC][DW][16];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double* ring = smem + (size_t)wib * P * SD;
  const int nx = a.nx, ny = a.ny, G = a.G;
  const int T = nx + 31;
  const int ns = (ny + 31) >> 5;
  const int items = ns * G;
  const int nchunks = (T + C - 1) / C;
  const int hchunks = (nx + C - 1) / C;
  const double empty = __longlong_as_double((long long)kEmpty);

  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < P; ++st) mbar_init(&bars[wib][st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t parity = 0;  // bit st: parity of the next completion of stage st

  for (;;) {
    int item = 0;
    if (lane == 0) {
      item = skip ? items : atomicAdd(a.ticket, 1);
      // every warp draws exactly one ticket past the end; the last of those
      // draws re-arms the counter for the next launch (no memset per launch)
      if (!skip && item == items + (int)(gridDim.x * blockDim.x / 32) - 1) atomicExch(a.ticket, 0);
    }
    item = __shfl_sync(kFull, item, 0);
    if (item >= items) break;
    const int s = item / G;
    const int g = item - s * G;
    const dlrsn_group* grp = a.groups + g;
    const int quad = grp->quad;
    const int nd = grp->ndir;

    __syncwarp();
    for (int e = lane; e < DW * 16; e += 32) {
      const int k = e >> 4, m = e & 15;
      s_S[wib][k][m] = k < nd ? grp->ox[k] * a.gxp[m] + grp->oy[k] * a.gyp[m] : 0.0;
    }
    const int64_t strip_vec = (int64_t)s * T * 128;  // SK offset of (s, t=0)
    double ox[DW], oy[DW], cw[DW];
    int64_t slot_off[DW], rhs_off[DW];
    const bool shared = a.rhs_shared != 0;
#pragma unroll
    for (int k = 0; k < DW; ++k) {
      const bool on = k < nd;
      ox[k] = on ? grp->ox[k] : 0.0;
      oy[k] = on ? grp->oy[k] : 0.0;
      cw[k] = on ? grp->cw[k] : 0.0;
      slot_off[k] = (on ? (int64_t)grp->slot[k] : 0) * a.vlen + strip_vec;
      rhs_off[k] = shared ? (int64_t)quad * a.vlen + strip_vec : slot_off[k];
    }
    const uint32_t nrhs = shared ? 1u : (uint32_t)nd;  // rhs slabs staged per chunk
    const double* sig = a.sigma_sk4 + (int64_t)quad * a.slen + (int64_t)s * T * 32;
    const double* scat = a.scat_sk4 ? a.scat_sk4 + (int64_t)quad * a.vlen + strip_vec : nullptr;
    double* phi_p = a.phi_sk ? a.phi_sk + (int64_t)g * a.vlen + strip_vec + 2 * lane : nullptr;
    __syncwarp();

    // TMA producer (lane 0 only): chunk m -> stage m % P.  Prologue: P-1 chunks.
    if (lane == 0) {
      for (int m = 0; m < P - 1 && m < nchunks; ++m) {
        const int st = m % P, t0 = m * C;
        const uint32_t n = (uint32_t)min(C, T - t0);
        double* buf = ring + st * SD;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[wib][st], n * (256u + (scat ? 1024u : 0u) + 1024u * nrhs));
        tma_load_1d(buf, sig + t0 * 32, n * 256u, &bars[wib][st]);
        if (scat) tma_load_1d(buf + C * 32, scat + t0 * 128, n * 1024u, &bars[wib][st]);
#pragma unroll
        for (int k = 0; k < DW; ++k)
          if (k < (int)nrhs)
            tma_load_1d(buf + C * 160 + k * C * 128, a.rhs_sk + rhs_off[k] + t0 * 128, n * 1024u,
                        &bars[wib][st]);
      }
    }

    const bool row_ok = (s << 5) + lane < ny;
    double2* hin = s > 0 ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)(s - 1) * G + g) * nx * DW
                         : nullptr;
    double2* hout = (s + 1 < ns) ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)s * G + g) * nx * DW
                                 : nullptr;
    // chunk h of the handoff: lane L < C*DW owns (column hC + L/DW, direction L%DW)
    const bool hlane = hin != nullptr && lane < C * DW;
    double2 h0 = make_double2(0.0, 0.0), h1 = h0, h2 = h0;
    const bool spec = (g_flags & 1) == 0;
    if (!spec) h0 = h1 = h2 = make_double2(empty, empty);
    if (spec && hlane && lane / DW < nx) h1 = __ldcg(hin + lane);
    if (spec && hlane && C + lane / DW < nx) h2 = __ldcg(hin + C * DW + lane);

    double xin[DW][2], yin[DW][2];
#pragma unroll
    for (int k = 0; k < DW; ++k) xin[k][0] = xin[k][1] = yin[k][0] = yin[k][1] = 0.0;

    for (int m = 0; m < nchunks; ++m) {
      if (g_trace && lane == 0 && m < g_trace_chunks) g_trace[((int64_t)item * g_trace_chunks + m) * 4] = gtimer();
      if (lane == 0 && m + P - 1 < nchunks) {
        const int mm = m + P - 1;
        const int st = mm % P, t0 = mm * C;
        const uint32_t n = (uint32_t)min(C, T - t0);
        double* buf = ring + st * SD;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[wib][st], n * (256u + (scat ? 1024u : 0u) + 1024u * nrhs));
        tma_load_1d(buf, sig + t0 * 32, n * 256u, &bars[wib][st]);
        if (scat) tma_load_1d(buf + C * 32, scat + t0 * 128, n * 1024u, &bars[wib][st]);
#pragma unroll
        for (int k = 0; k < DW; ++k)
          if (k < (int)nrhs)
            tma_load_1d(buf + C * 160 + k * C * 128, a.rhs_sk + rhs_off[k] + t0 * 128, n * 1024u,
                        &bars[wib][st]);
      }
      unsigned long long* tr = g_trace;
      if (tr && lane == 0 && m < g_trace_chunks) tr[((int64_t)item * g_trace_chunks + m) * 4 + 1] = gtimer();
      // y-inflow of lane 0 for this chunk's columns (strip below, via L2)
      h0 = h1;
      h1 = h2;
      {
        // Warp-uniform wait: every lane stays in the loop until all of this
        // chunk's slots have arrived (a divergent per-lane spin measurably
        // slowed the following compute 4x on sm_100a).
        const bool need = hlane && m < hchunks && m * C + lane / DW < nx;
        double2* slot = hin + (int64_t)m * C * DW + lane;
        int spins = 0;
        while (__any_sync(kFull, need && (is_empty(h0.x) || is_empty(h0.y)))) {
          __nanosleep(32);
          if (need && (is_empty(h0.x) || is_empty(h0.y))) h0 = __ldcv(slot);
          if (++spins > (1 << 26)) {  // report instead of hanging the GPU
            if (need) atomicOr(a.status, 2);
            h0 = make_double2(0.0, 0.0);
          }
        }
        if (need) __stcg(slot, make_double2(empty, empty));  // re-arm for the next launch
      }
      if (spec && hlane && m + 2 < hchunks && (m + 2) * C + lane / DW < nx)
        h2 = __ldcg(hin + (int64_t)(m + 2) * C * DW + lane);  // speculative prefetch
      if (tr && lane == 0 && m < g_trace_chunks) tr[((int64_t)item * g_trace_chunks + m) * 4 + 2] = gtimer();
      {
        const int st = m % P;
        mbar_wait_warp(&bars[wib][st], (parity >> st) & 1u);
        parity ^= 1u << st;
      }
      __syncwarp();
      if (tr && lane == 0 && m < g_trace_chunks) tr[((int64_t)item * g_trace_chunks + m) * 4 + 3] = gtimer();
      const double* buf = ring + (m % P) * SD;

#pragma unroll
      for (int tt = 0; tt < C; ++tt) {
        const int t = m * C + tt;
        const int ip = t - lane;
        // t >= T implies ip >= nx, so inactive lanes cover the tail chunk
        const bool act = row_ok && ip >= 0 && ip < nx;
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          const double y0 = __shfl_sync(kFull, h0.x, tt * DW + k);
          const double y1 = __shfl_sync(kFull, h0.y, tt * DW + k);
          if (lane == 0 && hin != nullptr && (g_flags & 2) == 0) { yin[k][0] = y0; yin[k][1] = y1; }
        }
        double ytop[DW][2];
#pragma unroll
        for (int k = 0; k < DW; ++k) ytop[k][0] = ytop[k][1] = 0.0;
        if (act) {
          const double sigma = buf[tt * 32 + lane];
          double sc[4] = {0.0, 0.0, 0.0, 0.0};
          if (scat) {
            const double2 u = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128)[lane];
            const double2 v = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128 + 64)[lane];
            sc[0] = u.x; sc[1] = u.y; sc[2] = v.x; sc[3] = v.y;
          }
          double ph[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int k = 0; k < DW; ++k) {
            if (k < nd) {
              const double* rb = buf + C * 160 + (shared ? 0 : k) * C * 128 + tt * 128;
              const double2 u = reinterpret_cast<const double2*>(rb)[lane];
              const double2 v = reinterpret_cast<const double2*>(rb + 64)[lane];
              double b[4] = {u.x + sc[0], u.y + sc[1], v.x + sc[2], v.y + sc[3]};
              // upwind couplings (transport_sn.py:312-320): x first, then y
              b[0] += ox[k] * (a.ex[0] * xin[k][0] + a.ex[1] * xin[k][1]);
              b[2] += ox[k] * (a.ex[2] * xin[k][0] + a.ex[3] * xin[k][1]);
              b[0] += oy[k] * (a.ey[0] * yin[k][0] + a.ey[1] * yin[k][1]);
              b[1] += oy[k] * (a.ey[2] * yin[k][0] + a.ey[3] * yin[k][1]);
              double A[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) A[q] = fma(sigma, a.mass[q], s_S[wib][k][q]);
              double x[4];
              solve4(A, b, x);
              if (a.psi_sk) {
                double2* po = reinterpret_cast<double2*>(a.psi_sk + slot_off[k] + (int64_t)t * 128 + 2 * lane);
                po[0] = make_double2(x[0], x[1]);
                po[32] = make_double2(x[2], x[3]);
              }
              xin[k][0] = x[1]; xin[k][1] = x[3];
              ytop[k][0] = x[2]; ytop[k][1] = x[3];
              ph[0] += cw[k] * x[0]; ph[1] += cw[k] * x[1];
              ph[2] += cw[k] * x[2]; ph[3] += cw[k] * x[3];
            }
          }
          if (phi_p) {
            double2* pp = reinterpret_cast<double2*>(phi_p + (int64_t)t * 128);
            pp[0] = make_double2(ph[0], ph[1]);
            pp[32] = make_double2(ph[2], ph[3]);
          }
          if (a.phi_atomic) {  // canonical cell and dof order of this lane-step
            const int ic = (quad & 1) ? nx - 1 - ip : ip;
            const int jo = (s << 5) + lane;
            const int jc = (quad & 2) ? ny - 1 - jo : jo;
            double* pa = a.phi_atomic + 4 * ((int64_t)jc * nx + ic);
            const int f = sk_flip(quad);
#pragma unroll
            for (int l = 0; l < 4; ++l) atomicAdd(pa + (l ^ f), ph[l]);
          }
          if (lane == 31 && hout) {
            double2* ho = hout + (int64_t)ip * DW;
#pragma unroll
            for (int k = 0; k < DW; ++k) __stcg(ho + k, make_double2(ytop[k][0], ytop[k][1]));
          }
        }
#pragma unroll
        for (int k = 0; k < DW; ++k) {
          const double y0 = __shfl_up_sync(kFull, ytop[k][0], 1);
          const double y1 = __shfl_up_sync(kFull, ytop[k][1], 1);
          if (lane > 0) { yin[k][0] = y0; yin[k][1] = y1; }
        }
      }
      __syncwarp();  // every lane is done with stage m % P before it is refilled
    }
  }
}


// ---- single-direction sweep, factorisation off the critical path ---------
// Same data flow as sweep_kernel<1> (TMA ring per warp, L2 strip handoff),
// but the per-step work is split by what it depends on:
//   phase 1 (independent across the chunk's C steps, ILP C): form A =
//     sigma_t M + S_omega, LU-factor it, and keep the factors plus the
//     source part of the rhs in registers -- all of it may run before the
//     strip below has delivered the chunk's inflow;
//   phase 2 (the dependent chain): add the upwind couplings to the rhs and
//     run the forward / back substitutions with pre-scaled factors: ~8
//     dependent FMAs per step instead of a whole factorisation (four
//     reciprocals) per step.
// Measured on C4 (1024^2, 64 directions): the chain-bound sweep_kernel<1>
// spent ~1200 cycles per warp-step ('wait' + handoff spin stalls).
struct Lu4 {
  double l1, l2, l3, m2, m3, n3;  // unit-lower multipliers
  double p0, p1, p2, p3;          // pivot reciprocals
  double u1, u2, u3, u6, u7, u11; // strictly upper part, row-scaled by its pivot reciprocal
  double b0, b1, b2, b3;          // source part of the rhs (rhs + scattering source)
};

template <int C, class SA>
__device__ __forceinline__ void lu4_factor(const SweepArgs& a, const SA& S, double sigma,
                                           Lu4& f) {
  double A[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) A[q] = fma(sigma, a.mass[q], S[q]);
  f.p0 = rcp64(A[0]);
  f.l1 = A[4] * f.p0; f.l2 = A[8] * f.p0; f.l3 = A[12] * f.p0;
  A[5] -= f.l1 * A[1]; A[6] -= f.l1 * A[2]; A[7] -= f.l1 * A[3];
  A[9] -= f.l2 * A[1]; A[10] -= f.l2 * A[2]; A[11] -= f.l2 * A[3];
  A[13] -= f.l3 * A[1]; A[14] -= f.l3 * A[2]; A[15] -= f.l3 * A[3];
  f.p1 = rcp64(A[5]);
  f.m2 = A[9] * f.p1; f.m3 = A[13] * f.p1;
  A[10] -= f.m2 * A[6]; A[11] -= f.m2 * A[7];
  A[14] -= f.m3 * A[6]; A[15] -= f.m3 * A[7];
  f.p2 = rcp64(A[10]);
  f.n3 = A[14] * f.p2;
  A[15] -= f.n3 * A[11];
  f.p3 = rcp64(A[15]);
  f.u1 = A[1] * f.p0; f.u2 = A[2] * f.p0; f.u3 = A[3] * f.p0;
  f.u6 = A[6] * f.p1; f.u7 = A[7] * f.p1;
  f.u11 = A[11] * f.p2;
}

// MINB > 1: that many CTAs per SM (registers capped accordingly), the
// direction's streaming operator S kept in shared memory instead of registers
template <int C, int P, int WPC, int MINB = 1>
__global__ void __launch_bounds__(WPC * 32, MINB)
sweep1s_kernel(const SweepArgs a) {
  const bool skip = a.skip != nullptr && *a.skip != 0;
  constexpr int SD = C * (32 + 128 + 128);  // doubles per stage: sigma | scat | rhs
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[WPC][P];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double* ring = smem + (size_t)wib * P * SD;
  const int nx = a.nx, ny = a.ny, G = a.G;
  const int T = nx + 31;
  const int ns = (ny + 31) >> 5;
  const int items = ns * G;
  const int nchunks = (T + C - 1) / C;
  const int hchunks = (nx + C - 1) / C;
  const double empty = __longlong_as_double((long long)kEmpty);
  const int flags = g_flags;  // debug bits, read once

  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < P; ++st) mbar_init(&bars[wib][st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t parity = 0;

  for (;;) {
    int item = 0;
    if (lane == 0) {
      item = skip ? items : atomicAdd(a.ticket, 1);
      if (!skip && item == items + (int)(gridDim.x * blockDim.x / 32) - 1) atomicExch(a.ticket, 0);
    }
    item = __shfl_sync(kFull, item, 0);
    if (item >= items) break;
    const int s = item / G;
    const int g = item - s * G;
    const dlrsn_group* grp = a.groups + g;
    const int quad = grp->quad;
    const double ox = grp->ox[0], oy = grp->oy[0], cw = grp->cw[0];
    double S_reg[MINB > 1 ? 1 : 16];
    __shared__ double s_S[WPC][16];
    if constexpr (MINB > 1) {
      __syncwarp();
      if (lane < 16) s_S[wib][lane] = ox * a.gxp[lane] + oy * a.gyp[lane];
      __syncwarp();
    } else {
#pragma unroll
      for (int m = 0; m < 16; ++m) S_reg[m] = ox * a.gxp[m] + oy * a.gyp[m];
    }
    const double cx0 = ox * a.ex[0], cx1 = ox * a.ex[1], cx2 = ox * a.ex[2], cx3 = ox * a.ex[3];
    const double cy0 = oy * a.ey[0], cy1 = oy * a.ey[1], cy2 = oy * a.ey[2], cy3 = oy * a.ey[3];
    const int64_t strip_vec = (int64_t)s * T * 128;
    const int64_t slot_off = (int64_t)grp->slot[0] * a.vlen + strip_vec;
    const double* sig = a.sigma_sk4 + (int64_t)quad * a.slen + (int64_t)s * T * 32;
    const double* scat = a.scat_sk4 ? a.scat_sk4 + (int64_t)quad * a.vlen + strip_vec : nullptr;
    const double* rhs = a.rhs_sk + slot_off;
    double* phi_p = a.phi_sk ? a.phi_sk + (int64_t)g * a.vlen + strip_vec + 2 * lane : nullptr;
    const uint32_t bytes_per_step = 256u + (scat ? 1024u : 0u) + 1024u;
    __syncwarp();

    auto issue = [&](int mm) {
      const int st = mm % P, t0 = mm * C;
      const uint32_t n = (uint32_t)min(C, T - t0);
      double* buf = ring + st * SD;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[wib][st], n * bytes_per_step);
      tma_load_1d(buf, sig + t0 * 32, n * 256u, &bars[wib][st]);
      if (scat) tma_load_1d(buf + C * 32, scat + t0 * 128, n * 1024u, &bars[wib][st]);
      tma_load_1d(buf + C * 160, rhs + t0 * 128, n * 1024u, &bars[wib][st]);
    };
    if (lane == 0)
      for (int m = 0; m < P - 1 && m < nchunks; ++m) issue(m);

    const bool row_ok = (s << 5) + lane < ny;
    double2* hin = s > 0 ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)(s - 1) * G + g) * nx
                         : nullptr;
    double2* hout = (s + 1 < ns) ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)s * G + g) * nx
                                 : nullptr;
    const bool hlane = hin != nullptr && lane < C;
    double2 h0 = make_double2(0.0, 0.0), h1 = h0, h2 = h0;
    const bool spec = (flags & 1) == 0;
    if (!spec) h0 = h1 = h2 = make_double2(empty, empty);
    if (spec && hlane && lane < nx) h1 = __ldcg(hin + lane);
    if (spec && hlane && C + lane < nx) h2 = __ldcg(hin + C + lane);
    const bool take_y = lane == 0 && hin != nullptr && (flags & 2) == 0;

    double xin0 = 0.0, xin1 = 0.0, yin0 = 0.0, yin1 = 0.0;
    for (int m = 0; m < nchunks; ++m) {
      if (lane == 0 && m + P - 1 < nchunks) issue(m + P - 1);
      {
        const int st = m % P;
        mbar_wait_warp(&bars[wib][st], (parity >> st) & 1u);
        parity ^= 1u << st;
      }
      __syncwarp();
      const double* buf = ring + (m % P) * SD;
      // phase 1: factors and source rhs of the chunk's C steps
      Lu4 f[C];
#pragma unroll
      for (int tt = 0; tt < C; ++tt) {
        const double sigma = buf[tt * 32 + lane];
        const double2 u = reinterpret_cast<const double2*>(buf + C * 160 + tt * 128)[lane];
        const double2 v = reinterpret_cast<const double2*>(buf + C * 160 + tt * 128 + 64)[lane];
        f[tt].b0 = u.x; f[tt].b1 = u.y; f[tt].b2 = v.x; f[tt].b3 = v.y;
        if (scat) {
          const double2 su = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128)[lane];
          const double2 sv = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128 + 64)[lane];
          f[tt].b0 += su.x; f[tt].b1 += su.y; f[tt].b2 += sv.x; f[tt].b3 += sv.y;
        }
        if constexpr (MINB > 1)
          lu4_factor<C>(a, s_S[wib], sigma, f[tt]);
        else
          lu4_factor<C>(a, S_reg, sigma, f[tt]);
      }
      __syncwarp();  // every lane has read stage m % P before it is refilled
      // the chunk's y-inflow of lane 0 (strip below, via L2)
      h0 = h1;
      h1 = h2;
      {
        const bool need = hlane && m < hchunks && m * C + lane < nx;
        double2* slot = hin + (int64_t)m * C + lane;
        int spins = 0;
        while (__any_sync(kFull, need && (is_empty(h0.x) || is_empty(h0.y)))) {
          __nanosleep(32);
          if (need && (is_empty(h0.x) || is_empty(h0.y))) h0 = __ldcv(slot);
          if (++spins > (1 << 26)) {
            if (need) atomicOr(a.status, 2);
            h0 = make_double2(0.0, 0.0);
          }
        }
        if (need) __stcg(slot, make_double2(empty, empty));
      }
      if (spec && hlane && m + 2 < hchunks && (m + 2) * C + lane < nx)
        h2 = __ldcg(hin + (int64_t)(m + 2) * C + lane);
      // phase 2: the dependent chain
#pragma unroll
      for (int tt = 0; tt < C; ++tt) {
        const int t = m * C + tt;
        const int ip = t - lane;
        const bool act = row_ok && ip >= 0 && ip < nx;
        {
          const double y0 = __shfl_sync(kFull, h0.x, tt);
          const double y1 = __shfl_sync(kFull, h0.y, tt);
          if (take_y) { yin0 = y0; yin1 = y1; }
        }
        const Lu4& F = f[tt];
        const double v0 = fma(cy1, yin1, fma(cy0, yin0, fma(cx1, xin1, fma(cx0, xin0, F.b0))));
        const double v1 = fma(cy3, yin1, fma(cy2, yin0, F.b1));
        const double v2 = fma(cx3, xin1, fma(cx2, xin0, F.b2));
        const double y1 = fma(-F.l1, v0, v1);
        const double y2 = fma(-F.m2, y1, fma(-F.l2, v0, v2));
        const double y3 = fma(-F.n3, y2, fma(-F.m3, y1, fma(-F.l3, v0, F.b3)));
        const double x3 = y3 * F.p3;
        const double x2 = fma(-F.u11, x3, y2 * F.p2);
        const double x1 = fma(-F.u6, x2, fma(-F.u7, x3, y1 * F.p1));
        const double x0 = fma(-F.u1, x1, fma(-F.u2, x2, fma(-F.u3, x3, v0 * F.p0)));
        double yt0 = 0.0, yt1 = 0.0;
        if (act) {
          double2* po = reinterpret_cast<double2*>(a.psi_sk + slot_off + (int64_t)t * 128 + 2 * lane);
          po[0] = make_double2(x0, x1);
          po[32] = make_double2(x2, x3);
          xin0 = x1; xin1 = x3;
          yt0 = x2; yt1 = x3;
          if (phi_p) {
            double2* pp = reinterpret_cast<double2*>(phi_p + (int64_t)t * 128);
            pp[0] = make_double2(cw * x0, cw * x1);
            pp[32] = make_double2(cw * x2, cw * x3);
          }
          if (lane == 31 && hout) __stcg(hout + ip, make_double2(x2, x3));
        }
        const double u0 = __shfl_up_sync(kFull, yt0, 1);
        const double u1 = __shfl_up_sync(kFull, yt1, 1);
        if (lane > 0) { yin0 = u0; yin1 = u1; }
      }
    }
  }
}

template <int C, int P, int WPC, int MINB = 1>
int launch_sweep1s(const SweepArgs& a, int max_ctas, cudaStream_t st) {
  constexpr size_t smem = (size_t)WPC * P * C * (32 + 128 + 128) * sizeof(double);
  int dev = 0, sms = 0, occ = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(sweep1s_kernel<C, P, WPC, MINB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep1s_kernel<C, P, WPC, MINB>,
                                                               WPC * 32, smem));
  const int items = sk_strips(a.ny) * a.G;
  int ctas = (items + WPC - 1) / WPC;
  const int cap = sms * (occ > 0 ? occ : 1);
  if (ctas > cap) ctas = cap;
  if (max_ctas > 0 && ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  sweep1s_kernel<C, P, WPC, MINB><<<ctas, WPC * 32, smem, st>>>(a);
  DLRSN_CHECK_LAUNCH("sweep1s_kernel");
  return DLRSN_OK;
}

// ---- grouped single-direction sweep with the closure fused --------------
// One CTA = up to WPC directions of ONE quadrant on one 32-row strip, a warp
// per direction, in lock step chunk by chunk: sigma_t and the scattering
// source are staged once per CTA (they are per cell), each warp stages its
// own rhs; after the dependent chain each warp leaves cw_d psi_d of the
// chunk in shared memory and the CTA sums the group's directions in fixed
// warp order into the group's closure partial (SK layout of the quadrant).
// So the source iteration never re-reads psi for phi (the separate closure
// pass read every swept direction once per iteration), and the reduction
// order is fixed (deterministic).  One CTA barrier per chunk.
template <int C, int P, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1)
sweep1g_kernel(const SweepArgs a, const CgTable* __restrict__ tab, double* __restrict__ part) {
  const bool skip = a.skip != nullptr && *a.skip != 0;
  constexpr int SD = C * (32 + 128) + WPC * C * 128;  // sigma | scat | rhs x WPC
  extern __shared__ __align__(128) double smem[];
  double* ring = smem;                    // P x SD
  double* phibuf = smem + (size_t)P * SD;  // 2 x WPC x C*128
  __shared__ __align__(8) uint64_t bars[P];
  __shared__ int s_item, s_ncg;
  __shared__ int s_first[kMaxCg], s_count[kMaxCg], s_quad[kMaxCg];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nx = a.nx, ny = a.ny;
  const int T = nx + 31;
  const int ns = (ny + 31) >> 5;
  const int nchunks = (T + C - 1) / C;
  const int hchunks = (nx + C - 1) / C;
  const double empty = __longlong_as_double((long long)kEmpty);
  const int flags = g_flags;
  if (tid == 0) {
    s_ncg = tab->ncg;
#pragma unroll
    for (int st = 0; st < P; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int ncg = s_ncg;
  for (int c = tid; c < ncg; c += blockDim.x) {
    s_first[c] = tab->first[c];
    s_count[c] = tab->count[c];
    s_quad[c] = tab->quad[c];
  }
  const int items = ns * ncg;
  uint32_t parity = 0;
  int mm_total = 0;  // chunks consumed by this CTA (phibuf parity)
  for (;;) {
    __syncthreads();  // previous item fully reduced; tables loaded
    if (tid == 0) {
      int item = skip ? items : atomicAdd(a.ticket, 1);
      if (!skip && item == items + (int)gridDim.x - 1) atomicExch(a.ticket, 0);
      s_item = item;
    }
    __syncthreads();
    const int item = s_item;
    if (item >= items) break;
    const int s = item / ncg;
    const int c = item - s * ncg;
    const int quad = s_quad[c], first = s_first[c], count = s_count[c];
    const bool active = w < count;
    const int gi = first + (active ? w : 0);
    const dlrsn_group* grp = a.groups + gi;
    const double ox = grp->ox[0], oy = grp->oy[0], cw = active ? grp->cw[0] : 0.0;
    double S[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) S[m] = ox * a.gxp[m] + oy * a.gyp[m];
    const double cx0 = ox * a.ex[0], cx1 = ox * a.ex[1], cx2 = ox * a.ex[2], cx3 = ox * a.ex[3];
    const double cy0 = oy * a.ey[0], cy1 = oy * a.ey[1], cy2 = oy * a.ey[2], cy3 = oy * a.ey[3];
    const int64_t strip_vec = (int64_t)s * T * 128;
    const int64_t slot_off = (int64_t)grp->slot[0] * a.vlen + strip_vec;
    const double* sig = a.sigma_sk4 + (int64_t)quad * a.slen + (int64_t)s * T * 32;
    const double* scat = a.scat_sk4 ? a.scat_sk4 + (int64_t)quad * a.vlen + strip_vec : nullptr;
    double* pout = part + (int64_t)c * a.vlen + strip_vec;
    __shared__ int64_t s_off[WPC];  // rhs offsets of the group's directions
    if (lane == 0) s_off[w] = slot_off;
    __syncthreads();

    auto issue = [&](int mm) {  // thread 0
      const int st = mm % P, t0 = mm * C;
      const uint32_t n = (uint32_t)min(C, T - t0);
      double* buf = ring + st * SD;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[st], n * (256u + (scat ? 1024u : 0u) + 1024u * count));
      tma_load_1d(buf, sig + t0 * 32, n * 256u, &bars[st]);
      if (scat) tma_load_1d(buf + C * 32, scat + t0 * 128, n * 1024u, &bars[st]);
      for (int k = 0; k < count; ++k)
        tma_load_1d(buf + C * 160 + k * C * 128, a.rhs_sk + s_off[k] + t0 * 128, n * 1024u, &bars[st]);
    };
    if (tid == 0)
      for (int m = 0; m < P - 1 && m < nchunks; ++m) issue(m);

    const bool row_ok = (s << 5) + lane < ny;
    const int D = a.G;  // handoff columns: one per single-direction group
    double2* hin = (active && s > 0)
                       ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)(s - 1) * D + gi) * nx
                       : nullptr;
    double2* hout = (active && s + 1 < ns)
                        ? reinterpret_cast<double2*>(a.handoff) + ((int64_t)s * D + gi) * nx
                        : nullptr;
    const bool hlane = hin != nullptr && lane < C;
    double2 h0 = make_double2(0.0, 0.0), h1 = h0, h2 = h0;
    const bool spec = (flags & 1) == 0;
    if (!spec) h0 = h1 = h2 = make_double2(empty, empty);
    if (spec && hlane && lane < nx) h1 = __ldcg(hin + lane);
    if (spec && hlane && C + lane < nx) h2 = __ldcg(hin + C + lane);
    const bool take_y = lane == 0 && hin != nullptr && (flags & 2) == 0;

    double xin0 = 0.0, xin1 = 0.0, yin0 = 0.0, yin1 = 0.0;
    for (int m = 0; m < nchunks; ++m, ++mm_total) {
      // stage (m + P - 1) % P was last read in chunk m - 1's phase 1, which
      // every warp finished before that chunk's barrier
      if (tid == 0 && m + P - 1 < nchunks) issue(m + P - 1);
      {
        const int st = m % P;
        mbar_wait_warp(&bars[st], (parity >> st) & 1u);
        parity ^= 1u << st;
      }
      __syncwarp();
      const double* buf = ring + (m % P) * SD;
      double* pb = phibuf + (size_t)(mm_total & 1) * WPC * C * 128 + (size_t)w * C * 128;
      if (active) {
        Lu4 f[C];
#pragma unroll
        for (int tt = 0; tt < C; ++tt) {
          const double sigma = buf[tt * 32 + lane];
          const double2 u = reinterpret_cast<const double2*>(buf + C * 160 + w * C * 128 + tt * 128)[lane];
          const double2 v = reinterpret_cast<const double2*>(buf + C * 160 + w * C * 128 + tt * 128 + 64)[lane];
          f[tt].b0 = u.x; f[tt].b1 = u.y; f[tt].b2 = v.x; f[tt].b3 = v.y;
          if (scat) {
            const double2 su = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128)[lane];
            const double2 sv = reinterpret_cast<const double2*>(buf + C * 32 + tt * 128 + 64)[lane];
            f[tt].b0 += su.x; f[tt].b1 += su.y; f[tt].b2 += sv.x; f[tt].b3 += sv.y;
          }
          lu4_factor<C>(a, S, sigma, f[tt]);
        }
        h0 = h1;
        h1 = h2;
        {
          const bool need = hlane && m < hchunks && m * C + lane < nx;
          double2* slot = hin + (int64_t)m * C + lane;
          int spins = 0;
          while (__any_sync(kFull, need && (is_empty(h0.x) || is_empty(h0.y)))) {
            __nanosleep(32);
            if (need && (is_empty(h0.x) || is_empty(h0.y))) h0 = __ldcv(slot);
            if (++spins > (1 << 26)) {
              if (need) atomicOr(a.status, 2);
              h0 = make_double2(0.0, 0.0);
            }
          }
          if (need) __stcg(slot, make_double2(empty, empty));
        }
        if (spec && hlane && m + 2 < hchunks && (m + 2) * C + lane < nx)
          h2 = __ldcg(hin + (int64_t)(m + 2) * C + lane);
#pragma unroll
        for (int tt = 0; tt < C; ++tt) {
          const int t = m * C + tt;
          const int ip = t - lane;
          const bool act = row_ok && ip >= 0 && ip < nx;
          {
            const double y0 = __shfl_sync(kFull, h0.x, tt);
            const double y1 = __shfl_sync(kFull, h0.y, tt);
            if (take_y) { yin0 = y0; yin1 = y1; }
          }
          const Lu4& F = f[tt];
          const double v0 = fma(cy1, yin1, fma(cy0, yin0, fma(cx1, xin1, fma(cx0, xin0, F.b0))));
          const double v1 = fma(cy3, yin1, fma(cy2, yin0, F.b1));
          const double v2 = fma(cx3, xin1, fma(cx2, xin0, F.b2));
          const double y1 = fma(-F.l1, v0, v1);
          const double y2 = fma(-F.m2, y1, fma(-F.l2, v0, v2));
          const double y3 = fma(-F.n3, y2, fma(-F.m3, y1, fma(-F.l3, v0, F.b3)));
          const double x3 = y3 * F.p3;
          const double x2 = fma(-F.u11, x3, y2 * F.p2);
          const double x1 = fma(-F.u6, x2, fma(-F.u7, x3, y1 * F.p1));
          const double x0 = fma(-F.u1, x1, fma(-F.u2, x2, fma(-F.u3, x3, v0 * F.p0)));
          double yt0 = 0.0, yt1 = 0.0;
          double2 q0 = make_double2(0.0, 0.0), q1 = q0;
          if (act) {
            double2* po = reinterpret_cast<double2*>(a.psi_sk + slot_off + (int64_t)t * 128 + 2 * lane);
            po[0] = make_double2(x0, x1);
            po[32] = make_double2(x2, x3);
            xin0 = x1; xin1 = x3;
            yt0 = x2; yt1 = x3;
            q0 = make_double2(cw * x0, cw * x1);
            q1 = make_double2(cw * x2, cw * x3);
            if (lane == 31 && hout) __stcg(hout + ip, make_double2(x2, x3));
          }
          reinterpret_cast<double2*>(pb + tt * 128)[lane] = q0;
          reinterpret_cast<double2*>(pb + tt * 128 + 64)[lane] = q1;
          const double u0 = __shfl_up_sync(kFull, yt0, 1);
          const double u1 = __shfl_up_sync(kFull, yt1, 1);
          if (lane > 0) { yin0 = u0; yin1 = u1; }
        }
      }
      __syncthreads();  // the chunk's cw psi of every direction is in phibuf
      {
        // group closure partial: fixed warp order
        const double* pbase = phibuf + (size_t)(mm_total & 1) * WPC * C * 128;
        const int t0 = m * C;
        const int nvalid = min(C, T - t0) * 128;
        for (int e = tid; e < nvalid; e += WPC * 32) {
          double v = 0.0;
          for (int k = 0; k < count; ++k) v += pbase[(size_t)k * C * 128 + e];
          pout[(int64_t)t0 * 128 + e] = v;
        }
      }
    }
  }
}

template <int C, int P, int WPC>
int launch_sweep1g(const SweepArgs& a, const CgTable* tab, double* part, cudaStream_t st) {
  constexpr size_t smem =
      ((size_t)P * (C * (32 + 128) + WPC * C * 128) + 2 * (size_t)WPC * C * 128) * sizeof(double);
  int dev = 0, sms = 0, occ = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(sweep1g_kernel<C, P, WPC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep1g_kernel<C, P, WPC>,
                                                               WPC * 32, smem));
  // items = strips x groups (known on the device only): one persistent
  // wave, every CTA draws tickets until they run out
  int ctas = sms * (occ > 0 ? occ : 1);
  const int max_items = sk_strips(a.ny) * a.G;  // groups <= single directions
  if (ctas > max_items) ctas = max_items;
  if (ctas < 1) ctas = 1;
  sweep1g_kernel<C, P, WPC><<<ctas, WPC * 32, smem, st>>>(a, tab, part);
  DLRSN_CHECK_LAUNCH("sweep1g_kernel");
  return DLRSN_OK;
}

// quadrant-ordered single-direction groups -> CTA groups of <= wpc
// directions of one quadrant, sizes balanced within the quadrant; cg_quad /
// cg_w (dmax entries) describe the partial slabs to the closure pass
__global__ void cgroup_plan_kernel(int G, const dlrsn_group* __restrict__ groups, int wpc, int dmax,
                                   CgTable* __restrict__ tab, int* __restrict__ cg_quad,
                                   double* __restrict__ cg_w) {
  if (threadIdx.x != 0) return;
  int ncg = 0;
  int i = 0;
  while (i < G) {
    const int q = groups[i].quad;
    int j = i;
    while (j < G && groups[j].quad == q) ++j;
    const int n = j - i;
    const int k = (n + wpc - 1) / wpc;
    const int base = n / k, rem = n % k;
    int f = i;
    for (int c = 0; c < k && ncg < kMaxCg; ++c) {
      const int cnt = base + (c < rem ? 1 : 0);
      tab->first[ncg] = f;
      tab->count[ncg] = cnt;
      tab->quad[ncg] = q;
      f += cnt;
      ++ncg;
    }
    i = j;
  }
  tab->ncg = ncg;
  for (int c = 0; c < dmax; ++c) {
    cg_quad[c] = c < ncg ? tab->quad[c] : -1;
    cg_w[c] = 1.0;
  }
}

__global__ void fill_empty_kernel(double* p, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = __longlong_as_double((long long)kEmpty);
}

// ---- tiled canonical <-> SK transposes ----------------------------------------
// A block owns a canonical tile of 8 x 32 cells and walks the directions in
// chunks of 8.  The canonical side moves whole 64-byte runs (8 directions of
// one dof row); the SK side is written / read along the skewed diagonals of
// the tile in the direction's own orientation, so 8 consecutive threads touch
// 8 consecutive SK lanes of one step (128-byte runs) instead of 32 scattered
// 16-byte pieces.  The chunk is staged in shared memory as [dof][dir][cell].
constexpr int kTrI = 8, kTrJ = 32, kTrD = 8, kTrCells = kTrI * kTrJ;
constexpr int kTrS = kTrCells + 1;  // cell stride (conflict-free staging writes)
constexpr size_t kTrSmem = (size_t)4 * kTrD * kTrS * sizeof(double);

// e-th cell of the tile in diagonal order of the oriented local frame:
// diagonal t' = il + jl, lanes jl rising along a diagonal
__device__ __forceinline__ void tr_diag_cell(int e, int& il, int& jl) {
  // diagonals t' = 0..38 hold min(t'+1, 8, 39-t') cells; walk the counts
  int t = 0, base = 0;
  for (;; ++t) {
    const int lo = t - (kTrI - 1) > 0 ? t - (kTrI - 1) : 0;
    const int hi = t < kTrJ - 1 ? t : kTrJ - 1;
    const int cnt = hi - lo + 1;
    if (e < base + cnt) {
      jl = lo + (e - base);
      il = t - jl;
      return;
    }
    base += cnt;
  }
}

// Both transposes are software-pipelined over the 8-direction chunks: the
// next chunk's loads are issued into registers (16 x 16 B per thread) before
// the current chunk's store phase, so every thread keeps 256 B in flight.
__global__ void __launch_bounds__(256) rhs_build_tiled_kernel(
    int nx, int ny, int D, const int* __restrict__ quad, const double* __restrict__ q,
    double inv_cdt, const double* __restrict__ pt, int ldp, const double* __restrict__ ex, int lde,
    double* __restrict__ out, int64_t vlen, dlrsn_cellops ops) {
  extern __shared__ double tr_sm[];  // [4][kTrD][kTrS]
  const int i0 = blockIdx.x * kTrI, j0 = blockIdx.y * kTrJ;
  const int ti = min(kTrI, nx - i0), tj = min(kTrJ, ny - j0);
  const int T = nx + 31;
  int il, jl;
  tr_diag_cell(threadIdx.x, il, jl);
  // canonical loads: element e -> (cell, dof, direction pair), pairs fastest
  // (64-byte runs of 8 directions); pt rows 16-byte aligned (ldp even)
  constexpr int kLd = kTrCells * 4 * (kTrD / 2) / 256;  // 16 per thread
  double2 R[kLd];
  auto load = [&](int d0) {
    const int dn = min(kTrD, D - d0);
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int dp = e & 3, l = (e >> 2) & 3, cl = e >> 4;
      const int ci = cl & (kTrI - 1), cj = cl >> 3;
      double2 v = make_double2(0.0, 0.0);
      if (ci < ti && cj < tj && 2 * dp < dn) {
        const int64_t c = (int64_t)(j0 + cj) * nx + i0 + ci;
        const double* src = pt + (4 * c + l) * ldp + d0 + 2 * dp;
        if (2 * dp + 1 < dn) v = __ldg(reinterpret_cast<const double2*>(src));
        else v.x = __ldg(src);
      }
      R[u] = v;
    }
  };
  auto park = [&]() {
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int dp = e & 3, l = (e >> 2) & 3, cl = e >> 4;
      tr_sm[(l * kTrD + 2 * dp) * kTrS + cl] = R[u].x;
      tr_sm[(l * kTrD + 2 * dp + 1) * kTrS + cl] = R[u].y;
    }
  };
  if (pt) load(0);
  for (int d0 = 0; d0 < D; d0 += kTrD) {
    const int dn = min(kTrD, D - d0);
    if (pt) {
      park();
      __syncthreads();
      if (d0 + kTrD < D) load(d0 + kTrD);  // in flight during the stores below
    }
    for (int dd = 0; dd < dn; ++dd) {
      const int d = d0 + dd;
      const int qd = quad[d];
      // oriented local (il, jl) -> canonical local cell of this direction
      const int ci = (qd & 1) ? ti - 1 - il : il;
      const int cj = (qd & 2) ? tj - 1 - jl : jl;
      if (il < ti && jl < tj) {
        const int cl = cj * kTrI + ci;
        const int64_t c = (int64_t)(j0 + cj) * nx + i0 + ci;
        const double qc = q[c];
        double v[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) v[l] = qc * ops.src_row[l];
        if (pt) {
          double u[4];
#pragma unroll
          for (int l = 0; l < 4; ++l) u[l] = tr_sm[(l * kTrD + dd) * kTrS + cl];
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const double mu = ops.mass[4 * l] * u[0] + ops.mass[4 * l + 1] * u[1] +
                              ops.mass[4 * l + 2] * u[2] + ops.mass[4 * l + 3] * u[3];
            v[l] += inv_cdt * mu;
          }
        }
        if (ex) {
#pragma unroll
          for (int l = 0; l < 4; ++l) v[l] += ex[(4 * c + l) * lde + d];
        }
        const int f = sk_flip(qd);
        int s, t, lane;
        sk_locate(i0 + ci, j0 + cj, qd, nx, ny, s, t, lane);
        double2* o = reinterpret_cast<double2*>(out + (int64_t)d * vlen);
        o[sk_vec_off(T, s, t, 0, lane) >> 1] = make_double2(v[0 ^ f], v[1 ^ f]);
        o[sk_vec_off(T, s, t, 1, lane) >> 1] = make_double2(v[2 ^ f], v[3 ^ f]);
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) sk_to_canonical_tiled_kernel(
    int nx, int ny, int D, const int* __restrict__ quad, const double* __restrict__ sk,
    double* __restrict__ psi, int ld, int64_t vlen) {
  extern __shared__ double tr_sm[];  // [4][kTrD][kTrS]
  const int i0 = blockIdx.x * kTrI, j0 = blockIdx.y * kTrJ;
  const int ti = min(kTrI, nx - i0), tj = min(kTrJ, ny - j0);
  const int T = nx + 31;
  int il, jl;
  tr_diag_cell(threadIdx.x, il, jl);
  const bool in = il < ti && jl < tj;
  const bool al = ((reinterpret_cast<uintptr_t>(psi) & 15) == 0) && (ld & 1) == 0;
  // SK loads of this thread's cell: 2 x 16 B per direction of the chunk
  double2 A[kTrD], B[kTrD];
  auto load = [&](int d0) {
    const int dn = min(kTrD, D - d0);
#pragma unroll
    for (int dd = 0; dd < kTrD; ++dd) {
      A[dd] = B[dd] = make_double2(0.0, 0.0);
      if (in && dd < dn) {
        const int d = d0 + dd;
        const int qd = quad[d];
        const int ci = (qd & 1) ? ti - 1 - il : il;
        const int cj = (qd & 2) ? tj - 1 - jl : jl;
        int s, t, lane;
        sk_locate(i0 + ci, j0 + cj, qd, nx, ny, s, t, lane);
        const double* src = sk + (int64_t)d * vlen;
        A[dd] = __ldcs(reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 0, lane)));
        B[dd] = __ldcs(reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 1, lane)));
      }
    }
  };
  load(0);
  for (int d0 = 0; d0 < D; d0 += kTrD) {
    const int dn = min(kTrD, D - d0);
#pragma unroll
    for (int dd = 0; dd < kTrD; ++dd) {
      if (in && dd < dn) {
        const int qd = quad[d0 + dd];
        const int ci = (qd & 1) ? ti - 1 - il : il;
        const int cj = (qd & 2) ? tj - 1 - jl : jl;
        const int cl = cj * kTrI + ci;
        const int f = sk_flip(qd);
        const double o[4] = {A[dd].x, A[dd].y, B[dd].x, B[dd].y};
#pragma unroll
        for (int l = 0; l < 4; ++l) tr_sm[(l * kTrD + dd) * kTrS + cl] = o[l ^ f];
      }
    }
    __syncthreads();
    if (d0 + kTrD < D) load(d0 + kTrD);  // in flight during the stores below
    // canonical stores: (cell, dof, direction pair), 16 B each
    for (int e = threadIdx.x; e < kTrCells * 4 * (kTrD / 2); e += blockDim.x) {
      const int dp = e & 3, l = (e >> 2) & 3, cl = e >> 4;
      const int ci = cl & (kTrI - 1), cj = cl >> 3;
      if (ci < ti && cj < tj && 2 * dp < dn) {
        const int64_t c = (int64_t)(j0 + cj) * nx + i0 + ci;
        double* dst = psi + (4 * c + l) * ld + d0 + 2 * dp;
        const double v0 = tr_sm[(l * kTrD + 2 * dp) * kTrS + cl];
        if (2 * dp + 1 < dn && al) {
          *reinterpret_cast<double2*>(dst) = make_double2(v0, tr_sm[(l * kTrD + 2 * dp + 1) * kTrS + cl]);
        } else {
          dst[0] = v0;
          if (2 * dp + 1 < dn) dst[1] = tr_sm[(l * kTrD + 2 * dp + 1) * kTrS + cl];
        }
      }
    }
    __syncthreads();
  }
}

// rhs_sk[d] = source_vector(q) + inv_cdt M psi_time[:, d] + extra[:, d]
__global__ void rhs_build_kernel(int nx, int ny, int D, const int* __restrict__ quad,
                                 const double* __restrict__ q, double inv_cdt,
                                 const double* __restrict__ pt, int ldp,
                                 const double* __restrict__ ex, int lde, double* __restrict__ out,
                                 int64_t vlen, dlrsn_cellops ops) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)nx * ny * D;
  if (idx >= n) return;
  const int c = (int)(idx / D);
  const int d = (int)(idx - (int64_t)c * D);
  const double qc = q[c];
  double v[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) v[l] = qc * ops.src_row[l];
  if (pt) {
    double u[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) u[l] = pt[(int64_t)(4 * c + l) * ldp + d];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const double mu = ops.mass[4 * l] * u[0] + ops.mass[4 * l + 1] * u[1] +
                        ops.mass[4 * l + 2] * u[2] + ops.mass[4 * l + 3] * u[3];
      v[l] += inv_cdt * mu;
    }
  }
  if (ex) {
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] += ex[(int64_t)(4 * c + l) * lde + d];
  }
  const int qd = quad[d];
  const int f = sk_flip(qd);
  int s, t, lane;
  sk_locate(c % nx, c / nx, qd, nx, ny, s, t, lane);
  const int T = nx + 31;
  double2* o = reinterpret_cast<double2*>(out + (int64_t)d * vlen);
  o[sk_vec_off(T, s, t, 0, lane) >> 1] = make_double2(v[0 ^ f], v[1 ^ f]);
  o[sk_vec_off(T, s, t, 1, lane) >> 1] = make_double2(v[2 ^ f], v[3 ^ f]);
}

// ---- isotropic inflow boundary (BASELINE config 3) -------------------------
// The reference is vacuum-only (transport_sn.py:11-13: exterior state 0).  An
// isotropic inflow psi_b on a wall is the upwind face flux of a constant
// exterior state: the inflow coupling |omega.n| * e2 (transport_sn.py:219-224)
// applied to psi_b [1, 1], i.e. |omega.n| psi_b (e2 row sums) on the wall's
// two edge dofs of every wall cell.  Added to the sweep rhs of each direction
// (the reference's `extra_source` slot, transport_sn.py:406-407).  In the
// oriented SK frame the x-inflow wall is i' = 0 (oriented dofs 0', 2') and the
// y-inflow wall j' = 0 (dofs 0', 1').  Thread (d, k): k < ny is the x-wall cell
// of oriented row k (it also adds the y term of the corner cell), k >= ny the
// y-wall cell of oriented column k - ny > 0, so no two threads touch a cell.
__global__ void inflow_add_kernel(int nx, int ny, int D, const int* __restrict__ quad,
                                  const double* __restrict__ om, const int* __restrict__ map,
                                  Inflow4 inflow, double exs, double eys,
                                  double* __restrict__ rhs, int64_t vlen) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int K = nx + ny;
  if (idx >= (int64_t)K * D) return;
  const int d = (int)(idx / K);
  const int k = (int)(idx - (int64_t)d * K);
  const int qd = quad[d];
  const int row = map ? map[d] : d;
  const double bx = inflow.v[(qd & 1) ? 1 : 0];
  const double by = inflow.v[(qd & 2) ? 3 : 2];
  const double ax = fabs(om[3 * (int64_t)row]) * bx * exs;
  const double ay = fabs(om[3 * (int64_t)row + 1]) * by * eys;
  const int T = nx + 31;
  double2* o = reinterpret_cast<double2*>(rhs + (int64_t)d * vlen);
  if (k < ny) {  // oriented (i' = 0, j' = k)
    const int s = k >> 5, lane = k & 31, t = lane;
    double2 p0 = o[sk_vec_off(T, s, t, 0, lane) >> 1];
    double2 p1 = o[sk_vec_off(T, s, t, 1, lane) >> 1];
    p0.x += ax;
    p1.x += ax;
    if (k == 0) {
      p0.x += ay;
      p0.y += ay;
    }
    o[sk_vec_off(T, s, t, 0, lane) >> 1] = p0;
    o[sk_vec_off(T, s, t, 1, lane) >> 1] = p1;
  } else {  // oriented (i' = k - ny, j' = 0), i' > 0
    const int ip = k - ny;
    if (ip == 0) return;
    double2 p0 = o[sk_vec_off(T, 0, ip, 0, 0) >> 1];
    p0.x += ay;
    p0.y += ay;
    o[sk_vec_off(T, 0, ip, 0, 0) >> 1] = p0;
  }
}

// h[w][k] = sum over the cells of wall w of (e2 row sums) . X[edge dofs][k]:
// X^T of the unit inflow load of wall w (block (k, w)); walls without inflow
// get 0.  Fixed-order block reduction (deterministic).
__global__ void __launch_bounds__(256) inflow_project_kernel(int nx, int ny, int r,
                                                             const double* __restrict__ X,
                                                             int ldx, Inflow4 inflow,
                                                             dlrsn_cellops ops,
                                                             double* __restrict__ h) {
  const int k = blockIdx.x, w = blockIdx.y;
  __shared__ double red[8];
  double acc = 0.0;
  if (inflow.v[w] != 0.0) {
    const bool vert = w < 2;
    const int ncell = vert ? ny : nx;
    const double* e2 = vert ? ops.e2x : ops.e2y;
    const double g0 = e2[0] + e2[1], g1 = e2[2] + e2[3];
    // edge dofs (mesh.py:34-39): left (0,2) right (1,3) bottom (0,1) top (2,3)
    const int l0 = w == 0 ? 0 : w == 1 ? 1 : w == 2 ? 0 : 2;
    const int l1 = w == 0 ? 2 : w == 1 ? 3 : w == 2 ? 1 : 3;
    for (int m = threadIdx.x; m < ncell; m += blockDim.x) {
      const int i = vert ? (w == 0 ? 0 : nx - 1) : m;
      const int j = vert ? m : (w == 2 ? 0 : ny - 1);
      const int64_t c = (int64_t)j * nx + i;
      acc = fma(g0, X[(4 * c + l0) * ldx + k], acc);
      acc = fma(g1, X[(4 * c + l1) * ldx + k], acc);
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
    h[w * r + k] = s;
  }
}

__global__ void cells_to_sk4_kernel(int nx, int ny, const double* __restrict__ v,
                                    double* __restrict__ out, int64_t slen) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nx * ny) return;
  const double x = v[c];
  const int T = nx + 31;
#pragma unroll
  for (int qd = 0; qd < 4; ++qd) {
    int s, t, lane;
    sk_locate(c % nx, c / nx, qd, nx, ny, s, t, lane);
    out[qd * slen + sk_sc_off(T, s, t, lane)] = x;
  }
}

__device__ inline void write_scat4(const dlrsn_cellops& ops, int c, const double* phi_c,
                                   double ss, double* scat, int64_t vlen) {
  // transport_sn.py:436: M (sigma_s phi) / 4 pi
  double u[4], w[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) u[l] = ss * phi_c[l];
#pragma unroll
  for (int l = 0; l < 4; ++l)
    w[l] = (ops.mass[4 * l] * u[0] + ops.mass[4 * l + 1] * u[1] + ops.mass[4 * l + 2] * u[2] +
            ops.mass[4 * l + 3] * u[3]) / kFourPi;
  const int nx = ops.nx, ny = ops.ny, T = nx + 31;
#pragma unroll
  for (int qd = 0; qd < 4; ++qd) {
    int s, t, lane;
    sk_locate(c % nx, c / nx, qd, nx, ny, s, t, lane);
    const int f = sk_flip(qd);
    double2* o = reinterpret_cast<double2*>(scat + qd * vlen);
    o[sk_vec_off(T, s, t, 0, lane) >> 1] = make_double2(w[0 ^ f], w[1 ^ f]);
    o[sk_vec_off(T, s, t, 1, lane) >> 1] = make_double2(w[2 ^ f], w[3 ^ f]);
  }
}

// The next iteration's scattering source M (sigma_s phi) / 4 pi in the 4
// quadrant SK slabs, written in SK order: thread = one SK element (strip,
// step, lane) of quadrant blockIdx.y, so a warp stores two contiguous 512-byte
// runs (writing by cell scatters 16-byte pieces over the 4 slabs: half-written
// sectors).  phi is read by cell (one 32-byte sector, from L2
// for the quadrants after the first).  Skipped once the iteration converged.
__global__ void __launch_bounds__(256) scat_quadrant_kernel(dlrsn_cellops ops,
                                                            const double* __restrict__ phi,
                                                            const double* __restrict__ ss,
                                                            double* __restrict__ scat, int64_t vlen,
                                                            const SiCtl* ctl) {
  if (ctl != nullptr && ctl->done != 0) return;
  const int nx = ops.nx, ny = ops.ny, T = nx + 31;
  const int qd = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (s, t, lane)
  const int lane = (int)(e & 31);
  const int64_t st = e >> 5;
  const int s = (int)(st / T), t = (int)(st - (int64_t)s * T);
  const int ip = t - lane, jp = 32 * s + lane;
  if (jp >= ny || ip < 0 || ip >= nx) return;
  const int i = (qd & 1) ? nx - 1 - ip : ip;
  const int j = (qd & 2) ? ny - 1 - jp : jp;
  const int64_t c = (int64_t)j * nx + i;
  const double2 a = __ldg(reinterpret_cast<const double2*>(phi) + 2 * c);
  const double2 b = __ldg(reinterpret_cast<const double2*>(phi) + 2 * c + 1);
  const double sg = __ldg(ss + c);
  const double u[4] = {sg * a.x, sg * a.y, sg * b.x, sg * b.y};
  double w[4];
#pragma unroll
  for (int l = 0; l < 4; ++l)
    w[l] = (ops.mass[4 * l] * u[0] + ops.mass[4 * l + 1] * u[1] + ops.mass[4 * l + 2] * u[2] +
            ops.mass[4 * l + 3] * u[3]) / kFourPi;
  const int f = sk_flip(qd);
  double2* o = reinterpret_cast<double2*>(scat + qd * vlen);
  o[sk_vec_off(T, s, t, 0, lane) >> 1] = make_double2(w[0 ^ f], w[1 ^ f]);
  o[sk_vec_off(T, s, t, 1, lane) >> 1] = make_double2(w[2 ^ f], w[3 ^ f]);
}

// *any |= (some v[i] != 0)  (the pure-absorber test of transport_sn.py:410)
__global__ void any_nonzero_kernel(int n, const double* __restrict__ v, int* any) {
  int nz = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (v[i] != 0.0) nz = 1;
  if (__any_sync(kFull, nz) && (threadIdx.x & 31) == 0) atomicOr(any, 1);
}

static int scat_quadrant_launch(const dlrsn_cellops* ops, const double* phi, const double* sigma_s,
                                double* scat_sk4, const SiCtl* ctl, cudaStream_t st) {
  const int nx = ops->nx, ny = ops->ny, ns = (ny + 31) / 32;
  const int64_t elems = (int64_t)ns * (nx + 31) * 32;
  scat_quadrant_kernel<<<dim3((unsigned)((elems + 255) / 256), 4), 256, 0, st>>>(
      *ops, phi, sigma_s, scat_sk4, sk_vec_len(nx, ny), ctl);
  DLRSN_CHECK_LAUNCH("scat_quadrant_kernel");
  return DLRSN_OK;
}

// convergence test of transport_sn.py:430-447 on the device
__device__ void si_decide(SiCtl* ctl, const double* w, int it, double tol, const int* any_scat) {
  const double change = sqrt(w[0]) / fmax(sqrt(w[1]), 1e-300);
  ctl->change = change;
  ctl->last = it;
  if (change <= tol || (it == 1 && any_scat && *any_scat == 0)) {
    ctl->iters = it;
    __threadfence();
    ctl->done = 1;
  }
}

__global__ void phi_combine_kernel(dlrsn_cellops ops, int G, const dlrsn_group* __restrict__ groups,
                                   const double* __restrict__ part, const double* __restrict__ psi,
                                   const double* __restrict__ phi_old,
                                   const double* __restrict__ ss, double* __restrict__ phi_new,
                                   double* __restrict__ scat, int64_t vlen, double* norms,
                                   double* partials, unsigned* counter, SiCtl* ctl, int it,
                                   double tol, const int* any_scat) {
  __shared__ double red[64];
  __shared__ bool last;
  if (ctl && ctl->done) return;
  const int nx = ops.nx, ny = ops.ny, T = nx + 31;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (c < nx * ny) {
    double p[4] = {0.0, 0.0, 0.0, 0.0};
    for (int g = 0; g < G; ++g) {
      const int qd = groups[g].quad;
      int s, t, lane;
      sk_locate(c % nx, c / nx, qd, nx, ny, s, t, lane);
      const int f = sk_flip(qd);
      if (part) {
        const double* src = part + (int64_t)g * vlen;
        const double2 a = *reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 0, lane));
        const double2 b = *reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 1, lane));
        const double o[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int l = 0; l < 4; ++l) p[l] += o[l ^ f];
      } else {
        // no per-group partials: closure straight from the swept psi
        const int nd = groups[g].ndir;
        for (int k = 0; k < nd; ++k) {
          const double* src = psi + (int64_t)groups[g].slot[k] * vlen;
          const double w = groups[g].cw[k];
          const double2 a = __ldcg(reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 0, lane)));
          const double2 b = __ldcg(reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 1, lane)));
          const double o[4] = {w * a.x, w * a.y, w * b.x, w * b.y};
#pragma unroll
          for (int l = 0; l < 4; ++l) p[l] += o[l ^ f];
        }
      }
    }
    const double2 oa = reinterpret_cast<const double2*>(phi_old)[2 * c];
    const double2 ob = reinterpret_cast<const double2*>(phi_old)[2 * c + 1];
    const double po[4] = {oa.x, oa.y, ob.x, ob.y};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const double dlt = p[l] - po[l];
      v[0] += dlt * dlt;
      v[1] += p[l] * p[l];
    }
    reinterpret_cast<double2*>(phi_new)[2 * c] = make_double2(p[0], p[1]);
    reinterpret_cast<double2*>(phi_new)[2 * c + 1] = make_double2(p[2], p[3]);
    if (scat) write_scat4(ops, c, p, ss[c], scat, vlen);
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = v[0];
    partials[2 * blockIdx.x + 1] = v[1];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    // fixed-order reduction of the per-block partials (deterministic)
    double w[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
      w[0] += __ldcg(partials + 2 * b);
      w[1] += __ldcg(partials + 2 * b + 1);
    }
    block_sum<2>(w, red);
    if (threadIdx.x == 0) {
      norms[0] = w[0];
      norms[1] = w[1];
      *counter = 0u;
      if (ctl && it > 0) si_decide(ctl, w, it, tol, any_scat);
    }
  }
}

// Closure flux of the one-call step in two coalesced passes.  Pass 1: for
// quadrant q (blockIdx.y), thread = one SK element (strip, step, lane) -- the
// same cell for every direction of that quadrant -- sums cw_k psi_k over the
// quadrant's slots in slot order (loads of 32 lanes contiguous) and writes
// the quadrant partial of that cell, canonical dofs, one 32-byte sector.
template <int UNR>
__global__ void __launch_bounds__(256) phi_quadrant_kernel(
    int nx, int ny, int D, const int* __restrict__ quads, const double* __restrict__ cw,
    const double* __restrict__ psi, int64_t vlen, double* __restrict__ phiq, int64_t nd,
    const SiCtl* ctl) {
  __shared__ int s_k[DLRSN_MAX_RANK];
  __shared__ double s_w[DLRSN_MAX_RANK];
  __shared__ int s_n;
  if (ctl != nullptr && ctl->done != 0) return;
  const int qd = blockIdx.y;
  if (threadIdx.x == 0) {
    int n = 0;
    for (int k = 0; k < D; ++k)
      if (quads[k] == qd) {
        s_k[n] = k;
        s_w[n] = cw[k];
        ++n;
      }
    s_n = n;
  }
  __syncthreads();
  const int n = s_n;
  const int T = nx + 31;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (s, t, lane)
  const int lane = (int)(e & 31);
  const int64_t st = e >> 5;
  const int s = (int)(st / T), t = (int)(st - (int64_t)s * T);
  const int ip = t - lane, jp = 32 * s + lane;
  if (jp >= ny || ip < 0 || ip >= nx) return;
  const int i = (qd & 1) ? nx - 1 - ip : ip;
  const int j = (qd & 2) ? ny - 1 - jp : jp;
  const int64_t off = sk_vec_off(T, s, t, 0, lane);
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  if (n > 0) {
    // batches of UNR directions: 2 UNR 16-byte loads in flight per thread,
    // then the sums in slot order
    int m = 0;
    for (; m + UNR <= n; m += UNR) {
      double2 a[UNR], b[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const double* src = psi + (int64_t)s_k[m + u] * vlen + off;
        a[u] = __ldcs(reinterpret_cast<const double2*>(src));
        b[u] = __ldcs(reinterpret_cast<const double2*>(src + 64));
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const double w = s_w[m + u];
        p[0] += w * a[u].x;
        p[1] += w * a[u].y;
        p[2] += w * b[u].x;
        p[3] += w * b[u].y;
      }
    }
    for (; m < n; ++m) {
      const double* src = psi + (int64_t)s_k[m] * vlen + off;
      const double2 a = __ldcs(reinterpret_cast<const double2*>(src));
      const double2 b = __ldcs(reinterpret_cast<const double2*>(src + 64));
      const double w = s_w[m];
      p[0] += w * a.x;
      p[1] += w * a.y;
      p[2] += w * b.x;
      p[3] += w * b.y;
    }
  }
  // oriented dof l is canonical dof l ^ quad
  const int f = sk_flip(qd);
  double o[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) o[l ^ f] = p[l];
  double2* dst = reinterpret_cast<double2*>(phiq + (int64_t)qd * nd + 4 * ((int64_t)j * nx + i));
  dst[0] = make_double2(o[0], o[1]);
  dst[1] = make_double2(o[2], o[3]);
}

// Pass 2: phi = ((q0 + q1) + q2) + q3 per dof; then the norms / scattering
// source / convergence decision of phi_combine_kernel (partial_out: write the
// rank-partial phi for the allreduce instead and stop).
__global__ void __launch_bounds__(256) phi_sum_kernel(
    dlrsn_cellops ops, const double* __restrict__ phiq, int64_t nd,
    const double* __restrict__ phi_old, const double* __restrict__ ss,
    double* __restrict__ phi_new, double* __restrict__ scat, int64_t vlen, double* norms,
    double* partials, unsigned* counter, SiCtl* ctl, int it, double tol, const int* any_scat,
    double* __restrict__ partial_out) {
  __shared__ double red[64];
  __shared__ bool last;
  if (ctl && ctl->done) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = c < ops.nx * ops.ny;
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  if (in) {
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
      const double2 a = __ldcg(reinterpret_cast<const double2*>(phiq + qd * nd) + 2 * c);
      const double2 b = __ldcg(reinterpret_cast<const double2*>(phiq + qd * nd) + 2 * c + 1);
      p[0] += a.x;
      p[1] += a.y;
      p[2] += b.x;
      p[3] += b.y;
    }
  }
  if (partial_out) {
    if (in) {
      reinterpret_cast<double2*>(partial_out)[2 * c] = make_double2(p[0], p[1]);
      reinterpret_cast<double2*>(partial_out)[2 * c + 1] = make_double2(p[2], p[3]);
    }
    return;
  }
  double v[2] = {0.0, 0.0};
  if (in) {
    const double2 oa = reinterpret_cast<const double2*>(phi_old)[2 * c];
    const double2 ob = reinterpret_cast<const double2*>(phi_old)[2 * c + 1];
    const double po[4] = {oa.x, oa.y, ob.x, ob.y};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const double dlt = p[l] - po[l];
      v[0] += dlt * dlt;
      v[1] += p[l] * p[l];
    }
    reinterpret_cast<double2*>(phi_new)[2 * c] = make_double2(p[0], p[1]);
    reinterpret_cast<double2*>(phi_new)[2 * c + 1] = make_double2(p[2], p[3]);
    if (scat) write_scat4(ops, c, p, ss[c], scat, vlen);
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = v[0];
    partials[2 * blockIdx.x + 1] = v[1];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    double w[2] = {0.0, 0.0};
    for (int b2 = threadIdx.x; b2 < (int)gridDim.x; b2 += blockDim.x) {
      w[0] += __ldcg(partials + 2 * b2);
      w[1] += __ldcg(partials + 2 * b2 + 1);
    }
    block_sum<2>(w, red);
    if (threadIdx.x == 0) {
      norms[0] = w[0];
      norms[1] = w[1];
      *counter = 0u;
      if (ctl && it > 0) si_decide(ctl, w, it, tol, any_scat);
    }
  }
}

// Sharded iteration: phi (canonical) already summed over ranks; compute the
// convergence norms against phi_old and the next scattering source.
__global__ void phi_finish_kernel(dlrsn_cellops ops, const double* __restrict__ phi_src,
                                  double* __restrict__ phi_dst,
                                  const double* __restrict__ phi_old,
                                  const double* __restrict__ ss, double* __restrict__ scat,
                                  int64_t vlen, double* norms, double* partials,
                                  unsigned* counter, SiCtl* ctl, int it, double tol,
                                  const int* any_scat) {
  __shared__ double red[64];
  __shared__ bool last;
  if (ctl && ctl->done) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (c < ops.nx * ops.ny) {
    double p[4], po[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      p[l] = phi_src[4 * c + l];
      if (phi_dst != phi_src) phi_dst[4 * c + l] = p[l];
      po[l] = phi_old[4 * c + l];
      const double d = p[l] - po[l];
      v[0] += d * d;
      v[1] += p[l] * p[l];
    }
    if (scat) write_scat4(ops, c, p, ss[c], scat, vlen);
  }
  block_sum<2>(v, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = v[0];
    partials[2 * blockIdx.x + 1] = v[1];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    double w[2] = {0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
      w[0] += __ldcg(partials + 2 * b);
      w[1] += __ldcg(partials + 2 * b + 1);
    }
    block_sum<2>(w, red);
    if (threadIdx.x == 0) {
      norms[0] = w[0];
      norms[1] = w[1];
      *counter = 0u;
      if (ctl && it > 0) si_decide(ctl, w, it, tol, any_scat);
    }
  }
}

__global__ void sk_to_canonical_kernel(int nx, int ny, int D, const int* __restrict__ quad,
                                       const double* __restrict__ sk, double* __restrict__ psi,
                                       int ld, int64_t vlen) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nx * ny * D) return;
  const int c = (int)(idx / D);
  const int d = (int)(idx - (int64_t)c * D);
  const int qd = quad[d];
  int s, t, lane;
  sk_locate(c % nx, c / nx, qd, nx, ny, s, t, lane);
  const int T = nx + 31;
  const double* src = sk + (int64_t)d * vlen;
  const double2 a = *reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 0, lane));
  const double2 b = *reinterpret_cast<const double2*>(src + sk_vec_off(T, s, t, 1, lane));
  const double o[4] = {a.x, a.y, b.x, b.y};
  const int f = sk_flip(qd);
#pragma unroll
  for (int l = 0; l < 4; ++l) psi[(int64_t)(4 * c + l) * ld + d] = o[l ^ f];
}

static int64_t handoff_offset_bytes(int, int, int) { return 256; }

// tiled canonical <-> SK transposes (DLRSN_TILED_TRANSPOSE=0: the
// thread-per-(cell, direction) kernels)
static bool tiled_transposes() {
  static const bool on = [] {
    const char* e = getenv("DLRSN_TILED_TRANSPOSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// configuration variant of the single-direction throughput kernel
static int sweep1_variant() {
  static const int v = [] {
    const char* e = getenv("DLRSN_SWEEP1_CFG");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int DW, int V = 0>
int launch_sweep(const SweepArgs& a, int max_ctas, cudaStream_t st) {
  constexpr int WPC = SweepCfg<DW, V>::WPC;
  constexpr size_t smem = sweep_smem_bytes<DW, V>();
  int dev = 0, sms = 0, occ = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  DLRSN_TRY_CUDA(cudaFuncSetAttribute(sweep_kernel<DW, V>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DLRSN_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_kernel<DW, V>, WPC * 32, smem));
  const int items = sk_strips(a.ny) * a.G;
  int ctas = (items + WPC - 1) / WPC;
  const int cap = sms * (occ > 0 ? occ : 1);
  if (ctas > cap) ctas = cap;
  if (max_ctas > 0 && ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  sweep_kernel<DW, V><<<ctas, WPC * 32, smem, st>>>(a);
  DLRSN_CHECK_LAUNCH("sweep_kernel");
  return DLRSN_OK;
}

}  // namespace dlrsn

using namespace dlrsn;

namespace dlrsn {

int phi_combine_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                       const double* phi_part_sk, const double* psi_sk, const double* phi_old,
                       const double* sigma_s, double* phi_new, double* scat_sk4, double* norms,
                       void* partial_ws, SiCtl* ctl, int it, double tol, const int* any_scat,
                       cudaStream_t st) {
  const int n = ops->nx * ops->ny;
  const int nb = (n + 255) / 256;
  unsigned* counter = reinterpret_cast<unsigned*>(partial_ws);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(partial_ws) + 256);
  DLRSN_REQUIRE(phi_part_sk || psi_sk, "phi_combine needs partials or psi");
  phi_combine_kernel<<<nb, 256, 0, st>>>(*ops, G, groups, phi_part_sk, psi_sk, phi_old, sigma_s,
                                         phi_new, scat_sk4, sk_vec_len(ops->nx, ops->ny), norms,
                                         partials, counter, ctl, it, tol, any_scat);
  DLRSN_CHECK_LAUNCH("phi_combine_kernel");
  return DLRSN_OK;
}

int phi_closure_launch(const dlrsn_cellops* ops, int D, const int* quads, const double* cw,
                       const double* psi_sk, double* phiq, const double* phi_old,
                       const double* sigma_s, double* phi_new, double* scat_sk4, double* norms,
                       void* partial_ws, SiCtl* ctl, int it, double tol, const int* any_scat,
                       double* partial_out, cudaStream_t st) {
  DLRSN_REQUIRE(D >= 1 && D <= DLRSN_MAX_RANK, "closure: 1..%d slots", DLRSN_MAX_RANK);
  const int nx = ops->nx, ny = ops->ny, ns = (ny + 31) / 32;
  const int64_t nd = 4 * (int64_t)nx * ny;
  const int64_t elems = (int64_t)ns * (nx + 31) * 32;
  static const int unr = getenv("DLRSN_PHIQ_UNR") ? atoi(getenv("DLRSN_PHIQ_UNR")) : 4;
  const dim3 gq((unsigned)((elems + 255) / 256), 4);
  if (unr >= 16)
    phi_quadrant_kernel<16><<<gq, 256, 0, st>>>(nx, ny, D, quads, cw, psi_sk, sk_vec_len(nx, ny), phiq, nd, ctl);
  else if (unr >= 8)
    phi_quadrant_kernel<8><<<gq, 256, 0, st>>>(nx, ny, D, quads, cw, psi_sk, sk_vec_len(nx, ny), phiq, nd, ctl);
  else
    phi_quadrant_kernel<4><<<gq, 256, 0, st>>>(nx, ny, D, quads, cw, psi_sk, sk_vec_len(nx, ny), phiq, nd, ctl);
  DLRSN_CHECK_LAUNCH("phi_quadrant_kernel");
  const int nb = (nx * ny + 255) / 256;
  unsigned* counter = reinterpret_cast<unsigned*>(partial_ws);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(partial_ws) + 256);
  phi_sum_kernel<<<nb, 256, 0, st>>>(*ops, phiq, nd, phi_old, sigma_s, phi_new, nullptr,
                                     sk_vec_len(nx, ny), norms, partials, counter, ctl, it, tol,
                                     any_scat, partial_out);
  DLRSN_CHECK_LAUNCH("phi_sum_kernel");
  // the next scattering source in SK order (skipped when this iteration converged)
  if (scat_sk4 && !partial_out) return scat_quadrant_launch(ops, phi_new, sigma_s, scat_sk4, ctl, st);
  return DLRSN_OK;
}

int phi_finish_launch(const dlrsn_cellops* ops, const double* phi_src, double* phi_dst,
                      const double* phi_old, const double* sigma_s, double* scat_sk4,
                      double* norms, void* partial_ws, SiCtl* ctl, int it, double tol,
                      const int* any_scat, cudaStream_t st) {
  const int n = ops->nx * ops->ny;
  const int nb = (n + 255) / 256;
  unsigned* counter = reinterpret_cast<unsigned*>(partial_ws);
  double* partials = reinterpret_cast<double*>(reinterpret_cast<char*>(partial_ws) + 256);
  phi_finish_kernel<<<nb, 256, 0, st>>>(*ops, phi_src, phi_dst, phi_old, sigma_s, nullptr,
                                        sk_vec_len(ops->nx, ops->ny), norms, partials, counter,
                                        ctl, it, tol, any_scat);
  DLRSN_CHECK_LAUNCH("phi_finish_kernel");
  if (scat_sk4) return scat_quadrant_launch(ops, phi_dst, sigma_s, scat_sk4, ctl, st);
  return DLRSN_OK;
}

}  // namespace dlrsn

extern "C" {

int64_t dlrsn_sweep_workspace_bytes(int nx, int ny, int n_groups, int dw) {
  return handoff_offset_bytes(nx, ny, n_groups) +
         (int64_t)sk_strips(ny) * n_groups * nx * dw * 2 * sizeof(double);
}

int dlrsn_rhs_build(const dlrsn_cellops* ops, int D, const int* quad, const double* q,
                    double inv_cdt, const double* psi_time, int ld_psi_time, const double* extra,
                    int ld_extra, double* rhs_sk, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(ops && D >= 0, "bad arguments to dlrsn_rhs_build");
  const int64_t n = (int64_t)ops->nx * ops->ny * D;
  if (n == 0) return DLRSN_OK;
  if (tiled_transposes() && (!psi_time || (((reinterpret_cast<uintptr_t>(psi_time) | (uintptr_t)ld_psi_time * 8) & 15) == 0))) {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(rhs_build_tiled_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrSmem));
    const dim3 grid((ops->nx + kTrI - 1) / kTrI, (ops->ny + kTrJ - 1) / kTrJ);
    rhs_build_tiled_kernel<<<grid, 256, kTrSmem, as_stream(stream)>>>(
        ops->nx, ops->ny, D, quad, q, inv_cdt, psi_time, ld_psi_time, extra, ld_extra, rhs_sk,
        sk_vec_len(ops->nx, ops->ny), *ops);
    DLRSN_CHECK_LAUNCH("rhs_build_tiled_kernel");
    return DLRSN_OK;
  }
  rhs_build_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      ops->nx, ops->ny, D, quad, q, inv_cdt, psi_time, ld_psi_time, extra, ld_extra, rhs_sk,
      sk_vec_len(ops->nx, ops->ny), *ops);
  DLRSN_CHECK_LAUNCH("rhs_build_kernel");
  return DLRSN_OK;
}

int dlrsn_inflow_add(const dlrsn_cellops* ops, int D, const int* quad, const double* omegas,
                     const int* map, const double* inflow, double* rhs_sk,
                     dlrsn_stream_t stream) {
  DLRSN_REQUIRE(ops && D >= 0 && inflow, "bad arguments to dlrsn_inflow_add");
  Inflow4 f;
  bool any = false;
  for (int w = 0; w < 4; ++w) {
    f.v[w] = inflow[w];
    any |= inflow[w] != 0.0;
  }
  const int64_t n = (int64_t)(ops->nx + ops->ny) * D;
  if (!any || n == 0) return DLRSN_OK;
  inflow_add_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      ops->nx, ops->ny, D, quad, omegas, map, f, ops->e2x[0] + ops->e2x[1],
      ops->e2y[0] + ops->e2y[1], rhs_sk, sk_vec_len(ops->nx, ops->ny));
  DLRSN_CHECK_LAUNCH("inflow_add_kernel");
  return DLRSN_OK;
}

int dlrsn_inflow_project(const dlrsn_cellops* ops, int r, const double* X, int ldx,
                         const double* inflow, double* h, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(ops && r > 0 && inflow, "bad arguments to dlrsn_inflow_project");
  Inflow4 f;
  for (int w = 0; w < 4; ++w) f.v[w] = inflow[w];
  inflow_project_kernel<<<dim3(r, 4), 256, 0, as_stream(stream)>>>(ops->nx, ops->ny, r, X, ldx,
                                                                    f, *ops, h);
  DLRSN_CHECK_LAUNCH("inflow_project_kernel");
  return DLRSN_OK;
}

int dlrsn_cells_to_sk4(const dlrsn_cellops* ops, const double* cell_values, double* out_sk4,
                       dlrsn_stream_t stream) {
  const int n = ops->nx * ops->ny;
  cells_to_sk4_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      ops->nx, ops->ny, cell_values, out_sk4, sk_scalar_len(ops->nx, ops->ny));
  DLRSN_CHECK_LAUNCH("cells_to_sk4_kernel");
  return DLRSN_OK;
}

int dlrsn_scatter_source(const dlrsn_cellops* ops, const double* phi, const double* sigma_s,
                         double* scat_sk4, int* any_scatter, dlrsn_stream_t stream) {
  const int n = ops->nx * ops->ny;
  // any_scatter from a scan of sigma_s, the slabs in SK order (coalesced)
  if (any_scatter) {
    const int nb = (n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024;
    any_nonzero_kernel<<<nb, 256, 0, as_stream(stream)>>>(
        n, sigma_s, any_scatter);
    DLRSN_CHECK_LAUNCH("any_nonzero_kernel");
  }
  return scat_quadrant_launch(ops, phi, sigma_s, scat_sk4, nullptr, as_stream(stream));
}

int dlrsn_phi_combine(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                      const double* phi_part_sk, const double* psi_sk, const double* phi_old,
                      const double* sigma_s,
                      double* phi_new, double* scat_sk4, double* norms, void* partial_ws,
                      dlrsn_stream_t stream) {
  return phi_combine_launch(ops, G, groups, phi_part_sk, psi_sk, phi_old, sigma_s, phi_new,
                            scat_sk4, norms, partial_ws, nullptr, 0, 0.0, nullptr,
                            as_stream(stream));
}

int dlrsn_phi_finish(const dlrsn_cellops* ops, const double* phi_new, const double* phi_old,
                     const double* sigma_s, double* scat_sk4, double* norms, void* partial_ws,
                     dlrsn_stream_t stream) {
  return phi_finish_launch(ops, phi_new, const_cast<double*>(phi_new), phi_old, sigma_s, scat_sk4,
                           norms, partial_ws, nullptr, 0, 0.0, nullptr, as_stream(stream));
}

int dlrsn_sk_to_canonical(const dlrsn_cellops* ops, int D, const int* quad, const double* psi_sk,
                          double* psi, int ld, dlrsn_stream_t stream) {
  const int64_t n = (int64_t)ops->nx * ops->ny * D;
  if (n == 0) return DLRSN_OK;
  if (tiled_transposes()) {
    DLRSN_TRY_CUDA(cudaFuncSetAttribute(sk_to_canonical_tiled_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTrSmem));
    const dim3 grid((ops->nx + kTrI - 1) / kTrI, (ops->ny + kTrJ - 1) / kTrJ);
    sk_to_canonical_tiled_kernel<<<grid, 256, kTrSmem, as_stream(stream)>>>(
        ops->nx, ops->ny, D, quad, psi_sk, psi, ld, sk_vec_len(ops->nx, ops->ny));
    DLRSN_CHECK_LAUNCH("sk_to_canonical_tiled_kernel");
    return DLRSN_OK;
  }
  sk_to_canonical_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      ops->nx, ops->ny, D, quad, psi_sk, psi, ld, sk_vec_len(ops->nx, ops->ny));
  DLRSN_CHECK_LAUNCH("sk_to_canonical_kernel");
  return DLRSN_OK;
}

int dlrsn_debug_flags(int flags) {
  DLRSN_TRY_CUDA(cudaMemcpyToSymbol(g_flags, &flags, sizeof(int)));
  return DLRSN_OK;
}

// optional CUDA-event timing of every sweep launch (bench.py roofline)
struct SweepTimer {
  cudaEvent_t start, stop;
  int G, dw;
};
static bool g_timing = false;
static std::vector<SweepTimer> g_timers;
static size_t g_timers_used = 0;
static SweepTimer* timer_slot(int G, int dw) {
  if (g_timers_used == g_timers.size()) {
    SweepTimer t;
    if (cudaEventCreate(&t.start) != cudaSuccess || cudaEventCreate(&t.stop) != cudaSuccess)
      return nullptr;
    g_timers.push_back(t);
  }
  SweepTimer* t = &g_timers[g_timers_used++];
  t->G = G;
  t->dw = dw;
  return t;
}

static unsigned long long* h_trace = nullptr;
static int h_trace_chunks = 0;

int dlrsn_debug_trace(unsigned long long* buf, int chunks) {
  h_trace = buf;
  h_trace_chunks = chunks;
  DLRSN_TRY_CUDA(cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)));
  DLRSN_TRY_CUDA(cudaMemcpyToSymbol(g_trace_chunks, &chunks, sizeof(int)));
  return DLRSN_OK;
}

int dlrsn_sweep_workspace_init(void* workspace, int64_t workspace_bytes, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(workspace && workspace_bytes >= 256, "sweep workspace too small");
  cudaStream_t st = as_stream(stream);
  DLRSN_TRY_CUDA(zero_async(workspace, 256, st));
  const int64_t n = (workspace_bytes - 256) / (int64_t)sizeof(double);
  if (n > 0) {
    fill_empty_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + 256), n);
    DLRSN_CHECK_LAUNCH("fill_empty_kernel");
  }
  return DLRSN_OK;
}

}  // extern "C"

namespace dlrsn {

static int sweep_launch_ex(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                           const double* sigma_t_sk4, const double* scat_sk4,
                           const double* rhs_sk, double* psi_sk, double* phi_part_sk,
                           void* workspace, int64_t workspace_bytes, int max_ctas,
                           const int* skip, int rhs_shared, double* phi_atomic, cudaStream_t st);

int sweep_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                 const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk,
                 double* psi_sk, double* phi_part_sk, void* workspace, int64_t workspace_bytes,
                 int max_ctas, const int* skip, cudaStream_t st) {
  DLRSN_REQUIRE(psi_sk, "null argument to dlrsn_sweep");
  return sweep_launch_ex(ops, G, groups, dw, sigma_t_sk4, scat_sk4, rhs_sk, psi_sk, phi_part_sk,
                         workspace, workspace_bytes, max_ctas, skip, 0, nullptr, st);
}

static int sweep_launch_ex(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                           const double* sigma_t_sk4, const double* scat_sk4,
                           const double* rhs_sk, double* psi_sk, double* phi_part_sk,
                           void* workspace, int64_t workspace_bytes, int max_ctas,
                           const int* skip, int rhs_shared, double* phi_atomic, cudaStream_t st) {
  DLRSN_REQUIRE(ops && groups && sigma_t_sk4 && rhs_sk && workspace && (psi_sk || phi_atomic),
                "null argument to dlrsn_sweep");
  DLRSN_REQUIRE(dw == 1 || dw == 2 || dw == 4 || dw == 8, "sweep width must be 1, 2, 4 or 8");
  const int64_t need = dlrsn_sweep_workspace_bytes(ops->nx, ops->ny, G, dw);
  DLRSN_REQUIRE(workspace_bytes >= need, "sweep workspace too small (%lld < %lld)",
                (long long)workspace_bytes, (long long)need);
  if (G == 0) return DLRSN_OK;
  const int64_t head = handoff_offset_bytes(ops->nx, ops->ny, G);
  // the work ticket is re-armed by the last draw of every launch (the
  // workspace starts zeroed: dlrsn_sweep_workspace_init)
  SweepArgs a;
  a.nx = ops->nx; a.ny = ops->ny; a.G = G;
  a.groups = groups;
  a.sigma_sk4 = sigma_t_sk4;
  a.scat_sk4 = scat_sk4;
  a.rhs_sk = rhs_sk;
  a.psi_sk = psi_sk;
  a.phi_sk = phi_part_sk;
  a.ticket = reinterpret_cast<int*>(workspace);
  a.status = reinterpret_cast<int*>(workspace) + 1;
  a.handoff = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + head);
  for (int m = 0; m < 16; ++m) {
    a.mass[m] = ops->mass[m];
    a.gxp[m] = ops->gx[m];
    a.gyp[m] = ops->gy[m];
  }
  // outflow edge masses: right edge dofs (1,3), top edge dofs (2,3)
  const int ix[2] = {1, 3}, iy[2] = {2, 3};
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      a.gxp[4 * ix[r] + ix[c]] += ops->e2x[2 * r + c];
      a.gyp[4 * iy[r] + iy[c]] += ops->e2y[2 * r + c];
    }
  for (int m = 0; m < 4; ++m) {
    a.ex[m] = ops->e2x[m];
    a.ey[m] = ops->e2y[m];
  }
  a.vlen = sk_vec_len(ops->nx, ops->ny);
  a.slen = sk_scalar_len(ops->nx, ops->ny);
  a.trace = h_trace;
  a.trace_chunks = h_trace_chunks;
  a.skip = skip;
  a.rhs_shared = rhs_shared;
  a.phi_atomic = phi_atomic;
  {
    static const char* dbg = getenv("DLRSN_SWEEP_DEBUG");
    a.debug = dbg ? atoi(dbg) : 0;
  }
  // single-direction groups: the warp-specialised kernel when the work items
  // barely fill the GPU (latency-bound regime), the multi-warp kernel when
  // there are enough items to hide the per-step latency by occupancy
  static const char* ws_env = getenv("DLRSN_SWEEP_WS");
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int items = sk_strips(ops->ny) * G;
  // crossover measured on B200 (scripts/sweep_bench.py, configs.py): WS wins
  // at 512 items (C3: 0.41 vs 0.63 ms) and 1024 items (1.31 vs 1.39 ms), the
  // multi-warp kernel at 1152 items (1.05 vs 1.13 ms) and 2048 (C4: 1.59 vs 2.57)
  bool use_ws = items <= 4 * sms;
  if (ws_env) use_ws = ws_env[0] == '1';
  if (phi_part_sk) use_ws = false;  // the warp-specialised kernel writes no closure partials
  if (rhs_shared || phi_atomic) use_ws = false;
  SweepTimer* tm = g_timing ? timer_slot(G, dw) : nullptr;
  if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->start, st));
  int rc;
  switch (dw) {
    case 1:
      if (use_ws) {
        rc = launch_sweep_ws(a, max_ctas, st);
        break;
      }
      if (rhs_shared || phi_atomic) {  // closure-only sweeps: the general kernel
        rc = launch_sweep<1, 0>(a, max_ctas, st);
        break;
      }
      switch (sweep1_variant()) {
        case 0: rc = launch_sweep1s<4, 3, 2>(a, max_ctas, st); break;
        case 10: rc = launch_sweep1s<2, 4, 2>(a, max_ctas, st); break;
        case 11: rc = launch_sweep1s<4, 2, 2>(a, max_ctas, st); break;
        case 12: rc = launch_sweep1s<2, 3, 4>(a, max_ctas, st); break;
        // 12 warps per SM (167 registers, S in shared memory): C4 1.46 vs
        // 1.32 ms, C5 29.9 vs 31.4 ms; 14-16 warps per SM (128 registers)
        // spill and run 2-3x slower
        case 15: rc = launch_sweep1s<2, 4, 2, 6>(a, max_ctas, st); break;
        case 9: rc = launch_sweep<1, 0>(a, max_ctas, st); break;
        case 1: rc = launch_sweep<1, 1>(a, max_ctas, st); break;
        case 2: rc = launch_sweep<1, 2>(a, max_ctas, st); break;
        case 3: rc = launch_sweep<1, 3>(a, max_ctas, st); break;
        case 4: rc = launch_sweep<1, 4>(a, max_ctas, st); break;
        case 5: rc = launch_sweep<1, 5>(a, max_ctas, st); break;
        case 6: rc = launch_sweep<1, 6>(a, max_ctas, st); break;
        case 7: rc = launch_sweep<1, 7>(a, max_ctas, st); break;
        default: rc = launch_sweep1s<4, 3, 2>(a, max_ctas, st); break;
      }
      break;
    case 2: rc = launch_sweep<2>(a, max_ctas, st); break;
    case 4: rc = launch_sweep<4>(a, max_ctas, st); break;
    default: rc = launch_sweep<8>(a, max_ctas, st); break;
  }
  if (tm && rc == DLRSN_OK) DLRSN_TRY_CUDA(cudaEventRecord(tm->stop, st));
  return rc;
}

// directions per CTA group of the grouped sweep (DLRSN_SWEEP_GROUP: 4 or 8;
// 0 = the ungrouped kernel + the separate closure pass).  Off by default:
// measured on C4 (1024^2, 64 directions) the lock step costs more than the
// closure pass it removes -- 32.0 (8 per group) / 32.5 ms (4) vs 30.0 ms
// per 4-iteration step: a CTA barrier per chunk keeps every warp of an SM in
// the same phase (all factorising, then all on the dependent chain), where
// independent warps overlap one's chain with another's factorisation.
int sweep_group_width() {
  static const int v = [] {
    const char* e = getenv("DLRSN_SWEEP_GROUP");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int cgroup_plan_launch(int G, const dlrsn_group* groups, int wpc, int dmax, CgTable* tab,
                       int* cg_quad, double* cg_w, cudaStream_t st) {
  cgroup_plan_kernel<<<1, 32, 0, st>>>(G, groups, wpc, dmax, tab, cg_quad, cg_w);
  DLRSN_CHECK_LAUNCH("cgroup_plan_kernel");
  return DLRSN_OK;
}

int sweep_grouped_launch(const dlrsn_cellops* ops, int G, const dlrsn_group* groups,
                         const CgTable* tab, const double* sigma_t_sk4, const double* scat_sk4,
                         const double* rhs_sk, double* psi_sk, double* part, void* workspace,
                         int64_t workspace_bytes, const int* skip, cudaStream_t st) {
  DLRSN_REQUIRE(ops && groups && tab && sigma_t_sk4 && rhs_sk && psi_sk && part && workspace,
                "null argument to the grouped sweep");
  const int64_t need = dlrsn_sweep_workspace_bytes(ops->nx, ops->ny, G, 1);
  DLRSN_REQUIRE(workspace_bytes >= need, "sweep workspace too small (%lld < %lld)",
                (long long)workspace_bytes, (long long)need);
  if (G == 0) return DLRSN_OK;
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.nx = ops->nx; a.ny = ops->ny; a.G = G;
  a.groups = groups;
  a.sigma_sk4 = sigma_t_sk4;
  a.scat_sk4 = scat_sk4;
  a.rhs_sk = rhs_sk;
  a.psi_sk = psi_sk;
  a.ticket = reinterpret_cast<int*>(workspace);
  a.status = reinterpret_cast<int*>(workspace) + 1;
  a.handoff = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) +
                                        handoff_offset_bytes(ops->nx, ops->ny, G));
  for (int m = 0; m < 16; ++m) {
    a.mass[m] = ops->mass[m];
    a.gxp[m] = ops->gx[m];
    a.gyp[m] = ops->gy[m];
  }
  const int ix[2] = {1, 3}, iy[2] = {2, 3};
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      a.gxp[4 * ix[r] + ix[c]] += ops->e2x[2 * r + c];
      a.gyp[4 * iy[r] + iy[c]] += ops->e2y[2 * r + c];
    }
  for (int m = 0; m < 4; ++m) {
    a.ex[m] = ops->e2x[m];
    a.ey[m] = ops->e2y[m];
  }
  a.vlen = sk_vec_len(ops->nx, ops->ny);
  a.slen = sk_scalar_len(ops->nx, ops->ny);
  a.skip = skip;
  SweepTimer* tm = g_timing ? timer_slot(G, 1) : nullptr;
  if (tm) DLRSN_TRY_CUDA(cudaEventRecord(tm->start, st));
  const int rc = sweep_group_width() == 4 ? launch_sweep1g<4, 3, 4>(a, tab, part, st)
                                          : launch_sweep1g<4, 3, 8>(a, tab, part, st);
  if (tm && rc == DLRSN_OK) DLRSN_TRY_CUDA(cudaEventRecord(tm->stop, st));
  return rc;
}

}  // namespace dlrsn

extern "C" {

int dlrsn_sweep_closure(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                        const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk4,
                        double* phi, void* workspace, int64_t workspace_bytes, int max_ctas,
                        dlrsn_stream_t stream) {
  DLRSN_REQUIRE(phi, "dlrsn_sweep_closure needs phi");
  return sweep_launch_ex(ops, G, groups, dw, sigma_t_sk4, scat_sk4, rhs_sk4, nullptr, nullptr,
                         workspace, workspace_bytes, max_ctas, nullptr, 1, phi, as_stream(stream));
}

int dlrsn_sweep(const dlrsn_cellops* ops, int G, const dlrsn_group* groups, int dw,
                const double* sigma_t_sk4, const double* scat_sk4, const double* rhs_sk,
                double* psi_sk, double* phi_part_sk, void* workspace, int64_t workspace_bytes,
                int max_ctas, dlrsn_stream_t stream) {
  return sweep_launch(ops, G, groups, dw, sigma_t_sk4, scat_sk4, rhs_sk, psi_sk, phi_part_sk,
                      workspace, workspace_bytes, max_ctas, nullptr, as_stream(stream));
}

}  // extern "C"

namespace dlrsn {
bool sweep_timing_enabled() { return g_timing; }
}  // namespace dlrsn

extern "C" {

int dlrsn_sweep_timing(int enable) {
  g_timing = enable != 0;
  g_timers_used = 0;
  return DLRSN_OK;
}

int dlrsn_sweep_timing_read(int cap, float* ms, int* groups, int* dw, int* count) {
  int n = 0;
  for (size_t k = 0; k < g_timers_used; ++k) {
    SweepTimer& t = g_timers[k];
    if (n < cap) {
      DLRSN_TRY_CUDA(cudaEventSynchronize(t.stop));
      DLRSN_TRY_CUDA(cudaEventElapsedTime(&ms[n], t.start, t.stop));
      groups[n] = t.G;
      dw[n] = t.dw;
    }
    ++n;
  }
  *count = n;
  return DLRSN_OK;
}

}  // extern "C"
