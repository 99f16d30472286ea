// K4: per-cell grey physics -- Newton linearisation and closed-form
// temperature update, fused into single HBM-bound elementwise passes.
// Restates physics.py:63-132 and driver.py:344-346,532-534.
#include <cmath>
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace dlrsn {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// planck (physics.py:63-75): B = (a c / 4pi) T^4, dB/dT = (a c / pi) T^3
__device__ inline void planck(double T, double scale, double& B, double& dB) {
  const double T2 = T * T;
  B = scale / kFourPi * (T2 * T2);
  dB = scale / kPi * (T2 * T);
}

__device__ inline void linearize_cell(double T0, double sa, double rc, double dt, double c,
                                      double a_r, double ssp, double qe, double& sigma_t,
                                      double& sigma_s, double& q, double& denom, int& bad) {
  if (!(T0 >= 0.0) || !(sa >= 0.0) || !(rc > 0.0)) bad = 1;
  double B, dB;
  planck(T0, a_r * c, B, dB);
  const double em = kFourPi * dt * sa * dB;
  denom = rc + em;
  sigma_s = sa * em / denom + ssp;
  q = sa * B * rc / denom + qe;
  sigma_t = sa + 1.0 / (c * dt) + ssp;
}

__global__ void linearize_kernel(int n, const double* __restrict__ T0,
                                 const double* __restrict__ sa, const double* __restrict__ rc,
                                 double dt, double c, double a_r, const double* __restrict__ ssp,
                                 const double* __restrict__ qe, double* __restrict__ st,
                                 double* __restrict__ ss, double* __restrict__ q,
                                 double* __restrict__ den, int* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int bad = 0;
  linearize_cell(T0[i], sa[i], rc[i], dt, c, a_r, ssp ? ssp[i] : 0.0, qe ? qe[i] : 0.0, st[i],
                 ss[i], q[i], den[i], bad);
  if (bad && status) atomicOr(status, 1);
}

__device__ inline double cell_mean4(const double* p, int i) {
  // dofs_to_cells: numpy mean over the 4 dofs (sequential add, then /4)
  const double2 a = reinterpret_cast<const double2*>(p)[2 * i];
  const double2 b = reinterpret_cast<const double2*>(p)[2 * i + 1];
  return (((a.x + a.y) + b.x) + b.y) / 4.0;
}

__device__ inline double new_temperature(double phi, double T0, double sa, double den, double dt,
                                         double c, double a_r, double t_floor) {
  double B0, dB;
  planck(T0, a_r * c, B0, dB);
  const double T = T0 + dt * sa * (phi - kFourPi * B0) / den;
  return fmax(T, t_floor);
}

__global__ void update_temperature_kernel(int n, const double* __restrict__ phi, int per_dof,
                                          const double* __restrict__ T0,
                                          const double* __restrict__ sa,
                                          const double* __restrict__ den, double dt, double c,
                                          double a_r, double t_floor, double* __restrict__ T) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double p = per_dof ? cell_mean4(phi, i) : phi[i];
  T[i] = new_temperature(p, T0[i], sa[i], den[i], dt, c, a_r, t_floor);
}

__global__ void advance_kernel(int n, const double* __restrict__ phi, const double* T_in,
                               double* T, const double* sa_in, const double* den_in, double* sa,
                               const double* __restrict__ sa0,
                               double power, const double* __restrict__ rc, double dt, double c,
                               double a_r, double t_floor, const double* __restrict__ ssp,
                               const double* __restrict__ qe, double* __restrict__ st,
                               double* __restrict__ ss, double* __restrict__ q,
                               double* den, double* __restrict__ T0_out, int* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // finish the step that produced phi (uses that step's sigma_a / denom)
  const double Tn = new_temperature(cell_mean4(phi, i), T_in[i], sa_in[i], den_in[i], dt, c, a_r,
                                    t_floor);
  if (T) T[i] = Tn;  // (T may alias T_in: each thread reads its cell first)
  if (T0_out) T0_out[i] = Tn;
  // linearise the next step about the new temperature
  const double s_a = power != 0.0 ? sa0[i] * pow(Tn, power) : sa0[i];
  sa[i] = s_a;
  int bad = 0;
  linearize_cell(Tn, s_a, rc[i], dt, c, a_r, ssp ? ssp[i] : 0.0, qe ? qe[i] : 0.0, st[i], ss[i],
                 q[i], den[i], bad);
  if (bad && status) atomicOr(status, 1);
}

int advance_launch(const dlrsn_advance* av, const double* phi, cudaStream_t st) {
  const int n = av->n;
  if (n == 0) return DLRSN_OK;
  advance_kernel<<<(n + 255) / 256, 256, 0, st>>>(
      n, phi, av->T_in, nullptr, av->sigma_a_in, av->denom_in, av->sigma_a, av->sigma_a0,
      av->opacity_power, av->rho_cv, av->dt, av->c, av->a_r, av->t_floor, av->ss_phys, av->q_ext,
      av->sigma_t, av->sigma_s, av->q, av->denom, av->T_out, nullptr);
  DLRSN_CHECK_LAUNCH("advance_kernel");
  return DLRSN_OK;
}

}  // namespace dlrsn

using namespace dlrsn;

extern "C" {

int dlrsn_version(void) { return 1; }

const char* dlrsn_last_error(void) { return g_err; }

int64_t dlrsn_launch_count(void) { return dlrsn::launch_counter().load(); }

int dlrsn_device_sm_count(int* out) {
  int dev = 0;
  DLRSN_TRY_CUDA(cudaGetDevice(&dev));
  DLRSN_TRY_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev));
  return DLRSN_OK;
}

int64_t dlrsn_sk_vec_len(int nx, int ny) { return sk_vec_len(nx, ny); }
int64_t dlrsn_sk_scalar_len(int nx, int ny) { return sk_scalar_len(nx, ny); }

int dlrsn_linearize(int n, const double* T0, const double* sigma_a, const double* rho_cv,
                    double dt, double c, double a_r, const double* ss_phys, const double* q_ext,
                    double* sigma_t, double* sigma_s, double* q, double* denom, int* status,
                    dlrsn_stream_t stream) {
  DLRSN_REQUIRE(dt > 0.0, "time step must be positive, got %g", dt);
  DLRSN_REQUIRE(n >= 0, "negative cell count");
  if (n == 0) return DLRSN_OK;
  linearize_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      n, T0, sigma_a, rho_cv, dt, c, a_r, ss_phys, q_ext, sigma_t, sigma_s, q, denom, status);
  DLRSN_CHECK_LAUNCH("linearize_kernel");
  return DLRSN_OK;
}

int dlrsn_update_temperature(int n, const double* phi, int phi_per_dof, const double* T0,
                             const double* sigma_a, const double* denom, double dt, double c,
                             double a_r, double t_floor, double* T, dlrsn_stream_t stream) {
  if (n == 0) return DLRSN_OK;
  update_temperature_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      n, phi, phi_per_dof, T0, sigma_a, denom, dt, c, a_r, t_floor, T);
  DLRSN_CHECK_LAUNCH("update_temperature_kernel");
  return DLRSN_OK;
}

int dlrsn_advance_relinearize(int n, const double* phi_dofs, double* T,
                              const double* sigma_a_in, const double* denom_in, double* sigma_a,
                              const double* sigma_a0, double opacity_power, const double* rho_cv,
                              double dt, double c, double a_r, double t_floor,
                              const double* ss_phys, const double* q_ext, double* sigma_t,
                              double* sigma_s, double* q, double* denom, double* T0_out,
                              int* status, dlrsn_stream_t stream) {
  DLRSN_REQUIRE(dt > 0.0, "time step must be positive, got %g", dt);
  if (n == 0) return DLRSN_OK;
  advance_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(
      n, phi_dofs, T, T, sigma_a_in, denom_in, sigma_a, sigma_a0, opacity_power, rho_cv, dt, c,
      a_r, t_floor, ss_phys, q_ext, sigma_t, sigma_s, q, denom, T0_out, status);
  DLRSN_CHECK_LAUNCH("advance_kernel");
  return DLRSN_OK;
}

}  // extern "C"
