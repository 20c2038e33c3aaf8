// Closed-form NLI model on the device:
// cfm_all_channels_nli, gn_closed_form.hpp:70-144.
//
// Per span:
//   cfm_alpha_kernel    one thread per channel: the ISRS-shaped effective
//                       length l_eff = sum_m rho_m width_m (ascending m, :93-97)
//                       and the bisection effective_alpha (:37-47, 200 steps);
//   cfm_channel_kernel  one CTA per channel i: SPM term (:111-118), then the
//                       XPM pair sum over pumps k (:120-128) split across the
//                       CTA's threads (thread t takes k = t, t + T, ...) and
//                       combined by a fixed-order tree, so the result does not
//                       depend on scheduling; eta_i accumulates across spans
//                       in span order like the reference (:129).
//   cfm_finalize_kernel nli_power = eta P^3, nli_psd = nli_power / B (:133-138).
// O(N^2) pair terms (347 k for 589 channels) of atan/log1p each: a few
// microseconds on 148 SMs, against ~0.1 s for the reference on one core.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "uwb_capi_internal.cuh"

namespace uwb {

namespace {

constexpr double kPiC = 3.14159265358979323846;  // units.hpp:11
constexpr double kCfmSpmCalibration = 1.9641;     // gn_closed_form.hpp:67
constexpr double kCfmXpmCalibration = 1.0571;     // gn_closed_form.hpp:68
constexpr int kCfmThreads = 128;

struct CfmParams {
  int n;
  const double* freq;
  const double* psd;
  const uint8_t* guard;
  const double* gamma;
  double bch, centre;
  double b2, b3, b4;
  // one span
  const double* log_rho;  // [n * steps] reference layout ch * steps + m
  const double* width;    // [steps]
  int steps;
  double length;
  double* alpha_eff;  // [n]
  double* eta;        // [n] accumulated across spans
  uint8_t* skipped;   // [n]
  double* nli_psd;
  double* nli_power;
};

// phi_xpm (gn_closed_form.hpp:23-27), same grouping
__device__ __forceinline__ double phi_xpm(double f_i, double f_k, const CfmParams& P) {
  const double bracket = P.b2 + kPiC * P.b3 * (f_i + f_k) +
                         (2.0 * kPiC * kPiC / 3.0) * P.b4 * (f_i * f_i + f_i * f_k + f_k * f_k);
  return -4.0 * kPiC * kPiC * bracket * (f_k - f_i);
}

// phi_spm (:30-33)
__device__ __forceinline__ double phi_spm(double f_i, const CfmParams& P) {
  return -4.0 * kPiC * kPiC *
         (P.b2 + 2.0 * kPiC * P.b3 * f_i + 2.0 * kPiC * kPiC * P.b4 * f_i * f_i);
}

// detail::xpm_island (:53-59)
__device__ __forceinline__ double xpm_island(double phi_abs, double bch, double alpha) {
  const double x = phi_abs * bch / (2.0 * alpha);
  if (x < 1e-3) return (0.75 - (5.0 / 24.0) * x * x) * bch * bch / (alpha * alpha);
  return 2.0 * bch / (alpha * phi_abs) * atan(x) - log1p(x * x) / (phi_abs * phi_abs);
}

__global__ void cfm_alpha_kernel(const CfmParams P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  double l_eff = 0.0;
  const double* lr = P.log_rho + static_cast<size_t>(i) * P.steps;
  for (int m = 0; m < P.steps; ++m) l_eff += exp(lr[m]) * P.width[m];
  double a = 1e-12;
  if (l_eff > 0.0) {
    const double le = l_eff < P.length ? l_eff : P.length;
    if (!(le >= P.length)) {  // effective_alpha (:37-47)
      double lo = 1e-12, hi = 1.0;
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        const double val = (1.0 - exp(-mid * P.length)) / mid;
        if (val > le) lo = mid; else hi = mid;
      }
      a = 0.5 * (lo + hi);
    }
  }
  P.alpha_eff[i] = a;
}

__global__ void __launch_bounds__(kCfmThreads) cfm_channel_kernel(const CfmParams P) {
  const int i = blockIdx.x;
  const int t = threadIdx.x;
  if (P.guard[i] || P.psd[i] <= 0.0) {
    if (t == 0) P.skipped[i] = 1;
    return;
  }
  const double bch = P.bch;
  const double p_i = P.psd[i] * bch;
  const double f_i = P.freq[i] - P.centre;
  const double g_i = P.gamma[i];
  double part = 0.0;
  for (int k = t; k < P.n; k += kCfmThreads) {
    if (k == i || P.guard[k] || P.psd[k] <= 0.0) continue;
    const double p_k = P.psd[k] * bch;
    const double phik = fabs(phi_xpm(f_i, P.freq[k] - P.centre, P));
    const double island = xpm_island(phik, bch, P.alpha_eff[k]);
    const double ratio = p_k / p_i;
    part += kCfmXpmCalibration * (32.0 / 27.0) * (g_i * P.gamma[k] / (bch * bch)) * ratio *
            ratio * island;
  }
  // fixed-order tree: warp xor-shuffle, then the warps in order
  __shared__ double wsum[kCfmThreads / 32];
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((t & 31) == 0) wsum[t >> 5] = part;
  __syncthreads();
  if (t == 0) {
    // SPM (:111-119)
    const double phi_i = fabs(phi_spm(f_i, P));
    const double a_i = P.alpha_eff[i];
    const double spm_arg = phi_i * bch * bch / (8.0 * a_i);
    double spm;
    if (spm_arg < 1e-3)
      spm = (kPiC / (a_i * fmax(phi_i, 1e-300))) * spm_arg;  // asinh(x) ~ x
    else
      spm = (kPiC / (a_i * phi_i)) * asinh(spm_arg);
    double eta_i = kCfmSpmCalibration * (16.0 / 27.0) * (g_i * g_i / (bch * bch)) * spm;
    double xpm = 0.0;
    for (int w = 0; w < kCfmThreads / 32; ++w) xpm += wsum[w];
    eta_i += xpm;
    P.eta[i] += eta_i;  // incoherent accumulation across spans (:129)
  }
}

__global__ void cfm_finalize_kernel(const CfmParams P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n || P.skipped[i]) return;
  const double p = P.psd[i] * P.bch;
  P.nli_power[i] = P.eta[i] * p * p * p;
  P.nli_psd[i] = P.nli_power[i] / P.bch;
}

}  // namespace

}  // namespace uwb

using namespace uwb;

extern "C" int uwb_cfm_all_channels_nli(uwb_ctx* c, const uwb_grid* grid, int n_spans,
                                        const uwb_span* spans, const double beta[3],
                                        const double* gamma, uwb_nli_result* out) {
  if (!c) return fail(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return uwb_cfm_all_channels_nli(c->subs[0], grid, n_spans, spans, beta, gamma, out);
  cudaSetDevice(c->device);
  reset_xfer(c);
  int rc = validate_grid(grid);
  if (rc) return rc;
  if (n_spans <= 0 || !spans) return fail(UWB_CONFIG_ERROR, "cfm: need at least one span");
  if (!gamma) return fail(UWB_CONFIG_ERROR, "missing per-channel gamma");
  if (!beta) return fail(UWB_CONFIG_ERROR, "missing beta coefficients");
  const int n = grid->n_ch;
  for (int k = 0; k < n_spans; ++k)
    if (!spans[k].log_rho || !spans[k].width || spans[k].steps < 1)
      return fail(UWB_CONFIG_ERROR, "cfm: span evolution does not match the grid");
  cudaStream_t st = c->stream;
  // inputs: freq, psd, gamma [3n] | guard [n bytes]; work: alpha_eff, eta, nli_psd, nli_power [4n]
  double* din = c->cfm_in.get<double>(3 * static_cast<size_t>(n) + (n + 7) / 8);
  double* dwk = c->cfm_work.get<double>(4 * static_cast<size_t>(n) + (n + 7) / 8);
  if (!din || !dwk) return fail(UWB_CUDA_ERROR, "device allocation failed");
  CfmParams P{};
  P.n = n;
  P.freq = din;
  P.psd = din + n;
  P.gamma = din + 2 * n;
  P.guard = reinterpret_cast<const uint8_t*>(din + 3 * n);
  P.bch = grid->bch;
  P.centre = grid->centre;
  P.b2 = beta[0];
  P.b3 = beta[1];
  P.b4 = beta[2];
  P.alpha_eff = dwk;
  P.eta = dwk + n;
  P.nli_psd = dwk + 2 * n;
  P.nli_power = dwk + 3 * n;
  P.skipped = reinterpret_cast<uint8_t*>(dwk + 4 * n);
  xfer(c, din, grid->freq, n * 8, cudaMemcpyHostToDevice, st);
  xfer(c, din + n, grid->psd, n * 8, cudaMemcpyHostToDevice, st);
  xfer(c, din + 2 * n, gamma, n * 8, cudaMemcpyHostToDevice, st);
  xfer(c, din + 3 * n, grid->guard, n, cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(dwk + n, 0, 3 * n * sizeof(double), st);
  cudaMemsetAsync(P.skipped, 0, n, st);
  cudaEventRecord(c->ev0, st);
  int launches = 0;
  for (int k = 0; k < n_spans; ++k) {
    const int steps = spans[k].steps;
    double* dspan = c->cfm_span.get<double>(static_cast<size_t>(n) * steps + steps);
    if (!dspan) return fail(UWB_CUDA_ERROR, "device allocation failed");
    // spans that share the previous span's tables skip the upload
    if (k == 0 || spans[k].log_rho != spans[k - 1].log_rho || spans[k].width != spans[k - 1].width ||
        steps != spans[k - 1].steps) {
      xfer(c, dspan, spans[k].log_rho, static_cast<size_t>(n) * steps * 8, cudaMemcpyHostToDevice, st);
      xfer(c, dspan + static_cast<size_t>(n) * steps, spans[k].width, steps * 8,
           cudaMemcpyHostToDevice, st);
    }
    P.log_rho = dspan;
    P.width = dspan + static_cast<size_t>(n) * steps;
    P.steps = steps;
    P.length = spans[k].length;
    cfm_alpha_kernel<<<(n + 127) / 128, 128, 0, st>>>(P);
    cfm_channel_kernel<<<n, kCfmThreads, 0, st>>>(P);
    launches += 2;
  }
  cfm_finalize_kernel<<<(n + 127) / 128, 128, 0, st>>>(P);
  ++launches;
  cudaEventRecord(c->ev1, st);
  if (out) {
    if (out->eta) xfer(c, out->eta, P.eta, n * 8, cudaMemcpyDeviceToHost, st);
    if (out->nli_psd) xfer(c, out->nli_psd, P.nli_psd, n * 8, cudaMemcpyDeviceToHost, st);
    if (out->nli_power) xfer(c, out->nli_power, P.nli_power, n * 8, cudaMemcpyDeviceToHost, st);
    if (out->skipped) xfer(c, out->skipped, P.skipped, n, cudaMemcpyDeviceToHost, st);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "cfm_all_channels_nli");
  if (out) {
    if (out->quadrant)  // the closed form has no quadrants (reference: zeros)
      for (int i = 0; i < 4 * n; ++i) out->quadrant[i] = 0.0;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    out->elapsed_seconds = ms * 1e-3;
  }
  c->last_launches = launches;
  return UWB_OK;
}
