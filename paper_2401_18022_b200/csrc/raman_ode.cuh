// Device ISRS power-evolution solve: launch interface (raman_ode.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "nli_kernel.cuh"

namespace uwb {

constexpr int kMaxOdeChannels = 2560;  // 512 threads x 5 channels per thread
constexpr int kMaxRamanSegments = 4;  // linear pieces of the gain table in d = |j - i|

struct OdeParams {
  int n;                 // channels
  int raman;             // RamanSolveOptions::include_raman
  const double* alpha;   // [n] 1/m
  double* coef_a;        // [n] f_i aeff_ref / aeff_i          (filled on device)
  double* coef_u;        // [n] P_i / f_i                      (filled on device)
  double* coef_v;        // [n] aeff_ref P_i / aeff_i          (filled on device)
  int n_seg;             // gain table as G = a + b d on d in [dlo, dhi]
  int seg_dlo[kMaxRamanSegments];
  int seg_dhi[kMaxRamanSegments];
  double seg_a[kMaxRamanSegments];
  double seg_b[kMaxRamanSegments];
  int steps;             // distance-grid steps (midpoints)
  int col_stride;        // row stride of log2rho / log_rho (>= steps)
  int lane_k;            // > 0: log2rho in the integrand's lane order lane_pos(m, lane_k)
  const double* mid;     // [steps]
  double length;
  double rtol, atol;
  int continuous;        // 0: restart at every midpoint like the reference; 1: carry h across
  double* log2rho;       // [n * col_stride] out: log2(rho) in the NLI layout
  double* log_rho;       // [n * col_stride] out: ln(rho) (may be null)
  double* rho_end;       // [n] out
  int* status;           // out: 0 ok, 1 non-positive rho, 2 step budget, 3 step underflow
  long long* rhs_evals;  // out (may be null)
};

// Gain table (x, y) -> d-segments for channel spacing `spacing` (host).
// Returns 0, or -1 if the table does not fit kMaxRamanSegments.
int raman_segments(const double* x, const double* y, int rn, double spacing, int n_ch,
                   OdeParams* P);

// Fills the per-channel coupling factors from the launch PSD and runs the
// one-CTA ODE kernel.  Returns kernel launches issued, or < 0 on failure.
// max_ept > 0 overrides the channels-per-thread choice (5 keeps the 589-ch
// solve on 128 threads x <= 255 registers: it then fits on an SM beside one
// integrand CTA, for overlapped batches).
int launch_raman_ode(OdeParams P, const double* freq, const double* psd, double bch,
                     const double* aeff, double aeff_ref, cudaStream_t st, int max_ept = 0);

}  // namespace uwb
