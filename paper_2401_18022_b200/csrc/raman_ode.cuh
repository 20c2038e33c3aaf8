// Device ISRS power-evolution solve: launch interface (raman_ode.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "nli_kernel.cuh"

namespace uwb {

// Channels the device ODE takes: 32 warps x 7 channels per thread.  Combs
// whose prefix arrays fit the opt-in shared memory run from shared memory,
// larger ones from an L1/L2-resident global work buffer (OdeParams::gwork).
constexpr int kMaxOdeChannels = 32 * 32 * 7;
// Linear pieces of the gain table in d = |j - i| (TabulatedProfile rows - 1
// plus zero fill between pieces); edges = pieces + 1.
constexpr int kMaxRamanSegments = 64;
constexpr int kMaxRamanEdges = kMaxRamanSegments + 1;

struct OdeParams {
  int n;                 // channels
  int raman;             // RamanSolveOptions::include_raman
  const double* alpha;   // [n] 1/m
  double* coef_a;        // [n] f_i aeff_ref / aeff_i          (filled on device)
  double* coef_u;        // [n] P_i / f_i                      (filled on device)
  double* coef_v;        // [n] aeff_ref P_i / aeff_i          (filled on device)
  // Gain table G(d), d = |j - i|, as contiguous pieces a_g + b_g d on
  // [edge[g], edge[g + 1]), written in summation-by-parts form: the window
  // sums of piece g enter through their two edges, so edge k carries the
  // jumps da_k = a_k - a_{k-1}, db_k = b_k - b_{k-1} (a_{-1} = a_{n_seg} = 0),
  // folded into the per-edge gather coefficients cu_k = da_k + db_k E_k,
  // cv_k = da_k + db_k (E_k - 1) (raman_ode.cu rhs).
  int n_seg;
  int edge[kMaxRamanEdges];
  double cu[kMaxRamanEdges];
  double cv[kMaxRamanEdges];
  double db[kMaxRamanEdges];
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
  double2* gwork;        // global prefix-array fallback, ode_gwork_double2(n) entries
  long long* prof;       // instrumented build only (UWB_ODE_PROF): phase cycle sums
};

// Gain table (x, y) -> pieces and edges for channel spacing `spacing` (host).
// Returns 0, or -1 if the table needs more than kMaxRamanSegments pieces.
int raman_segments(const double* x, const double* y, int rn, double spacing, int n_ch,
                   OdeParams* P);

// double2 entries of the global work buffer launch_raman_ode may use (callers
// allocate it once and pass it in OdeParams::gwork).
size_t ode_gwork_double2(int n);

// Fills the per-channel coupling factors from the launch PSD and runs the
// one-CTA ODE kernel.  Returns kernel launches issued, or < 0 on failure
// (-1: n out of range, -2: launch error).
// coresident: the ODE runs beside the integrand (overlapped batch): the
// 224-register instantiation, which fits in a partly occupied SM.
int launch_raman_ode(OdeParams P, const double* freq, const double* psd, double bch,
                     const double* aeff, double aeff_ref, cudaStream_t st,
                     bool coresident = false);

// Shared memory (dynamic + static) of the ODE CTA launch_raman_ode issues for
// n channels with the given gain table (0 when it runs from global memory).
size_t raman_ode_smem_bytes(const OdeParams& P);

// The (warps, channels per thread) split launch_raman_ode picks for n
// channels (UWB_ODE_SPLIT="W,EPT" overrides it for experiments).
void ode_split(int n, int* warps, int* ept);

}  // namespace uwb
