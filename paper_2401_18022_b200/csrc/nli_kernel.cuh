// Device-side data layout and launch interface of the ISRS-GN NLI engine.
// See DESIGN.md §3 for the HBM layout and the roofline of each kernel.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace uwb {

// Lane order of the distance steps.  A column of NS = 16 K
// doubles holds step m at position (m % K) * 16 + m / K: lane sl of a 16-lane
// segment owns the K consecutive steps m = sl K + b, b = 0..K-1, and for a
// fixed b the 16 lanes read 16 consecutive doubles (one 128-byte line).
__host__ __device__ __forceinline__ int lane_pos(int m, int K) { return (m % K) * 16 + m / K; }

// Everything the integrand kernel reads.  All pointers are device memory.
struct NliParams {
  // ChannelGrid (channel_grid.hpp:15-22)
  int n_ch;
  const double* freq;
  const double* psd;
  double spacing, bch, centre, half_band;
  double inv_spacing;  // 1 / spacing (host): the row setup multiplies instead of dividing
  // Spans: log2(rho) tables [span][ch][lane_pos(m)] (the reference's log_rho
  // ch*steps+m scaled by log2 e so the integrand can use exp2), span-absolute
  // step geometry, all in lane order.
  int n_spans;
  int steps;              // steps of the longest span (every span's when span_steps is null)
  const int* span_steps;  // [n_spans] each span's own step count, or null (all equal)
  int col_stride;         // NS = 16 * ceil(steps / 16): padded column length (doubles)
  const double* log2rho;  // [n_spans][n_ch + 1][NS]: log2 rho, zero pad column n and pad steps
  size_t span_stride;     // (n_ch + 1) * NS, or 0 when every span shares one table
  const double* zedge;    // [n_spans][NS] z_base + edge[m + 1] (pad steps repeat the span end)
  const double* zstart;   // [n_spans]     z_base + edge[0]
  const double* zmid;     // [n_spans][NS] z_base + mid[m]
  const double* width;    // [n_spans][NS]
  const double* wlast;    // [n_spans] width.back(): fast/slow switch (gn_integral.hpp:156)
  double zmid_max;        // max |z_mid| over spans: bounds the sinc-branch phase |phi z|
  int slow_tiny;          // 1: every sinc-branch phase |phi z| <= 2^-6 (slow_tiny_ok)
  double beta2, beta3, beta4;
  // GnSolverConfig
  int n_r;
  int u1_uniform;
  double ln_min;  // log(u1_min_ratio), host-computed
  int n_q;        // 3 with mirror_q4, else 4
  // probes
  int n_probes;
  const double* probe_nu;  // [n_probes]
  // [n_probes] channel of each probe, or null.  When set (the prepared /
  // resident path), rows of a probe whose channel has psd <= 0 in this
  // evaluation are skipped on the device: the reference's per-call skip set
  // (gn_integral.hpp:349-352) re-derived from the launch profile.
  const int* probe_chan;
  double* hl2;             // [n_probes][n_spans][NS] 16 x log2 half-power of the probe
  // work queue + outputs
  int total_rows;               // n_probes * n_q * n_r
  unsigned int* counter;        // row queue head (zeroed before launch)
  // Split evaluation (launch_nli_setup / launch_nli_lists): the rows' point
  // records written by the setup pass while the Raman ODE runs, [row][n_r]
  // records of nli_point_record_bytes() each, and each row's record count
  // (-1: the row is skipped).  Null: the fused kernel.
  void* plist;
  int* plist_n;
  unsigned long long* n_eval;   // [2]: |K|^2 evaluations, active points (stats)
  unsigned long long* n_active; // = n_eval + 1
  uint2* rowcnt;                // [total_rows] (|K|^2 evaluations, active points) per row
  unsigned long long* probe_work;  // [n_probes] |K|^2 evaluations per probe (null: off);
                                  // the multi-GPU partition's cost model
  int mirror_u2;                // share |K|^2 across u2 -> -u2 in symmetric rows
  int mixed;                    // 1: compensated-FP32 step arithmetic (uwb_set_precision)
  double* rowsum;               // [total_rows]; NaN => row not added (reference `continue`)
  double* rowpar;               // [total_rows][4] su, u1, lo, du2 (+ du1 in rowsum until the
                                // row is done); su < 0: the row is skipped (row_params_kernel)
};

struct FinalizeParams {
  // per probe
  int n_probes;
  const double* probe_gamma;  // [n_probes]
  double* probe_g;            // [n_probes] (16/27) gamma^2 sum_q quad
  double* probe_quad;         // [n_probes * 4]
  int mirror_q4;
  // per channel (n_ch = 0 skips the channel stage: nli_psd_at mode)
  int n_ch;
  const double* psd;       // launch PSD per channel
  double bch;
  int simpson;
  const int* chan_probe0;  // [n_ch] first probe of the channel or -1 (skipped)
  double* eta;
  double* nli_psd;
  double* nli_power;
  double* quad;      // [n_ch * 4]
  uint8_t* skipped;  // [n_ch]
};

// Host: append one span's lane-ordered geometry (the NliParams zedge / zstart /
// zmid / width / wlast arrays) for a span starting at z_base.
struct SpanTables {
  std::vector<double> zend, zstart, zmid, width, wlast;
  double zmid_max = 0.0;  // largest |z| of a step midpoint over all spans
};
inline void append_span_tables(const double* edge, const double* mid, const double* width,
                               int steps, double z_base, SpanTables* t, int NS = 0) {
  if (NS <= 0) NS = 16 * ((steps + 15) / 16);  // else the longest span's padded length
  const int K = NS / 16;
  const size_t o = t->zend.size();
  t->zend.resize(o + NS);
  t->zmid.resize(o + NS);
  t->width.resize(o + NS);
  for (int m = 0; m < NS; ++m) {
    const int e = lane_pos(m, K);
    const int mm = std::min(m, steps - 1);
    t->zend[o + e] = z_base + edge[std::min(m + 1, steps)];
    t->zmid[o + e] = z_base + mid[mm];
    t->width[o + e] = width[mm];
  }
  t->zstart.push_back(z_base + edge[0]);
  t->wlast.push_back(width[steps - 1]);
  for (int m = 0; m < steps; ++m) t->zmid_max = std::max(t->zmid_max, std::fabs(z_base + mid[m]));
}

// Issue the NLI pipeline on `stream`: queue reset, probe half-log columns,
// integrand rows (persistent, grid_ctas CTAs), per-probe and per-channel
// finalize.  ev_k0/ev_k1 (may be null) bracket the integrand kernel.
// Returns the number of kernel launches (memset excluded).
// coresident_smem: shared memory another kernel must find free on an SM next
// to the integrand's CTAs (the overlapped batch's Raman ODE); it raises the
// integrand's shared-memory carveout accordingly (0: smallest carveout, most L1).
int launch_nli(const NliParams& p, const FinalizeParams& f, int grid_ctas, cudaStream_t stream,
               cudaEvent_t ev_k0, cudaEvent_t ev_k1, size_t coresident_smem = 0);

// Split evaluation of single-span FP64 problems with K <= 8 (nli_split_ok):
// launch_nli_setup issues the row parameters and the per-row point records
// (everything the launch PSD decides; nothing depends on the power profile)
// on `side`, with `grid_ctas` CTAs -- it runs beside the Raman ODE; then
// launch_nli_lists evaluates the listed points (probe half-logs, rows,
// finalize) on `stream` once the ODE and the setup are done.  The row sums
// are bit-identical to launch_nli's.
bool nli_split_ok(const NliParams& p);
size_t nli_point_record_bytes();
int nli_list_ctas_per_sm(const NliParams& p);  // resident nli_list_kernel CTAs per SM
int nli_setup_ctas_per_sm();
int launch_nli_setup(const NliParams& p, int grid_ctas, cudaStream_t side);
int launch_nli_lists(const NliParams& p, const FinalizeParams& f, int grid_ctas,
                     cudaStream_t stream, cudaEvent_t ev_k0, cudaEvent_t ev_k1);

// CTAs per SM the integrand kernel reaches for a given step count.
int nli_ctas_per_sm(int steps, bool one_span, int n_r, bool mixed = false, bool tiny = false,
                    bool ragged = false);

// Sinc-branch points have |phi| w_last <= 1e-4 (gn_integral.hpp:156), so their
// phases satisfy |phi z| <= 1e-4 z_max / w_last; the Taylor sincos of the TINY
// kernels is exact to < 1e-19 for |phi z| <= 2^-6.
inline bool slow_tiny_ok(const SpanTables& t) {
  double wmin = 0.0;
  for (size_t k = 0; k < t.wlast.size(); ++k)
    wmin = k == 0 ? t.wlast[k] : std::min(wmin, t.wlast[k]);
  return wmin > 0.0 && 1e-4 * t.zmid_max <= 0.015625 * wmin;
}
// Steps per span: up to 512 (16 lanes x 32 unrolled steps per lane) take the
// specialised kernels, longer spans the rolled K = 0 kernel.
constexpr int kMaxSteps = 16 * 4096;
// Elements allocated past the end of log2rho / zedge / hl2: the integrand's
// lanes with m >= N load them and mask the result (branch-free tail).
constexpr int kTablePad = 32;

// Live FP64 pipe peak (TFLOP/s): independent DFMA chains on every SM, timed
// with CUDA events.  The roofline denominator for the integrand kernel.
double fp64_fma_peak_tflops(int sm_count, cudaStream_t stream);
// First failing line of the bounds-checked build (0: none; -1: not built with
// -DUWB_BOUNDS_CHECK=1).  Per translation unit: nli_kernel.cu / raman_ode.cu.
int nli_bounds_status();
int ode_bounds_status();  // 16 lanes x 16 steps per lane

}  // namespace uwb
