// C-ABI of the ISRS-GN NLI engine (include/uwb_nli.h): validation with the
// reference's error contract, HBM upload of the path's inputs, probe
// construction, launch and read-back.  Host side only; kernels live in
// nli_kernel.cu / raman_ode.cu / link_report.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/uwb_nli.h"
#include "nli_kernel.cuh"
#include "uwb_capi_internal.cuh"
#include "uwb_ctx.cuh"
#include "uwb_devmath.cuh"
#include "uwb_multi.cuh"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace uwb {

int fail(int code, const std::string& msg) { return set_err(code, msg); }

int cuda_fail(cudaError_t e, const char* what) {
  return set_err(UWB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// Grid checks of the NLI entry points (all_channels_nli / nli_psd_at /
// channel_nli).  The reference does NOT call ChannelGrid::validate on that
// path (gn_integral.hpp:218-363): psd_at and stencil_for simply assume the
// equal spacing, and so does the device.  These are the checks that keep the
// device's index arithmetic defined (non-empty, positive spacing/width,
// ascending, no negative PSD); the ODE and link entry points run the full
// ChannelGrid::validate (validate_grid_full) exactly where the reference does.
int validate_grid(const uwb_grid* g) {
  if (!g || g->n_ch < 1 || !g->freq || !g->psd || !g->guard)
    return fail(UWB_CONFIG_ERROR, "channel grid is empty");
  if (!(g->spacing > 0.0) || !(g->bch > 0.0))
    return fail(UWB_CONFIG_ERROR, "grid spacing and width must be > 0");
  if (g->bch > g->spacing + 1e-9) return fail(UWB_CONFIG_ERROR, "channel width exceeds spacing");
  for (int i = 0; i < g->n_ch; ++i) {
    if (g->psd[i] < 0.0) return fail(UWB_CONFIG_ERROR, "negative launch PSD");
    if (i > 0 && !(g->freq[i] > g->freq[i - 1]))
      return fail(UWB_CONFIG_ERROR, "grid must ascend in frequency");
  }
  return UWB_OK;
}

// ChannelGrid::validate (channel_grid.hpp:44-61), every check in the
// reference's order: solve_power_evolution calls it first (raman_power.hpp:56),
// so uwb_power_evolution, uwb_evaluate_link and uwb_evaluate_link_prepare do
// too.  The device ODE's separable coupling relies on the equal spacing
// (raman_ode.cu: f_j - f_i = (j - i) spacing).
int validate_grid_full(const uwb_grid* g) {
  if (!g || g->n_ch < 1 || !g->freq || !g->psd || !g->guard)
    return fail(UWB_CONFIG_ERROR, "channel grid is empty");
  if (!(g->spacing > 0.0) || !(g->bch > 0.0))
    return fail(UWB_CONFIG_ERROR, "grid spacing and width must be > 0");
  if (g->bch > g->spacing + 1e-9) return fail(UWB_CONFIG_ERROR, "channel width exceeds spacing");
  for (int i = 0; i < g->n_ch; ++i) {
    if (g->psd[i] < 0.0) return fail(UWB_CONFIG_ERROR, "negative launch PSD");
    if (i > 0 && !(g->freq[i] > g->freq[i - 1]))
      return fail(UWB_CONFIG_ERROR, "grid must ascend in frequency");
    if (i > 0 && std::abs((g->freq[i] - g->freq[i - 1]) - g->spacing) > 1e-3)
      return fail(UWB_CONFIG_ERROR, "grid must be equally spaced");
  }
  const double need = std::max(std::abs(g->freq[0] - g->centre),
                               std::abs(g->freq[g->n_ch - 1] - g->centre)) + 0.5 * g->bch;
  if (g->half_band + 1e-3 < need)
    return fail(UWB_CONFIG_ERROR, "half_band smaller than occupied hull");
  return UWB_OK;
}

// Upload the grid + span tables; fills the grid/span part of NliParams.
int upload_path_inputs(uwb_ctx* c, const uwb_grid* g, int n_spans, const uwb_span* spans,
                       const double beta[3], NliParams* P) {
  // nli_psd_at's checks, in the reference's order (gn_integral.hpp:223-240)
  if (n_spans <= 0 || !spans) return fail(UWB_CONFIG_ERROR, "nli_psd_at: need at least one span");
  const int n = g->n_ch;
  // Each span keeps its own step count (the reference walks every span's own
  // distance grid, gn_integral.hpp:231-251): the columns are padded to the
  // longest span, and a span's lanes past its own count are masked.
  int steps = 0;
  bool ragged = false;
  for (int k = 0; k < n_spans; ++k) {
    if (!spans[k].log_rho || !spans[k].edge || !spans[k].mid || !spans[k].width)
      return fail(UWB_CONFIG_ERROR, "nli_psd_at: span evolution does not match the channel grid");
    if (spans[k].steps < 1 || spans[k].steps > kMaxSteps)
      return fail(UWB_CONFIG_ERROR, "uwb: distance steps per span must be in [1, 65536]");
    if (k > 0 && spans[k].steps != spans[0].steps) ragged = true;
    steps = std::max(steps, spans[k].steps);
  }

  // Padded device layout (nli_kernel.cuh): columns NS = 16 ceil(N/16) long,
  // one zero pad column n per span, edges past N repeat the span end.
  const int NS = 16 * ((steps + 15) / 16);
  const size_t cols = static_cast<size_t>(n + 1) * NS;
  std::vector<double> tab(static_cast<size_t>(n_spans) * cols, 0.0);
  SpanTables stb;
  const int K = NS / 16;
  double z_base = 0.0;
  std::vector<int> span_steps(n_spans);
  long long total_steps = 0;
  for (int k = 0; k < n_spans; ++k) {
    const uwb_span& s = spans[k];
    const int sk = s.steps;
    span_steps[k] = sk;
    total_steps += sk;
    double* t = tab.data() + static_cast<size_t>(k) * cols;
    for (int ch = 0; ch < n; ++ch)
      for (int m = 0; m < sk; ++m)
        t[static_cast<size_t>(ch) * NS + lane_pos(m, K)] =
            s.log_rho[static_cast<size_t>(ch) * sk + m] * kLog2e;
    append_span_tables(s.edge, s.mid, s.width, sk, z_base, &stb, NS);
    z_base += s.length;
  }
  int* d_ss = nullptr;
  if (ragged) {
    d_ss = c->span_steps.get<int>(n_spans);
    if (!d_ss) return fail(UWB_CUDA_ERROR, "device allocation failed");
    xfer(c, d_ss, span_steps.data(), n_spans * sizeof(int), cudaMemcpyHostToDevice, c->stream);
  }
  const std::vector<double>& ze = stb.zend;
  const std::vector<double>& zm = stb.zmid;
  const std::vector<double>& wd = stb.width;
  const std::vector<double>& wl = stb.wlast;
  const std::vector<double>& zs = stb.zstart;
  double* d_freq = c->freq.get<double>(n);
  double* d_psd = c->psd.get<double>(n);
  double* d_tab = c->log2rho.get<double>(tab.size());
  double* d_ze = c->zedge.get<double>(ze.size());
  double* d_zm = c->zmid.get<double>(zm.size());
  double* d_wd = c->width.get<double>(wd.size());
  double* d_wl = c->wlast.get<double>(wl.size());
  double* d_zs = c->zstart.get<double>(zs.size());
  if (!d_freq || !d_psd || !d_tab || !d_ze || !d_zm || !d_wd || !d_wl || !d_zs)
    return fail(UWB_CUDA_ERROR, "device allocation failed");
  cudaStream_t st = c->stream;
  xfer(c, d_freq, g->freq, n * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_psd, g->psd, n * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_ze, ze.data(), ze.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_zm, zm.data(), zm.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_wd, wd.data(), wd.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_wl, wl.data(), wl.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  xfer(c, d_zs, zs.data(), zs.size() * sizeof(double), cudaMemcpyHostToDevice, st);
  // the vectors die at return: make the copies complete first
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "upload");

  P->n_ch = n;
  P->freq = d_freq;
  P->psd = d_psd;
  P->spacing = g->spacing;
  P->inv_spacing = 1.0 / g->spacing;
  P->bch = g->bch;
  P->centre = g->centre;
  P->half_band = g->half_band;
  P->n_spans = n_spans;
  P->steps = steps;
  P->span_steps = d_ss;
  P->log2rho = d_tab;
  P->col_stride = NS;
  P->span_stride = cols;
  P->zedge = d_ze;
  P->zstart = d_zs;
  P->zmid_max = stb.zmid_max;
  P->slow_tiny = slow_tiny_ok(stb) ? 1 : 0;
  P->zmid = d_zm;
  P->width = d_wd;
  P->wlast = d_wl;
  P->beta2 = beta[0];
  P->beta3 = beta[1];
  P->beta4 = beta[2];
  c->last_total_steps = static_cast<double>(total_steps);
  return UWB_OK;
}

int set_cfg(const uwb_nli_cfg* cfg, NliParams* P, int precision) {
  if (!cfg) return fail(UWB_CONFIG_ERROR, "missing solver config");
  if (cfg->n_r < 2) return fail(UWB_CONFIG_ERROR, "nli_psd_at: n_r must be >= 2");
  P->n_r = cfg->n_r;
  P->u1_uniform = cfg->u1_uniform ? 1 : 0;
  P->ln_min = std::log(cfg->u1_min_ratio);
  P->n_q = cfg->mirror_q4 ? 3 : 4;
  // UWB_NLI_NO_MIRROR=1 evaluates every column of symmetric rows (A/B checks)
  static const bool no_mirror = [] {
    const char* e = std::getenv("UWB_NLI_NO_MIRROR");
    return e && e[0] == '1';
  }();
  P->mirror_u2 = no_mirror ? 0 : 1;
  P->mixed = precision == UWB_PRECISION_MIXED ? 1 : 0;
  return UWB_OK;
}

// Upload probes, run the pipeline, leave results in the context buffers.
int run_probes(uwb_ctx* c, NliParams& P, const uwb_nli_cfg* cfg, const std::vector<double>& nu,
               const std::vector<double>& gam, const std::vector<int>* chan_probe0,
               bool sync_stats) {
  // quadrant_limits' range check (gn_integral.hpp:64-66), probe by probe
  for (double v : nu) {
    const double f = v - P.centre;
    if (std::abs(f) > P.half_band)
      return fail(UWB_CONFIG_ERROR,
                  "quadrant_limits: channel offset must lie inside the half band");
  }
  const int np = static_cast<int>(nu.size());
  FinalizeParams F{};
  F.n_probes = np;
  F.mirror_q4 = cfg->mirror_q4 ? 1 : 0;
  c->last_launches = 0;
  c->last_kernel_ms = 0.0;
  c->last_inner_steps = 0.0;
  c->last_points = 0.0;
  if (np == 0 && !chan_probe0) return UWB_OK;
  double* d_nu = c->probe_nu.get<double>(std::max(np, 1));
  double* d_g = c->probe_gamma.get<double>(std::max(np, 1));
  P.n_probes = np;
  P.total_rows = np * P.n_q * P.n_r;
  P.probe_nu = d_nu;
  P.hl2 = c->hl2.get<double>(static_cast<size_t>(std::max(np, 1)) * P.n_spans * P.col_stride);
  P.rowsum = c->rowsum.get<double>(std::max(P.total_rows, 1));
  P.rowpar = c->rowpar.get<double>(4 * static_cast<size_t>(std::max(P.total_rows, 1)));
  P.counter = c->counter.get<unsigned int>(1);
  P.n_eval = c->n_eval.get<unsigned long long>(2);
  P.n_active = P.n_eval + 1;
  P.probe_work = c->probe_work.get<unsigned long long>(std::max(np, 1));
  P.rowcnt = c->rowcnt.get<uint2>(std::max(P.total_rows, 1));
  F.probe_gamma = d_g;
  F.probe_g = c->probe_g.get<double>(std::max(np, 1));
  F.probe_quad = c->probe_quad.get<double>(4 * std::max(np, 1));
  if (!P.hl2 || !P.rowsum || !P.rowpar || !P.counter || !F.probe_g || !F.probe_quad || !d_nu || !d_g)
    return fail(UWB_CUDA_ERROR, "device allocation failed");
  cudaStream_t st = c->stream;
  if (np) {
    xfer(c, d_nu, nu.data(), np * sizeof(double), cudaMemcpyHostToDevice, st);
    xfer(c, d_g, gam.data(), np * sizeof(double), cudaMemcpyHostToDevice, st);
  }
  c->last_n_probes = np;
  c->last_probes_per_chan = cfg->simpson ? 3 : 1;
  if (chan_probe0) c->last_chan_probe0 = *chan_probe0;
  else c->last_chan_probe0.clear();
  if (chan_probe0) {
    const int n = P.n_ch;
    int* d_cp = c->chan_probe0.get<int>(n);
    F.n_ch = n;
    F.psd = P.psd;
    F.bch = P.bch;
    F.simpson = cfg->simpson ? 1 : 0;
    F.chan_probe0 = d_cp;
    F.eta = c->eta.get<double>(n);
    F.nli_psd = c->nli_psd.get<double>(n);
    F.nli_power = c->nli_power.get<double>(n);
    F.quad = c->quad.get<double>(4 * n);
    F.skipped = c->skipped.get<uint8_t>(n);
    xfer(c, d_cp, chan_probe0->data(), n * sizeof(int), cudaMemcpyHostToDevice, st);
  }
  cudaEventRecord(c->ev0, st);
  if (np) {
    const int per_sm = nli_ctas_per_sm(P.steps, P.n_spans == 1, P.n_r, P.mixed != 0, P.slow_tiny != 0,
                                       P.span_steps != nullptr);
    if (per_sm <= 0) return fail(UWB_CUDA_ERROR, "integrand kernel cannot be resident");
    const int launched = launch_nli(P, F, c->sm_count * per_sm, st, c->evk0, c->evk1);
    if (launched < 0) return fail(UWB_CONFIG_ERROR, "unsupported step count");
    c->last_launches = launched;
    c->nli_events_valid = true;
  } else {
    // every channel skipped: only the channel epilogue
    c->last_launches = launch_finalize_channels_only(F, st);
  }
  cudaEventRecord(c->ev1, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "launch");
  if (sync_stats) {
    e = cudaEventSynchronize(c->ev1);
    if (e != cudaSuccess) return cuda_fail(e, "nli kernels");
    float ms = 0.f;
    if (np) {
      cudaEventElapsedTime(&ms, c->evk0, c->evk1);
      c->last_kernel_ms = ms;
      unsigned long long ne[2] = {0, 0};
      xfer_sync(c, ne, P.n_eval, sizeof ne, cudaMemcpyDeviceToHost);
      c->last_points = static_cast<double>(ne[0]);
      c->last_active = static_cast<double>(ne[1]);
      c->last_inner_steps = static_cast<double>(ne[0]) * c->last_total_steps;
    }
  }
  return UWB_OK;
}

// Probe list of all_channels_nli (gn_integral.hpp:348-353, channel_nli :316-329).
// include_dark: also probe non-guard channels with psd <= 0 (the prepared
// path, whose device kernels re-derive the skip set per evaluation);
// probe_chan (may be null) receives each probe's channel.
void channel_probes(const uwb_grid* g, const double* gamma, const uwb_nli_cfg* cfg,
                    const std::vector<int>& subset, std::vector<double>* nu,
                    std::vector<double>* gam, std::vector<int>* chan_probe0, bool include_dark,
                    std::vector<int>* probe_chan) {
  const int n = g->n_ch;
  std::vector<uint8_t> want(n, subset.empty() ? 1 : 0);
  for (int ch : subset)
    if (ch >= 0 && ch < n) want[ch] = 1;
  chan_probe0->assign(n, -1);
  for (int ch = 0; ch < n; ++ch) {
    if (!want[ch] || g->guard[ch] || (!include_dark && g->psd[ch] <= 0.0)) continue;
    (*chan_probe0)[ch] = static_cast<int>(nu->size());
    const double f = g->freq[ch];
    const int np = cfg->simpson ? 3 : 1;
    nu->push_back(f);
    if (cfg->simpson) {
      nu->push_back(f - 0.5 * g->bch);
      nu->push_back(f + 0.5 * g->bch);
    }
    for (int k = 0; k < np; ++k) {
      gam->push_back(gamma[ch]);
      if (probe_chan) probe_chan->push_back(ch);
    }
  }
}

}  // namespace uwb

using namespace uwb;

extern "C" {

const char* uwb_last_error(void) { return g_err.c_str(); }

int uwb_abi_version(void) { return UWB_ABI_VERSION; }

int uwb_device_count(int* n) {
  if (!n) return set_err(UWB_CONFIG_ERROR, "null output");
  *n = 0;
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    return set_err(UWB_CUDA_ERROR, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  return UWB_OK;
}

int uwb_ctx_create(int device, uwb_ctx** out) {
  if (!out) return set_err(UWB_CONFIG_ERROR, "null output");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return set_err(UWB_CUDA_ERROR, "no CUDA device visible (the engine has no CPU fallback)");
  if (device < 0 || device >= n) return set_err(UWB_CONFIG_ERROR, "device index out of range");
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "props");
  if (prop.major < 10)
    return set_err(UWB_CUDA_ERROR, "the engine is built for sm_100a (B200); device is sm_" +
                                       std::to_string(prop.major) + std::to_string(prop.minor));
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto* c = new uwb_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->cc_major = prop.major;
  c->cc_minor = prop.minor;
  if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "stream");
  }
  cudaEventCreate(&c->ev0);
  cudaEventCreate(&c->ev1);
  cudaEventCreate(&c->evk0);
  cudaEventCreate(&c->evk1);
  // probe the kernel image: fails loudly if the fatbin has no sm_100a code
  if (nli_ctas_per_sm(112, true, 150) <= 0) {
    uwb_ctx_destroy(c);
    return set_err(UWB_CUDA_ERROR, "integrand kernel not loadable on this device");
  }
  *out = c;
  return UWB_OK;
}

void uwb_ctx_destroy(uwb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  release_link_state(c);
  for (uwb_ctx* s : c->subs) uwb_ctx_destroy(s);
  for (uwb_ctx* s : c->bsubs) uwb_ctx_destroy(s);
  c->subs.clear();
  c->bsubs.clear();
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  for (DBuf* b : {&c->freq, &c->psd, &c->gamma, &c->log2rho, &c->zedge, &c->zstart, &c->zmid, &c->width,
                  &c->wlast, &c->span_steps, &c->probe_nu, &c->probe_chan, &c->probe_work, &c->rowcnt, &c->probe_gamma, &c->hl2, &c->rowsum, &c->rowpar, &c->up_dev, &c->plist, &c->plist_n, &c->counter,
                  &c->n_eval, &c->probe_g, &c->probe_quad, &c->chan_probe0, &c->eta, &c->nli_psd,
                  &c->nli_power, &c->quad, &c->skipped, &c->batch_psd, &c->batch_report, &c->batch_ode, &c->alpha, &c->aeff, &c->raman_x,
                  &c->raman_y, &c->nf_db, &c->guard, &c->rho_end, &c->ode_work, &c->ode_gwork, &c->report,
                  &c->mid, &c->edge})
    b->release();
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->up_pinned) cudaFreeHost(c->up_pinned);
  if (c->batch) {
    for (cudaEvent_t ev : {c->batch->ev_start, c->batch->ev_ode[0], c->batch->ev_ode[1],
                           c->batch->ev_nli[0], c->batch->ev_nli[1]})
      if (ev) cudaEventDestroy(ev);
    if (c->batch->s_ode) cudaStreamDestroy(c->batch->s_ode);
    delete c->batch;
    c->batch = nullptr;
  }
  if (c->s_setup) cudaStreamSynchronize(c->s_setup);
  for (cudaEvent_t ev : {c->ev0, c->ev1, c->evk0, c->evk1, c->ev_fork, c->ev_join, c->ev_lists})
    if (ev) cudaEventDestroy(ev);
  if (c->s_setup) cudaStreamDestroy(c->s_setup);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int uwb_device_info(uwb_ctx* c, int* sm_count, int* cc_major, int* cc_minor) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return uwb_device_info(c->subs[0], sm_count, cc_major, cc_minor);
  if (sm_count) *sm_count = c->sm_count;
  if (cc_major) *cc_major = c->cc_major;
  if (cc_minor) *cc_minor = c->cc_minor;
  return UWB_OK;
}

int uwb_set_channel_subset(uwb_ctx* c, int n, const int* channels) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return set_err(UWB_CONFIG_ERROR, "a multi-GPU context partitions the channels itself");
  c->subset.assign(channels, channels + std::max(n, 0));
  if (n > 0 && !channels) return set_err(UWB_CONFIG_ERROR, "null channel list");
  return UWB_OK;
}

int uwb_all_channels_nli(uwb_ctx* c, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                         const double beta[3], const double* gamma, const uwb_nli_cfg* cfg,
                         uwb_nli_result* out) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return multi_all_channels_nli(c, grid, n_spans, spans, beta, gamma, cfg, out);
  cudaSetDevice(c->device);
  release_link_state(c);  // shares buffers with the prepared evaluation
  reset_xfer(c);
  int rc = validate_grid(grid);
  if (rc) return rc;
  NliParams P{};
  if ((rc = set_cfg(cfg, &P, c->precision))) return rc;
  if (!gamma) return set_err(UWB_CONFIG_ERROR, "missing per-channel gamma");
  std::vector<double> nu, gam;
  std::vector<int> cp;
  channel_probes(grid, gamma, cfg, c->subset, &nu, &gam, &cp);
  // Like the reference, an all-guard grid never reaches nli_psd_at's checks.
  if (!nu.empty()) {
    if ((rc = upload_path_inputs(c, grid, n_spans, spans, beta, &P))) return rc;
  } else {
    const int n = grid->n_ch;
    P.n_ch = n;
    P.psd = c->psd.get<double>(n);
    P.bch = grid->bch;
    xfer(c, const_cast<double*>(P.psd), grid->psd, n * sizeof(double),
                    cudaMemcpyHostToDevice, c->stream);
  }
  if ((rc = run_probes(c, P, cfg, nu, gam, &cp, true))) return rc;
  const int n = grid->n_ch;
  cudaStream_t st = c->stream;
  if (out) {
    if (out->eta) xfer(c, out->eta, c->eta.ptr<double>(), n * 8, cudaMemcpyDeviceToHost, st);
    if (out->nli_psd)
      xfer(c, out->nli_psd, c->nli_psd.ptr<double>(), n * 8, cudaMemcpyDeviceToHost, st);
    if (out->nli_power)
      xfer(c, out->nli_power, c->nli_power.ptr<double>(), n * 8, cudaMemcpyDeviceToHost, st);
    if (out->quadrant)
      xfer(c, out->quadrant, c->quad.ptr<double>(), n * 32, cudaMemcpyDeviceToHost, st);
    if (out->skipped)
      xfer(c, out->skipped, c->skipped.ptr<uint8_t>(), n, cudaMemcpyDeviceToHost, st);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "all_channels_nli");
  if (out) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    out->elapsed_seconds = ms * 1e-3;
  }
  return UWB_OK;
}

int uwb_nli_psd_at(uwb_ctx* c, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                   const double beta[3], const uwb_nli_cfg* cfg, int n_probe, const double* nu,
                   const double* gamma, double* out, double* quadrant4) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi())
    return uwb_nli_psd_at(c->subs[0], grid, n_spans, spans, beta, cfg, n_probe, nu, gamma, out, quadrant4);
  cudaSetDevice(c->device);
  release_link_state(c);
  reset_xfer(c);
  int rc = validate_grid(grid);
  if (rc) return rc;
  NliParams P{};
  if ((rc = upload_path_inputs(c, grid, n_spans, spans, beta, &P))) return rc;
  if ((rc = set_cfg(cfg, &P, c->precision))) return rc;
  if (n_probe <= 0) return UWB_OK;
  std::vector<double> vnu(nu, nu + n_probe), vg(gamma, gamma + n_probe);
  if ((rc = run_probes(c, P, cfg, vnu, vg, nullptr, true))) return rc;
  cudaStream_t st = c->stream;
  if (out) xfer(c, out, c->probe_g.ptr<double>(), n_probe * 8, cudaMemcpyDeviceToHost, st);
  if (quadrant4)
    xfer(c, quadrant4, c->probe_quad.ptr<double>(), n_probe * 32, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "nli_psd_at");
  return UWB_OK;
}

int uwb_channel_nli(uwb_ctx* c, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                    const double beta[3], double gamma_ch, const uwb_nli_cfg* cfg, int ch,
                    double* out, double* quadrant4) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (!grid || ch < 0 || ch >= grid->n_ch) return set_err(UWB_CONFIG_ERROR, "channel out of range");
  if (!cfg) return set_err(UWB_CONFIG_ERROR, "missing solver config");
  const double f = grid->freq[ch];
  double nu[3] = {f, f - 0.5 * grid->bch, f + 0.5 * grid->bch};
  double g3[3] = {gamma_ch, gamma_ch, gamma_ch};
  double res[3] = {0, 0, 0};
  double q12[12];
  const int np = cfg->simpson ? 3 : 1;
  int rc = uwb_nli_psd_at(c, grid, n_spans, spans, beta, cfg, np, nu, g3, res, q12);
  if (rc) return rc;
  double psd_c = res[0];
  if (cfg->simpson) psd_c = (res[1] + 4.0 * psd_c + res[2]) / 6.0;
  if (out) *out = psd_c;
  if (quadrant4) std::memcpy(quadrant4, q12, 4 * sizeof(double));
  return UWB_OK;
}

int uwb_last_launch_count(uwb_ctx* c) {
  if (!c) return 0;
  return c->multi() ? c->subs[0]->last_launches : c->last_launches;
}

int uwb_last_nli_stats(uwb_ctx* c, double* kernel_ms, double* inner_steps,
                       double* evaluated_points) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) {  // max kernel time over devices, summed work
    double km = 0.0, st = 0.0, pt = 0.0;
    for (uwb_ctx* s : c->subs) {
      double a = 0.0, b = 0.0, d = 0.0;
      uwb_last_nli_stats(s, &a, &b, &d);
      km = std::max(km, a);
      st += b;
      pt += d;
    }
    c->last_active = 0.0;
    for (uwb_ctx* s : c->subs) c->last_active += s->last_active;
    if (kernel_ms) *kernel_ms = km;
    if (inner_steps) *inner_steps = st;
    if (evaluated_points) *evaluated_points = pt;
    return UWB_OK;
  }
  // Resolved lazily from the events/counter of the last integrand launch (the
  // caller has synchronised), so the resident path pays nothing per call.
  if (c->nli_events_valid) {
    float ms = 0.f;
    if (cudaEventSynchronize(c->evk1) == cudaSuccess &&
        cudaEventElapsedTime(&ms, c->evk0, c->evk1) == cudaSuccess)
      c->last_kernel_ms = ms;
    const unsigned long long* d_ne = c->n_eval.ptr<unsigned long long>();
    unsigned long long ne[2] = {0, 0};
    if (d_ne) cudaMemcpy(ne, d_ne, sizeof ne, cudaMemcpyDeviceToHost);
    c->last_points = static_cast<double>(ne[0]);
    c->last_active = static_cast<double>(ne[1]);
    c->last_inner_steps = static_cast<double>(ne[0]) * c->last_total_steps;
  }
  if (kernel_ms) *kernel_ms = c->last_kernel_ms;
  if (inner_steps) *inner_steps = c->last_inner_steps;
  if (evaluated_points) *evaluated_points = c->last_points;
  return UWB_OK;
}

int uwb_last_nli_active(uwb_ctx* c, double* active_points) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (active_points) *active_points = c->last_active;  // resolved by uwb_last_nli_stats
  return UWB_OK;
}

int uwb_last_transfer_bytes(uwb_ctx* c, unsigned long long* h2d, unsigned long long* d2h) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return uwb_last_transfer_bytes(c->subs[0], h2d, d2h);
  if (h2d) *h2d = c->h2d_bytes;
  if (d2h) *d2h = c->d2h_bytes;
  return UWB_OK;
}

int uwb_set_precision(uwb_ctx* c, int mode) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  for (uwb_ctx* s : c->subs) uwb_set_precision(s, mode);
  for (uwb_ctx* s : c->bsubs) uwb_set_precision(s, mode);
  if (mode != UWB_PRECISION_FP64 && mode != UWB_PRECISION_MIXED)
    return set_err(UWB_CONFIG_ERROR, "uwb_set_precision: unknown mode");
  c->precision = mode;
  return UWB_OK;
}

int uwb_set_ode_stepping(uwb_ctx* c, int mode) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  for (uwb_ctx* s : c->subs) uwb_set_ode_stepping(s, mode);
  for (uwb_ctx* s : c->bsubs) uwb_set_ode_stepping(s, mode);
  if (mode != UWB_ODE_RESTART && mode != UWB_ODE_CONTINUOUS)
    return set_err(UWB_CONFIG_ERROR, "uwb_set_ode_stepping: unknown mode");
  c->ode_continuous = mode == UWB_ODE_CONTINUOUS ? 1 : 0;
  return UWB_OK;
}

int uwb_debug_bounds(int* nli_line, int* ode_line) {
  if (nli_line) *nli_line = nli_bounds_status();
  if (ode_line) *ode_line = ode_bounds_status();
  return UWB_OK;
}

int uwb_fp64_peak(uwb_ctx* c, double* tflops) {
  if (!c) return set_err(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return uwb_fp64_peak(c->subs[0], tflops);
  cudaSetDevice(c->device);
  const double t = fp64_fma_peak_tflops(c->sm_count, c->stream);
  if (!(t > 0)) return set_err(UWB_CUDA_ERROR, "fp64 microbenchmark failed");
  if (tflops) *tflops = t;
  return UWB_OK;
}

}  // extern "C"
