// Full SNR evaluation on the device: evaluate_link (link_optimizer.hpp:241-245)
// = build_distance_grid (host, 113 numbers) + Raman ODE (raman_ode.cu) + NLI
// (nli_kernel.cu) + assemble_link_report (link_optimizer.hpp:194-237, here).
// Also the C-ABI entry points uwb_power_evolution / uwb_evaluate_link /
// uwb_evaluate_link_prepare / uwb_evaluate_link_resident.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/uwb_nli.h"
#include "nli_kernel.cuh"
#include "raman_ode.cuh"
#include "uwb_capi_internal.cuh"
#include "uwb_ctx.cuh"
#include "uwb_devmath.cuh"
#include "uwb_link.cuh"
#include "uwb_multi.cuh"

namespace uwb {

namespace {

constexpr double kPlanck = 6.62607015e-34;  // units.hpp:10



// Per-channel part of assemble_link_report (link_optimizer.hpp:206-224).
__global__ void link_channels_kernel(LinkDev L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n) return;
  double* eta_o = L.out;
  double* pase_o = L.out + L.n;
  double* snr_o = L.out + 2 * L.n;
  double* cap_o = L.out + 3 * L.n;
  eta_o[i] = pase_o[i] = snr_o[i] = cap_o[i] = 0.0;
  L.tmp[i] = L.tmp[L.n + i] = L.tmp[2 * L.n + i] = 0.0;
  if (L.guard[i] || L.psd[i] <= 0.0) {
    L.tmp[i] = -1.0;  // marker: not an active channel
    return;
  }
  const double p = L.psd[i] * L.bch;
  const double eta = L.eta[i];
  const double gain = 1.0 / L.rho_end[i];
  const double nf = L.nf_db[i];
  // ase_power (link_optimizer.hpp:22-26) with max(gain, 1)
  const double g1 = gain > 1.0 ? gain : 1.0;
  const double n_sp = 0.5 * pow(10.0, nf / 10.0);
  const double pase =
      static_cast<double>(L.span_count) * (2.0 * n_sp * kPlanck * L.freq[i] * (g1 - 1.0) * L.bch);
  double denom = eta * p * p * p + pase;
  if (L.use_snr_trx) denom += p / L.snr_trx;
  const double snr = p / denom;
  eta_o[i] = eta;
  pase_o[i] = pase;
  snr_o[i] = 10.0 * log10(snr);
  const double l2 = log2(1.0 + snr);
  cap_o[i] = 2.0 * L.bch * l2;
  L.tmp[i] = p;
  L.tmp[L.n + i] = cap_o[i];
  L.tmp[2 * L.n + i] = l2;
}

// Link totals (loss, capacity, total and per-band power, :224-235).  One
// warp per sum: lane l adds a contiguous run of channels in ascending order,
// then a fixed xor-shuffle tree combines the 32 partials.  The order is fixed
// (results are reproducible and identical on every path) but it is not the
// reference's single sequential loop, so totals agree with the reference to
// rounding (~1e-16 relative), not bit for bit.  Warp 0: loss, capacity, total
// power; warp 1 + b: band b (bands beyond the warps loop).
constexpr int kTotalsThreads = 256;

__device__ __forceinline__ double warp_sum_fixed(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kTotalsThreads) link_totals_kernel(LinkDev L) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int n = L.n;
  const int run = (n + 31) / 32;
  const int i0 = lane * run, i1 = min(n, i0 + run);
  const double* tp = L.tmp;           // p (< 0: inactive)
  const double* tc = L.tmp + n;       // capacity
  const double* tl = L.tmp + 2 * n;   // log2(1 + snr)
  if (warp == 0) {
    double loss = 0.0, cap = 0.0, total_w = 0.0;
    for (int i = i0; i < i1; ++i) {
      const double p = tp[i];
      const bool act = p >= 0.0;
      loss -= act ? tl[i] : 0.0;
      cap += act ? tc[i] : 0.0;
      total_w += act ? p : 0.0;
    }
    loss = warp_sum_fixed(loss);
    cap = warp_sum_fixed(cap);
    total_w = warp_sum_fixed(total_w);
    if (lane == 0) {
      L.out[4 * n + 0] = loss;
      L.out[4 * n + 1] = cap;
      L.out[4 * n + 2] = total_w > 0.0 ? 10.0 * log10(total_w / 1e-3) : -300.0;
    }
    return;
  }
  double* op = L.out + 4 * n + 3;
  double* oc = op + L.n_bands;
  for (int b = warp - 1; b < L.n_bands; b += nw - 1) {
    double bp = 0.0, bc = 0.0;
    for (int i = i0; i < i1; ++i) {
      const bool in = tp[i] >= 0.0 && L.band && L.band[i] == b;
      bp += in ? tp[i] : 0.0;
      bc += in ? tc[i] : 0.0;
    }
    bp = warp_sum_fixed(bp);
    bc = warp_sum_fixed(bc);
    if (lane == 0) {
      op[b] = bp > 0.0 ? 10.0 * log10(bp / 1e-3) : -300.0;
      oc[b] = bc;
    }
  }
}

}  // namespace

// build_distance_grid (distance_grid.hpp:23-73), host: 113 numbers.
int distance_grid_host(double length_m, double density, std::vector<double>* edge,
                  std::vector<double>* mid, std::vector<double>* width) {
  if (!(length_m > 0.0)) return fail(UWB_CONFIG_ERROR, "build_distance_grid: length must be > 0");
  if (!(density > 0.0)) return fail(UWB_CONFIG_ERROR, "build_distance_grid: density must be > 0");
  long n_edges = std::lround(density * length_m / 1e3) + 1;
  if (n_edges < 2) n_edges = 2;
  const size_t n = static_cast<size_t>(n_edges);
  const double n_steps = static_cast<double>(n - 1);
  edge->assign(n, 0.0);
  const double uniform_step = length_m / n_steps;
  const double first_target = 1e3 / (10.0 * density);
  if (first_target >= uniform_step * 0.999) {
    for (size_t i = 0; i < n; ++i) (*edge)[i] = length_m * static_cast<double>(i) / n_steps;
  } else {
    auto first_step = [&](double z0) { return z0 * std::expm1(std::log1p(length_m / z0) / n_steps); };
    double lo = length_m * 1e-12, hi = length_m * 1e12;
    for (int it = 0; it < 200; ++it) {
      const double m = std::sqrt(lo * hi);
      (first_step(m) < first_target ? lo : hi) = m;
    }
    const double z0 = std::sqrt(lo * hi);
    const double t = std::log1p(length_m / z0);
    for (size_t i = 0; i < n; ++i) (*edge)[i] = z0 * std::expm1(t * static_cast<double>(i) / n_steps);
  }
  edge->front() = 0.0;
  edge->back() = length_m;
  mid->resize(n - 1);
  width->resize(n - 1);
  for (size_t i = 0; i + 1 < n; ++i) {
    (*mid)[i] = 0.5 * ((*edge)[i] + (*edge)[i + 1]);
    (*width)[i] = (*edge)[i + 1] - (*edge)[i];
  }
  return UWB_OK;
}

namespace {

// Host-to-device copy of n elements into the buffer b; while the context
// defers uploads (prepare) the bytes are staged and go with the next flush.
void stage_upload(uwb_ctx* c, void* dst, const void* src, size_t bytes) {
  if (!c->up_defer) {
    xfer(c, dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
    return;
  }
  const size_t off = (c->up_host.size() + 15) & ~static_cast<size_t>(15);
  c->up_host.resize(off + bytes);
  std::memcpy(c->up_host.data() + off, src, bytes);
  c->up_segs.push_back({dst, off, bytes});
}

template <class T>
T* up(uwb_ctx* c, DBuf& b, const T* src, size_t n) {
  T* d = b.get<T>(std::max<size_t>(n, 1));
  if (d && src && n) stage_upload(c, d, src, n * sizeof(T));
  return d;
}

constexpr int kMaxScatter = 32;
struct ScatterDesc {
  int n;
  unsigned char* dst[kMaxScatter];
  unsigned off[kMaxScatter];
  unsigned bytes[kMaxScatter];
};

// one CTA per staged segment: 8-byte words where both ends are aligned (every
// double / int array), bytes otherwise (the guard flags)
__global__ void scatter_uploads_kernel(const unsigned char* src, ScatterDesc d) {
  const int s = blockIdx.x;
  if (s >= d.n) return;
  unsigned char* dst = d.dst[s];
  const unsigned char* p = src + d.off[s];
  const unsigned nb = d.bytes[s];
  if (((reinterpret_cast<uintptr_t>(dst) | d.off[s] | nb) & 7u) == 0) {
    for (unsigned i = threadIdx.x; i < nb / 8; i += blockDim.x)
      reinterpret_cast<unsigned long long*>(dst)[i] = reinterpret_cast<const unsigned long long*>(p)[i];
  } else {
    for (unsigned i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = p[i];
  }
}

// Issue the staged uploads: one pinned host-to-device copy, one scatter launch
// per 32 segments.  Clears the staging and the deferral.
int flush_uploads(uwb_ctx* c) {
  c->up_defer = false;
  const size_t total = c->up_host.size();
  int rc = UWB_OK;
  if (total) {
    if (c->up_pinned_cap < total) {
      if (c->up_pinned) cudaFreeHost(c->up_pinned);
      c->up_pinned = nullptr;
      c->up_pinned_cap = 0;
      if (cudaMallocHost(&c->up_pinned, total) != cudaSuccess) rc = fail(UWB_CUDA_ERROR, "pinned alloc");
      else c->up_pinned_cap = total;
    }
    unsigned char* dev = c->up_dev.get<unsigned char>(total);
    if (!rc && !dev) rc = fail(UWB_CUDA_ERROR, "device allocation failed");
    if (!rc) {
      std::memcpy(c->up_pinned, c->up_host.data(), total);
      xfer(c, dev, c->up_pinned, total, cudaMemcpyHostToDevice, c->stream);
      for (size_t b = 0; b < c->up_segs.size(); b += kMaxScatter) {
        ScatterDesc d{};
        d.n = static_cast<int>(std::min<size_t>(kMaxScatter, c->up_segs.size() - b));
        for (int k = 0; k < d.n; ++k) {
          const uwb_ctx::UpSeg& u = c->up_segs[b + k];
          d.dst[k] = static_cast<unsigned char*>(u.dst);
          d.off[k] = static_cast<unsigned>(u.off);
          d.bytes[k] = static_cast<unsigned>(u.bytes);
        }
        scatter_uploads_kernel<<<d.n, 128, 0, c->stream>>>(dev, d);
      }
    }
  }
  c->up_host.clear();
  c->up_segs.clear();
  return rc;
}

// Defers the context's uploads for a scope; an early return drops them.
struct UploadBatch {
  uwb_ctx* c;
  explicit UploadBatch(uwb_ctx* cc) : c(cc) {
    c->up_defer = true;
    c->up_host.clear();
    c->up_segs.clear();
  }
  ~UploadBatch() {
    c->up_defer = false;
    c->up_host.clear();
    c->up_segs.clear();
  }
};

}  // namespace

// Everything evaluate_link keeps resident between calls.
}  // namespace uwb


namespace uwb {

void release_link_state(uwb_ctx* c) {
  if (!c->prep) return;
  delete c->prep;
  c->prep = nullptr;
}

int prepare(uwb_ctx* c, const uwb_grid* g, const uwb_fibre* fb, const uwb_link_cfg* lk,
            const uwb_nli_cfg* cfg, bool sync) {
  UploadBatch uploads(c);  // every host array of the link goes with one transfer
  // the buffers below are shared with the previous prepared link: it is gone
  // from here on, and the new one is published only once complete
  release_link_state(c);
  int rc = validate_grid_full(g);  // solve_power_evolution's grid.validate() (raman_power.hpp:56)
  if (rc) return rc;
  if (!fb || !lk || !cfg) return fail(UWB_CONFIG_ERROR, "missing fibre / link / solver config");
  if (!fb->alpha || !fb->aeff || !fb->gamma || !lk->nf_db)
    return fail(UWB_CONFIG_ERROR, "missing per-channel fibre arrays");
  if (fb->span_count < 1) return fail(UWB_CONFIG_ERROR, "span count must be >= 1");
  if (lk->include_raman && (fb->raman_n < 2 || !fb->raman_x || !fb->raman_y))
    return fail(UWB_CONFIG_ERROR, "raman gain: table needs at least two (x, y) rows");
  std::vector<double> edge, mid, width;
  if ((rc = distance_grid_host(fb->length_m, lk->density, &edge, &mid, &width))) return rc;
  const int steps = static_cast<int>(mid.size());
  if (steps > kMaxSteps)
    return fail(UWB_CONFIG_ERROR, "uwb: distance steps per span must be in [1, 65536]");
  const int n = g->n_ch;
  std::unique_ptr<uwb_ctx::Prepared> owner(new uwb_ctx::Prepared());
  uwb_ctx::Prepared* pr = owner.get();
  pr->n = n;
  pr->steps = steps;
  pr->span_count = fb->span_count;
  pr->include_raman = lk->include_raman;
  pr->rtol = lk->rtol > 0 ? lk->rtol : 1e-9;
  pr->atol = lk->atol > 0 ? lk->atol : 1e-16;
  pr->length = fb->length_m;
  pr->cfg = *cfg;
  NliParams& P = pr->P;
  if ((rc = set_cfg(cfg, &P, c->precision))) return rc;

  // static uploads
  const double* d_freq = up(c, c->freq, g->freq, n);
  pr->d_psd = up(c, c->psd, g->psd, n);
  const uint8_t* d_guard = up(c, c->guard, g->guard, n);
  const double* d_alpha = up(c, c->alpha, fb->alpha, n);
  pr->d_aeff = up(c, c->aeff, fb->aeff, n);
  pr->raman_n = fb->raman_n;
  pr->aeff_ref = fb->raman_aeff_ref;
  const double* d_nf = up(c, c->nf_db, lk->nf_db, n);
  std::vector<int> band(n, -1);
  if (lk->band) std::copy(lk->band, lk->band + n, band.begin());
  const double* d_mid = up(c, c->mid, mid.data(), mid.size());
  // span-absolute grids: every span is a copy of the one evolution
  // (solve_link_noise :185); padded layout of nli_kernel.cuh
  const int NS = 16 * ((steps + 15) / 16);
  SpanTables st;
  double z_base = 0.0;
  for (int k = 0; k < fb->span_count; ++k) {
    append_span_tables(edge.data(), mid.data(), width.data(), steps, z_base, &st);
    z_base += fb->length_m;
  }
  P.n_ch = n;
  P.freq = d_freq;
  P.psd = pr->d_psd;
  P.spacing = g->spacing;
  P.inv_spacing = 1.0 / g->spacing;
  P.bch = g->bch;
  P.centre = g->centre;
  P.half_band = g->half_band;
  P.n_spans = fb->span_count;
  P.steps = steps;
  const size_t cols = static_cast<size_t>(n + 1) * NS;
  P.log2rho = c->log2rho.get<double>(cols);
  cudaMemsetAsync(const_cast<double*>(P.log2rho), 0, cols * sizeof(double), c->stream);  // pads
  P.col_stride = NS;
  P.span_stride = 0;
  P.zedge = up(c, c->zedge, st.zend.data(), st.zend.size());
  P.zstart = up(c, c->zstart, st.zstart.data(), st.zstart.size());
  P.zmid_max = st.zmid_max;
  P.slow_tiny = slow_tiny_ok(st) ? 1 : 0;
  P.zmid = up(c, c->zmid, st.zmid.data(), st.zmid.size());
  P.width = up(c, c->width, st.width.data(), st.width.size());
  P.wlast = up(c, c->wlast, st.wlast.data(), st.wlast.size());
  P.beta2 = fb->beta[0];
  P.beta3 = fb->beta[1];
  P.beta4 = fb->beta[2];
  c->last_total_steps = static_cast<double>(steps) * fb->span_count;

  // Probes: every non-guard channel of the subset, lit or dark.  The
  // reference re-derives its skip set (guard or psd <= 0, gn_integral.hpp:
  // 349-352) on every call; the resident path takes a new launch profile per
  // call, so the device re-derives it too: rows of a probe whose channel is
  // dark in THIS evaluation exit at once (NliParams::probe_chan) and
  // finalize_channels_kernel reports the channel skipped.  A channel dark at
  // prepare time may therefore light up later and gets its NLI.  (The grid is
  // validated, so every channel lies inside the half band: no quadrant_limits
  // error can depend on the launch profile.)
  std::vector<double> nu, gam;
  std::vector<int> cp, pch;
  channel_probes(g, fb->gamma, cfg, c->subset, &nu, &gam, &cp, /*include_dark=*/true, &pch);
  for (double v : nu)
    if (std::abs(v - g->centre) > g->half_band)
      return fail(UWB_CONFIG_ERROR, "quadrant_limits: channel offset must lie inside the half band");
  const int np = static_cast<int>(nu.size());
  P.n_probes = np;
  P.total_rows = np * P.n_q * P.n_r;
  P.probe_nu = up(c, c->probe_nu, nu.data(), nu.size());
  P.probe_chan = up(c, c->probe_chan, pch.data(), pch.size());
  P.hl2 = c->hl2.get<double>(static_cast<size_t>(std::max(np, 1)) * P.n_spans * NS);
  P.rowsum = c->rowsum.get<double>(std::max(P.total_rows, 1));
  P.rowpar = c->rowpar.get<double>(4 * static_cast<size_t>(std::max(P.total_rows, 1)));
  P.counter = c->counter.get<unsigned int>(1);
  P.n_eval = c->n_eval.get<unsigned long long>(2);
  P.n_active = P.n_eval + 1;
  P.probe_work = c->probe_work.get<unsigned long long>(std::max(np, 1));
  P.rowcnt = c->rowcnt.get<uint2>(std::max(P.total_rows, 1));
  c->last_n_probes = np;
  c->last_probes_per_chan = cfg->simpson ? 3 : 1;
  c->last_chan_probe0 = cp;
  FinalizeParams& F = pr->F;
  F.n_probes = np;
  F.probe_gamma = up(c, c->probe_gamma, gam.data(), gam.size());
  F.probe_g = c->probe_g.get<double>(std::max(np, 1));
  F.probe_quad = c->probe_quad.get<double>(4 * std::max(np, 1));
  F.mirror_q4 = cfg->mirror_q4 ? 1 : 0;
  F.n_ch = n;
  F.psd = pr->d_psd;
  F.bch = g->bch;
  F.simpson = cfg->simpson ? 1 : 0;
  F.chan_probe0 = up(c, c->chan_probe0, cp.data(), cp.size());
  F.eta = c->eta.get<double>(n);
  F.nli_psd = c->nli_psd.get<double>(n);
  F.nli_power = c->nli_power.get<double>(n);
  F.quad = c->quad.get<double>(4 * n);
  F.skipped = c->skipped.get<uint8_t>(n);

  // ODE (raman_ode.cu): separable coupling factors + gain-table segments
  OdeParams& O = pr->O;
  O.n = n;
  O.raman = lk->include_raman ? 1 : 0;
  O.alpha = d_alpha;
  if (O.raman && raman_segments(fb->raman_x, fb->raman_y, fb->raman_n, g->spacing, n, &O))
    return fail(UWB_CONFIG_ERROR, "raman gain table has too many linear pieces");
  if (n > kMaxOdeChannels) return fail(UWB_CONFIG_ERROR, "uwb: at most 7168 channels");
  // global fallback for the ODE's running-sum arrays (combs too wide for
  // shared memory), two halves for the overlapped batch's two ODEs in flight
  const size_t gw = ode_gwork_double2(n);
  O.gwork = c->ode_gwork.get<double2>(2 * gw);
  if (!O.gwork) return fail(UWB_CUDA_ERROR, "device allocation failed");
  // ode_work: coef a|u|v [3n] | rho_end [n] | status, rhs [2] | band [n ints] | link tmp [3n]
  double* w = c->ode_work.get<double>(3 * static_cast<size_t>(n) + n + 2 + n + 3 * n + 8);
  if (!w) return fail(UWB_CUDA_ERROR, "device allocation failed");
  O.coef_a = w;
  O.coef_u = w + n;
  O.coef_v = w + 2 * n;
  double* d_rho_end = w + 3 * n;
  pr->d_status = reinterpret_cast<int*>(w + 4 * n);
  pr->d_rhs = reinterpret_cast<long long*>(w + 4 * n + 1);
  int* d_band2 = reinterpret_cast<int*>(w + 4 * n + 2);
  double* d_tmp = w + 5 * n + 2;
  O.steps = steps;
  O.col_stride = NS;
  O.lane_k = NS / 16;
  O.mid = d_mid;
  O.length = fb->length_m;
  O.rtol = pr->rtol;
  O.atol = pr->atol;
  O.continuous = c->ode_continuous;
  O.log2rho = const_cast<double*>(P.log2rho);
  O.log_rho = nullptr;
  O.rho_end = d_rho_end;
  O.status = pr->d_status;
  O.rhs_evals = pr->d_rhs;
  stage_upload(c, d_band2, band.data(), n * sizeof(int));

  // assembly
  LinkDev& L = pr->L;
  L.n = n;
  L.freq = d_freq;
  L.psd = pr->d_psd;
  L.guard = d_guard;
  L.bch = g->bch;
  L.eta = F.eta;
  L.rho_end = d_rho_end;
  L.nf_db = d_nf;
  L.band = d_band2;
  L.n_bands = std::max(lk->n_bands, 0);
  L.span_count = fb->span_count;
  L.use_snr_trx = lk->use_snr_trx;
  L.snr_trx = lk->use_snr_trx ? std::pow(10.0, lk->snr_trx_db / 10.0) : 0.0;
  L.out = c->report.get<double>(4 * static_cast<size_t>(n) + 3 + 2 * L.n_bands);
  L.tmp = d_tmp;

  const int per_sm = nli_ctas_per_sm(steps, P.n_spans == 1, P.n_r, P.mixed != 0, P.slow_tiny != 0);
  if (per_sm <= 0) return fail(UWB_CUDA_ERROR, "integrand kernel cannot be resident");
  pr->grid_ctas = c->sm_count * per_sm;
  // Split evaluation: the rows' point setup runs beside the Raman ODE (which
  // holds one SM for ~2 ms) and the integrand proper only walks the listed
  // points.  One record slot per (row, column), allocated by
  // the first single evaluation (batches keep the fused kernel); the fused
  // kernel when the lists exceed the budget (UWB_NLI_SPLIT_MB, default 8 GB).
  P.plist = nullptr;
  P.plist_n = nullptr;
  pr->setup_ctas = 0;
  pr->list_ctas = 0;
  pr->split_bytes = 0;
  if (nli_split_ok(P) && P.total_rows > 0) {
    static const double budget_mb = [] {
      const char* e = std::getenv("UWB_NLI_SPLIT_MB");
      return e ? std::atof(e) : 8192.0;
    }();
    const size_t bytes = static_cast<size_t>(P.total_rows) * P.n_r * nli_point_record_bytes();
    const int sp = nli_setup_ctas_per_sm();
    const int lp = nli_list_ctas_per_sm(P);
    if (sp > 0 && lp > 0 && static_cast<double>(bytes) <= budget_mb * 1048576.0) {
      pr->list_ctas = c->sm_count * lp;
      static const int setup_env = [] {  // UWB_NLI_SETUP_CTAS: the setup pass's grid (A/B)
        const char* e = std::getenv("UWB_NLI_SETUP_CTAS");
        return e ? std::atoi(e) : 0;
      }();
      // two CTAs per SM, the ODE's SM left alone: the third resident CTA per
      // SM slowed the concurrent ODE by 4 % (profiles/r02_integrand_experiments.md)
      pr->setup_ctas = setup_env > 0 ? setup_env : std::max(1, c->sm_count - 1) * std::min(sp, 2);
      pr->split_bytes = bytes;
    }
  }
  if (!P.log2rho || !P.zedge || !P.zstart || !P.zmid || !P.width || !P.wlast || !P.probe_nu ||
      !P.probe_chan || !P.hl2 || !P.rowsum || !P.rowpar || !P.counter || !P.n_eval || !P.probe_work || !P.rowcnt ||
      !F.probe_gamma ||
      !F.probe_g || !F.probe_quad || !F.chan_probe0 || !F.eta || !F.nli_psd || !F.nli_power ||
      !F.quad || !F.skipped || !L.out || !d_freq || !pr->d_psd || !d_guard || !d_alpha ||
      !pr->d_aeff || !d_nf || !d_mid)
    return fail(UWB_CUDA_ERROR, "device allocation failed");
  if ((rc = flush_uploads(c))) return rc;
  cudaError_t e = sync ? cudaStreamSynchronize(c->stream) : cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "prepare");
  c->prep = owner.release();  // complete: publish
  return UWB_OK;
}

// Noise stage of one evaluation on the prepared state (solve_link_noise,
// link_optimizer.hpp:181-190): Raman ODE + NLI for the context's channels.
// psd_dev = launch PSD (device) or null to keep the prepared one.
int run_noise(uwb_ctx* c, const double* psd_dev, cudaStream_t st, bool reset_status) {
  uwb_ctx::Prepared* pr = c->prep;
  int launches = 0;
  if (psd_dev && psd_dev != pr->d_psd)
    xfer(c, pr->d_psd, psd_dev, pr->n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  // (a batch keeps the first failure: atomicExch writes are never cleared)
  if (reset_status) cudaMemsetAsync(pr->d_status, 0, sizeof(int), st);
  cudaEventRecord(c->ev0, st);
  if (pr->split_bytes && !pr->P.plist && pr->P.n_probes > 0) {
    pr->P.plist = c->plist.get<unsigned char>(pr->split_bytes);
    pr->P.plist_n = c->plist_n.get<int>(pr->P.total_rows);
    if (!pr->P.plist || !pr->P.plist_n) {  // out of memory: the fused kernel from now on
      cudaGetLastError();
      pr->P.plist = nullptr;
      pr->P.plist_n = nullptr;
      pr->split_bytes = 0;
    }
  }
  const bool split = pr->P.plist && pr->P.n_probes > 0;
  if (split) {
    if (!c->s_setup) {
      cudaError_t e = cudaStreamCreateWithFlags(&c->s_setup, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_lists, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(e, "split evaluation stream");
    }
    cudaEventRecord(c->ev_fork, st);  // the PSD copy and status reset above come first
  }
  const int lo = launch_raman_ode(pr->O, pr->P.freq, pr->d_psd, pr->P.bch, pr->d_aeff,
                                  pr->aeff_ref, st);
  if (lo < 0) return fail(UWB_CUDA_ERROR, "raman ODE launch failed");
  launches += lo;
  if (split) {
    cudaStreamWaitEvent(c->s_setup, c->ev_fork, 0);
    // the previous list pass may have run on another stream: it must be done
    // reading the point lists before this setup pass rewrites them
    cudaStreamWaitEvent(c->s_setup, c->ev_lists, 0);
    const int ls = launch_nli_setup(pr->P, pr->setup_ctas, c->s_setup);
    if (ls < 0) return fail(UWB_CONFIG_ERROR, "unsupported step count");
    cudaEventRecord(c->ev_join, c->s_setup);
    cudaStreamWaitEvent(st, c->ev_join, 0);
    const int ln = launch_nli_lists(pr->P, pr->F, pr->list_ctas, st, c->evk0, c->evk1);
    if (ln < 0) return fail(UWB_CONFIG_ERROR, "unsupported step count");
    cudaEventRecord(c->ev_lists, st);
    launches += ls + ln;
    c->nli_events_valid = true;
  } else if (pr->P.n_probes > 0) {
    const int ln = launch_nli(pr->P, pr->F, pr->grid_ctas, st, c->evk0, c->evk1);
    if (ln < 0) return fail(UWB_CONFIG_ERROR, "unsupported step count");
    launches += ln;
    c->nli_events_valid = true;
  } else {
    launches += launch_finalize_channels_only(pr->F, st);
    c->nli_events_valid = false;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "evaluate_link launch");
  c->last_launches = launches;
  return UWB_OK;
}

// Report stage (assemble_link_report, link_optimizer.hpp:194-237).
int run_report(uwb_ctx* c, cudaStream_t st, const LinkDev* Lp) {
  LinkDev L = Lp ? *Lp : c->prep->L;
  link_channels_kernel<<<(L.n + 127) / 128, 128, 0, st>>>(L);
  link_totals_kernel<<<1, kTotalsThreads, 0, st>>>(L);
  c->last_launches += 2;
  cudaEventRecord(c->ev1, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "assemble_link_report launch");
  return UWB_OK;
}

int run_prepared(uwb_ctx* c, const double* psd_dev, cudaStream_t st, bool reset_status) {
  int rc = run_noise(c, psd_dev, st, reset_status);
  if (rc) return rc;
  const int l = c->last_launches;
  rc = run_report(c, st);
  c->last_launches = l + 2;
  return rc;
}

int status_error(int status) {
  switch (status) {
    case 0: return UWB_OK;
    case 1: return fail(UWB_SOLVER_ERROR, "power evolution: non-positive rho");
    case 2: return fail(UWB_SOLVER_ERROR, "rk45: step budget exhausted");
    default: return fail(UWB_SOLVER_ERROR, "rk45: step size underflow");
  }
}

int check_status(uwb_ctx* c) {
  int status = 0;
  xfer_sync(c, &status, c->prep->d_status, sizeof(int), cudaMemcpyDeviceToHost);
  return status_error(status);
}

}  // namespace uwb

using namespace uwb;

extern "C" {

int uwb_evaluate_link_prepare(uwb_ctx* c, const uwb_grid* grid, const uwb_fibre* fibre,
                              const uwb_link_cfg* link, const uwb_nli_cfg* cfg) {
  if (!c) return fail(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return multi_prepare(c, grid, fibre, link, cfg, true);
  cudaSetDevice(c->device);
  return prepare(c, grid, fibre, link, cfg);
}

int uwb_evaluate_link_resident(uwb_ctx* c, const double* psd_dev, double* report_dev,
                               void* stream) {
  if (c && c->multi()) return multi_resident(c, psd_dev, report_dev, stream);
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  reset_xfer(c);
  int rc = run_prepared(c, psd_dev, st);
  if (rc) return rc;
  if (report_dev) {
    const size_t cnt = 4 * static_cast<size_t>(c->prep->n) + 3 + 2 * c->prep->L.n_bands;
    xfer(c, report_dev, c->prep->L.out, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  return UWB_OK;
}

static int ensure_batch_state(uwb_ctx* c) {
  if (c->batch) return UWB_OK;
  auto* B = new uwb_ctx::BatchState();
  // the ODE stream gets the highest priority: when the ODE of evaluation e + 1 and
  // the integrand of evaluation e become ready together, the block scheduler
  // places the one ODE CTA first and the integrand's CTAs fill around it
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  cudaError_t e = cudaStreamCreateWithPriority(&B->s_ode, cudaStreamNonBlocking, hi_prio);
  for (cudaEvent_t* ev : {&B->ev_start, &B->ev_ode[0], &B->ev_ode[1], &B->ev_nli[0], &B->ev_nli[1]})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  c->batch = B;
  if (e != cudaSuccess) return cuda_fail(e, "batch streams");
  return UWB_OK;
}

int uwb_evaluate_link_many(uwb_ctx* c, int n_eval, const double* psd_host, double* loss_host,
                           double* report_host) {
  if (c && c->multi()) return multi_many(c, n_eval, psd_host, loss_host, report_host);
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  if (n_eval < 0 || (n_eval > 0 && !psd_host)) return fail(UWB_CONFIG_ERROR, "bad batch");
  cudaSetDevice(c->device);
  reset_xfer(c);
  uwb_ctx::Prepared* pr = c->prep;
  const size_t n = pr->n;
  const size_t rl = 4 * n + 3 + 2 * pr->L.n_bands;
  if (n_eval == 0) return UWB_OK;
  double* d_psd = c->batch_psd.get<double>(n_eval * n);
  double* d_rep = c->batch_report.get<double>(n_eval * rl);
  if (!d_psd || !d_rep) return fail(UWB_CUDA_ERROR, "device allocation failed");
  cudaStream_t st = c->stream;
  xfer(c, d_psd, psd_host, n_eval * n * sizeof(double), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(pr->d_status, 0, sizeof(int), st);
  int launches = 0;
  static const bool serial = [] {  // UWB_BATCH_SERIAL=1: no ODE/NLI overlap (A/B)
    const char* e = std::getenv("UWB_BATCH_SERIAL");
    return e && e[0] == '1';
  }();
  if (n_eval >= 2 && pr->P.n_probes > 0 && !serial) {
    // Overlapped batch: the Raman ODE of evaluation e + 1 (one small CTA, on
    // its own stream) runs while the integrand of evaluation e occupies the
    // other SMs.  Two ODE output buffers alternate; the integrand grid leaves
    // one SM's worth of CTAs free, and the ODE runs its 224-register build
    // (7,168 registers per warp: it fits in an SM sub-partition beside one
    // integrand CTA's warps), so it finds room wherever the integrand's CTAs
    // were placed; the integrand's carveout leaves it shared memory.
    int rc = ensure_batch_state(c);
    if (rc) return rc;
    uwb_ctx::BatchState& B = *c->batch;
    const int per_sm = pr->grid_ctas / c->sm_count;
    static const int free_ctas = [] {  // UWB_BATCH_FREE: integrand CTAs left out (A/B)
      const char* e = std::getenv("UWB_BATCH_FREE");
      return e ? std::atoi(e) : -1;
    }();
    const int grid = std::max(1, pr->grid_ctas - (free_ctas >= 0 ? free_ctas : per_sm));
    NliParams Pb[2] = {pr->P, pr->P};
    Pb[0].probe_work = Pb[1].probe_work = nullptr;  // two evaluations in flight
    FinalizeParams Fb[2] = {pr->F, pr->F};
    OdeParams Ob[2] = {pr->O, pr->O};
    LinkDev Lb[2] = {pr->L, pr->L};
    const size_t tab = static_cast<size_t>(n + 1) * pr->P.col_stride;
    double* wb = c->batch_ode.get<double>(tab + 4 * n);
    if (!wb) return fail(UWB_CUDA_ERROR, "device allocation failed");
    cudaMemcpyAsync(wb, pr->P.log2rho, tab * sizeof(double), cudaMemcpyDeviceToDevice, st);  // pads
    Pb[1].log2rho = wb;
    Ob[1].log2rho = wb;
    Ob[1].rho_end = wb + tab;
    Lb[1].rho_end = wb + tab;
    Ob[1].coef_a = wb + tab + n;
    Ob[1].coef_u = wb + tab + 2 * n;
    Ob[1].coef_v = wb + tab + 3 * n;
    Ob[1].gwork = pr->O.gwork + ode_gwork_double2(static_cast<int>(n));
    // the ODE CTA must find its shared memory free on an SM that runs
    // integrand CTAs: the integrand's carveout leaves room for it
    const size_t ode_smem = raman_ode_smem_bytes(Ob[0]);
    cudaEventRecord(B.ev_start, st);
    cudaStreamWaitEvent(B.s_ode, B.ev_start, 0);  // uploads / status reset first
    for (int e = 0; e < n_eval; ++e) {
      const int b = e & 1;
      const double* psd_e = d_psd + e * n;
      Pb[b].psd = Fb[b].psd = Lb[b].psd = psd_e;
      if (e >= 2) cudaStreamWaitEvent(B.s_ode, B.ev_nli[b], 0);  // eval e-2 done with buffer b
      const int lo = launch_raman_ode(Ob[b], pr->P.freq, psd_e, pr->P.bch, pr->d_aeff, pr->aeff_ref,
                                      B.s_ode, /*coresident=*/true);
      if (lo < 0) return fail(UWB_CUDA_ERROR, "raman ODE launch failed");
      cudaEventRecord(B.ev_ode[b], B.s_ode);
      cudaStreamWaitEvent(st, B.ev_ode[b], 0);
      const int ln = launch_nli(Pb[b], Fb[b], grid, st, nullptr, nullptr, ode_smem);
      if (ln < 0) return fail(UWB_CONFIG_ERROR, "unsupported step count");
      if ((rc = run_report(c, st, &Lb[b]))) return rc;
      xfer(c, d_rep + e * rl, pr->L.out, rl * sizeof(double), cudaMemcpyDeviceToDevice, st);
      cudaEventRecord(B.ev_nli[b], st);
      launches += lo + ln + 2;
    }
  } else {
    for (int e = 0; e < n_eval; ++e) {
      int rc = run_prepared(c, d_psd + e * n, st, /*reset_status=*/false);
      if (rc) return rc;
      launches += c->last_launches;
      xfer(c, d_rep + e * rl, pr->L.out, rl * sizeof(double), cudaMemcpyDeviceToDevice, st);
    }
  }
  if (loss_host) {  // the loss of each report, one strided copy
    c->d2h_bytes += n_eval * sizeof(double);
    cudaMemcpy2DAsync(loss_host, sizeof(double), d_rep + 4 * n, rl * sizeof(double),
                      sizeof(double), n_eval, cudaMemcpyDeviceToHost, st);
  }
  if (report_host)
    xfer(c, report_host, d_rep, n_eval * rl * sizeof(double), cudaMemcpyDeviceToHost, st);
  c->last_launches = launches;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "evaluate_link_many");
  return check_status(c);
}

int uwb_evaluate_link(uwb_ctx* c, const uwb_grid* grid, const uwb_fibre* fibre,
                      const uwb_link_cfg* link, const uwb_nli_cfg* cfg, uwb_link_report* out) {
  if (!c) return fail(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return multi_evaluate_link(c, grid, fibre, link, cfg, out);
  cudaSetDevice(c->device);
  reset_xfer(c);
  int rc = prepare(c, grid, fibre, link, cfg, /*sync=*/false);  // same stream throughout
  if (rc) return rc;
  uwb_ctx::Prepared* pr = c->prep;
  if ((rc = run_prepared(c, nullptr, c->stream))) return rc;
  const int n = pr->n;
  cudaStream_t st = c->stream;
  // report, status word and work counters land in pinned staging: one
  // synchronisation for all of them
  const size_t rl = 4 * static_cast<size_t>(n) + 3 + 2 * pr->L.n_bands;
  const size_t need = (rl + 4) * sizeof(double);
  if (c->pinned_cap < need) {
    if (c->pinned) cudaFreeHost(c->pinned);
    c->pinned = nullptr;
    c->pinned_cap = 0;
    if (cudaMallocHost(&c->pinned, need) != cudaSuccess) return fail(UWB_CUDA_ERROR, "pinned alloc");
    c->pinned_cap = need;
  }
  double* rep = static_cast<double*>(c->pinned);
  int* status = reinterpret_cast<int*>(rep + rl);
  unsigned long long* ne = reinterpret_cast<unsigned long long*>(rep + rl + 1);
  xfer(c, rep, pr->L.out, rl * sizeof(double), cudaMemcpyDeviceToHost, st);
  xfer(c, status, pr->d_status, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (pr->P.n_probes > 0)
    xfer(c, ne, pr->P.n_eval, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (out && out->rho_end)
    xfer(c, out->rho_end, pr->O.rho_end, n * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "evaluate_link");
  if ((rc = status_error(*status))) return rc;
  if (out) {
    if (out->eta) std::memcpy(out->eta, rep, n * sizeof(double));
    if (out->p_ase) std::memcpy(out->p_ase, rep + n, n * sizeof(double));
    if (out->snr_db) std::memcpy(out->snr_db, rep + 2 * n, n * sizeof(double));
    if (out->capacity) std::memcpy(out->capacity, rep + 3 * n, n * sizeof(double));
    out->loss_value = rep[4 * n];
    out->total_capacity = rep[4 * n + 1];
    out->total_power_dbm = rep[4 * n + 2];
    const int nb = pr->L.n_bands;
    if (out->band_power_dbm) std::memcpy(out->band_power_dbm, rep + 4 * n + 3, nb * 8);
    if (out->band_capacity) std::memcpy(out->band_capacity, rep + 4 * n + 3 + nb, nb * 8);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    out->elapsed_seconds = ms * 1e-3;
    float kms = 0.f;
    if (pr->P.n_probes > 0) cudaEventElapsedTime(&kms, c->ev0, c->evk0);
    out->ode_seconds = kms * 1e-3;
  }
  if (pr->P.n_probes > 0) {
    float kms = 0.f;
    cudaEventElapsedTime(&kms, c->evk0, c->evk1);
    c->last_kernel_ms = kms;
    c->last_points = static_cast<double>(ne[0]);
    c->last_active = static_cast<double>(ne[1]);
    c->last_inner_steps = static_cast<double>(ne[0]) * c->last_total_steps;
  }
  return UWB_OK;
}

int uwb_evaluate_link_resident_noise(uwb_ctx* c, const double* psd_dev, void* stream) {
  if (c && c->multi())
    return fail(UWB_CONFIG_ERROR, "the split noise/report stages belong to one device; a multi-GPU "
                                  "context gathers eta itself (uwb_evaluate_link_resident)");
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  cudaSetDevice(c->device);
  reset_xfer(c);
  return run_noise(c, psd_dev, stream ? static_cast<cudaStream_t>(stream) : c->stream);
}

int uwb_evaluate_link_resident_report(uwb_ctx* c, double* report_dev, void* stream) {
  if (c && c->multi())
    return fail(UWB_CONFIG_ERROR, "the split noise/report stages belong to one device; a multi-GPU "
                                  "context gathers eta itself (uwb_evaluate_link_resident)");
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  c->last_launches = 0;
  int rc = run_report(c, st);
  if (rc) return rc;
  if (report_dev) {
    const size_t cnt = 4 * static_cast<size_t>(c->prep->n) + 3 + 2 * c->prep->L.n_bands;
    xfer(c, report_dev, c->prep->L.out, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  return UWB_OK;
}

int uwb_report_len(uwb_ctx* c, int* len) {
  if (c && c->multi()) return uwb_report_len(c->subs[0], len);
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  if (len) *len = 4 * c->prep->n + 3 + 2 * c->prep->L.n_bands;
  return UWB_OK;
}

int uwb_link_eta_buffer(uwb_ctx* c, double** eta_dev, int* n_ch) {
  if (c && c->multi())
    return fail(UWB_CONFIG_ERROR, "the split noise/report stages belong to one device; a multi-GPU "
                                  "context gathers eta itself (uwb_evaluate_link_resident)");
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  if (eta_dev) *eta_dev = c->prep->F.eta;
  if (n_ch) *n_ch = c->prep->n;
  return UWB_OK;
}

int uwb_last_ode_stats(uwb_ctx* c, double* ode_ms, long long* rhs_evals) {
  if (c && c->multi()) return uwb_last_ode_stats(c->subs[0], ode_ms, rhs_evals);
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  uwb_ctx::Prepared* pr = c->prep;
  float ms = 0.f;
  if (cudaEventSynchronize(c->evk0) != cudaSuccess ||
      cudaEventElapsedTime(&ms, c->ev0, c->evk0) != cudaSuccess)
    ms = 0.f;
  long long n = 0;
  xfer_sync(c, &n, pr->d_rhs, sizeof n, cudaMemcpyDeviceToHost);
  if (ode_ms) *ode_ms = ms;
  if (rhs_evals) *rhs_evals = n;
  return UWB_OK;
}

int uwb_resident_status(uwb_ctx* c) {
  if (c && c->multi()) return multi_status(c);
  if (!c || !c->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  return check_status(c);
}

int uwb_power_evolution(uwb_ctx* c, const uwb_grid* grid, const uwb_fibre* fibre,
                        const uwb_link_cfg* link, int steps, const double* mid, double* log_rho,
                        double* rho_end) {
  if (!c) return fail(UWB_CONFIG_ERROR, "null context");
  if (c->multi()) return uwb_power_evolution(c->subs[0], grid, fibre, link, steps, mid, log_rho, rho_end);
  cudaSetDevice(c->device);
  release_link_state(c);  // shares buffers with the prepared evaluation
  reset_xfer(c);
  int rc = validate_grid_full(grid);  // raman_power.hpp:56
  if (rc) return rc;
  if (!fibre || !link || !fibre->alpha || !fibre->aeff)
    return fail(UWB_CONFIG_ERROR, "missing fibre arrays");
  if (steps < 1 || !mid) return fail(UWB_CONFIG_ERROR, "distance grid has no steps");
  const int n = grid->n_ch;
  cudaStream_t st = c->stream;
  const double* d_freq = up(c, c->freq, grid->freq, n);
  const double* d_psd = up(c, c->psd, grid->psd, n);
  const double* d_alpha = up(c, c->alpha, fibre->alpha, n);
  const double* d_aeff = up(c, c->aeff, fibre->aeff, n);
  const double* d_mid = up(c, c->mid, mid, steps);
  if (link->include_raman && (fibre->raman_n < 2 || !fibre->raman_x || !fibre->raman_y))
    return fail(UWB_CONFIG_ERROR, "raman gain: table needs at least two (x, y) rows");
  if (n > kMaxOdeChannels) return fail(UWB_CONFIG_ERROR, "uwb: at most 7168 channels");
  // ode_work: log2 [n*steps] | ln [n*steps] | rho_end [n] | status, rhs [2] | coef a|u|v [3n]
  const size_t ns = static_cast<size_t>(n) * steps;
  double* w = c->ode_work.get<double>(2 * ns + n + 2 + 3 * n);
  if (!w) return fail(UWB_CUDA_ERROR, "device allocation failed");
  OdeParams O{};
  O.n = n;
  O.raman = link->include_raman ? 1 : 0;
  O.alpha = d_alpha;
  if (O.raman && raman_segments(fibre->raman_x, fibre->raman_y, fibre->raman_n, grid->spacing, n, &O))
    return fail(UWB_CONFIG_ERROR, "raman gain table has too many linear pieces");
  double* d_l2 = w;
  double* d_ln = w + ns;
  double* d_re = w + 2 * ns;
  int* d_status = reinterpret_cast<int*>(d_re + n);
  long long* d_rhs = reinterpret_cast<long long*>(d_re + n + 1);
  O.coef_a = d_re + n + 2;
  O.coef_u = O.coef_a + n;
  O.coef_v = O.coef_u + n;
  O.steps = steps;
  O.col_stride = steps;
  O.lane_k = 0;
  O.mid = d_mid;
  O.length = fibre->length_m;
  O.rtol = link->rtol > 0 ? link->rtol : 1e-9;
  O.atol = link->atol > 0 ? link->atol : 1e-16;
  O.continuous = c->ode_continuous;
  O.log2rho = d_l2;
  O.log_rho = d_ln;
  O.rho_end = d_re;
  O.status = d_status;
  O.rhs_evals = d_rhs;
  O.gwork = c->ode_gwork.get<double2>(ode_gwork_double2(n));
  if (!O.gwork) return fail(UWB_CUDA_ERROR, "device allocation failed");
  cudaMemsetAsync(d_status, 0, sizeof(int), st);
  const int lo = launch_raman_ode(O, d_freq, d_psd, grid->bch, d_aeff, fibre->raman_aeff_ref, st);
  if (lo < 0) return fail(UWB_CUDA_ERROR, "raman ODE launch failed");
  c->last_launches = lo;
  if (log_rho) xfer(c, log_rho, d_ln, static_cast<size_t>(n) * steps * 8, cudaMemcpyDeviceToHost, st);
  if (rho_end) xfer(c, rho_end, d_re, n * 8, cudaMemcpyDeviceToHost, st);
  int status = 0;
  xfer(c, &status, d_status, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "power evolution");
  if (status == 1) return fail(UWB_SOLVER_ERROR, "power evolution: non-positive rho");
  if (status == 2) return fail(UWB_SOLVER_ERROR, "rk45: step budget exhausted");
  if (status) return fail(UWB_SOLVER_ERROR, "rk45: step size underflow");
  return UWB_OK;
}

}  // extern "C"
