// Multi-GPU contexts behind the C-ABI (uwb_ctx_create_multi).
//
// The reference's only parallelism is channel-level data parallelism:
// all_channels_nli deals the channels of interest to cfg.workers host threads
// in contiguous batches (gn_integral.hpp:348-359 -> parallel_for_batches,
// parallel.hpp:21-47), each channel writing its own output slot, and the
// result is bit-identical for any worker count (test_gn_integral.cpp:291-300).
// Here the workers are GPUs:
//
//  * a multi context owns one sub-context per device entry; subs[0] leads;
//  * single evaluations (uwb_all_channels_nli, uwb_evaluate_link,
//    uwb_evaluate_link_resident) split the channels into contiguous ranges,
//    balanced by the per-channel work the previous NLI measured (|K|^2
//    evaluations per channel: active points x the sinc/fast mix, counted on
//    the device); every device runs the (tiny, replicated) Raman ODE and the
//    NLI of its range; the eta slices are gathered on the lead with one
//    cudaMemcpyPeerAsync per device (NVLink / NVSwitch), and the lead
//    assembles the SNR report;
//  * batches (uwb_evaluate_link_many: the optimiser's value and forward-
//    difference calls, link_optimizer.hpp:294-309) deal WHOLE evaluations to
//    the devices, so no evaluation waits on another device.
//
// Each channel's reduction order does not depend on the split, so results
// are bit-identical to a single device for any device list (tested with
// several sub-contexts on one GPU).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/uwb_nli.h"
#include "nli_kernel.cuh"
#include "uwb_capi_internal.cuh"
#include "uwb_ctx.cuh"
#include "uwb_link.cuh"
#include "uwb_multi.cuh"

namespace uwb {

namespace {

// Run fn(d) for every sub-context on its own host thread; first error wins
// (parallel_for_batches rethrows the first worker exception, parallel.hpp:39-46).
template <class F>
int for_each_sub(const std::vector<uwb_ctx*>& subs, F&& fn) {
  const size_t n = subs.size();
  std::vector<int> rc(n, UWB_OK);
  std::vector<std::string> msg(n);
  std::vector<std::thread> th;
  th.reserve(n);
  for (size_t d = 0; d < n; ++d)
    th.emplace_back([&, d] {
      cudaSetDevice(subs[d]->device);
      rc[d] = fn(d);
      if (rc[d]) msg[d] = uwb_last_error();
    });
  for (auto& t : th) t.join();
  for (size_t d = 0; d < n; ++d)
    if (rc[d]) return fail(rc[d], msg[d]);
  return UWB_OK;
}

// Contiguous channel ranges [lo[d], lo[d+1]) over the channels that will be
// probed, balanced by `cost` (uniform when it does not match the grid).
void split_channels(const uwb_grid* g, bool include_dark, int n_dev, const std::vector<double>& cost,
                    std::vector<int>* lo, std::vector<std::vector<int>>* parts) {
  const int n = g->n_ch;
  std::vector<int> act;
  for (int ch = 0; ch < n; ++ch)
    if (!g->guard[ch] && (include_dark || g->psd[ch] > 0.0)) act.push_back(ch);
  const bool have_cost = static_cast<int>(cost.size()) == n;
  double total = 0.0;
  for (int ch : act) total += have_cost && cost[ch] > 0.0 ? cost[ch] : 1.0;
  lo->assign(n_dev + 1, n);
  (*lo)[0] = 0;
  parts->assign(n_dev, {});
  double cum = 0.0;
  int d = 0;
  for (int ch : act) {
    const double w = have_cost && cost[ch] > 0.0 ? cost[ch] : 1.0;
    // move on once this device holds its share (the midpoint rule keeps the
    // split stable under small cost changes)
    while (d + 1 < n_dev && cum + 0.5 * w > total * (d + 1) / n_dev) {
      ++d;
      (*lo)[d] = ch;
    }
    (*parts)[d].push_back(ch);
    cum += w;
  }
  for (int k = d + 1; k < n_dev; ++k) (*lo)[k] = n;  // devices left without channels
  (*lo)[n_dev] = n;
}

int set_subset(uwb_ctx* s, const std::vector<int>& part) {
  // an empty part must not mean "all channels": -1 selects none
  static const int none = -1;
  return part.empty() ? uwb_set_channel_subset(s, 1, &none)
                      : uwb_set_channel_subset(s, static_cast<int>(part.size()), part.data());
}

// Per-channel |K|^2 evaluations of a sub-context's last NLI (synchronises).
void add_channel_work(uwb_ctx* s, std::vector<double>* cost) {
  const int np = s->last_n_probes;
  if (np <= 0 || s->last_chan_probe0.empty() || !s->probe_work.ptr<unsigned long long>()) return;
  std::vector<unsigned long long> w(np);
  cudaSetDevice(s->device);
  if (cudaMemcpy(w.data(), s->probe_work.ptr<unsigned long long>(), np * sizeof(w[0]),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  const int n = static_cast<int>(s->last_chan_probe0.size());
  if (static_cast<int>(cost->size()) != n) cost->assign(n, 0.0);
  for (int ch = 0; ch < n; ++ch) {
    const int p0 = s->last_chan_probe0[ch];
    if (p0 < 0) continue;
    double sum = 0.0;
    for (int k = 0; k < s->last_probes_per_chan && p0 + k < np; ++k) sum += static_cast<double>(w[p0 + k]);
    (*cost)[ch] = sum;
  }
}

void refresh_cost(uwb_ctx* m) {
  std::vector<double> cost;
  for (uwb_ctx* s : m->subs) add_channel_work(s, &cost);
  if (!cost.empty()) m->chan_cost = cost;
}

}  // namespace

int multi_all_channels_nli(uwb_ctx* m, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                           const double beta[3], const double* gamma, const uwb_nli_cfg* cfg,
                           uwb_nli_result* out) {
  int rc = validate_grid(grid);
  if (rc) return rc;
  const int n = grid->n_ch;
  const int nd = static_cast<int>(m->subs.size());
  std::vector<std::vector<int>> parts;
  split_channels(grid, false, nd, m->chan_cost, &m->part_lo, &parts);
  // per-device results, merged by channel ownership
  std::vector<std::vector<double>> eta(nd, std::vector<double>(n)), psd(nd, std::vector<double>(n)),
      pw(nd, std::vector<double>(n)), quad(nd, std::vector<double>(4 * n));
  std::vector<std::vector<uint8_t>> sk(nd, std::vector<uint8_t>(n));
  std::vector<double> secs(nd, 0.0);
  rc = for_each_sub(m->subs, [&](size_t d) {
    uwb_ctx* s = m->subs[d];
    int r = set_subset(s, parts[d]);
    if (r) return r;
    uwb_nli_result o{eta[d].data(), psd[d].data(), pw[d].data(), quad[d].data(), sk[d].data(), 0.0};
    r = uwb_all_channels_nli(s, grid, n_spans, spans, beta, gamma, cfg, &o);
    secs[d] = o.elapsed_seconds;
    return r;
  });
  if (rc) return rc;
  if (out) {
    for (int d = 0; d < nd; ++d)
      for (int ch = m->part_lo[d]; ch < m->part_lo[d + 1]; ++ch) {
        if (out->eta) out->eta[ch] = eta[d][ch];
        if (out->nli_psd) out->nli_psd[ch] = psd[d][ch];
        if (out->nli_power) out->nli_power[ch] = pw[d][ch];
        if (out->quadrant) std::memcpy(out->quadrant + 4 * ch, quad[d].data() + 4 * ch, 32);
        if (out->skipped) out->skipped[ch] = sk[d][ch];
      }
    out->elapsed_seconds = *std::max_element(secs.begin(), secs.end());
  }
  refresh_cost(m);
  return UWB_OK;
}

int multi_prepare(uwb_ctx* m, const uwb_grid* grid, const uwb_fibre* fibre, const uwb_link_cfg* link,
                  const uwb_nli_cfg* cfg, bool with_batch) {
  int rc = validate_grid_full(grid);
  if (rc) return rc;
  std::vector<std::vector<int>> parts;
  split_channels(grid, true, static_cast<int>(m->subs.size()), m->chan_cost, &m->part_lo, &parts);
  rc = for_each_sub(m->subs, [&](size_t d) {
    int r = set_subset(m->subs[d], parts[d]);
    if (r) return r;
    return uwb_evaluate_link_prepare(m->subs[d], grid, fibre, link, cfg);
  });
  if (rc) return rc;
  if (!with_batch) {  // a one-shot evaluation: no batch may run on an older link
    for (uwb_ctx* b : m->bsubs) {
      cudaSetDevice(b->device);
      release_link_state(b);
    }
    return UWB_OK;
  }
  // whole-evaluation contexts for batches
  return for_each_sub(m->bsubs, [&](size_t d) {
    return uwb_evaluate_link_prepare(m->bsubs[d], grid, fibre, link, cfg);
  });
}

// Noise on every device, eta slices gathered on the lead, report on the lead.
// psd_dev: launch PSD on the lead device (null: the prepared one).
int multi_run(uwb_ctx* m, const double* psd_dev, cudaStream_t lead_st) {
  uwb_ctx* lead = m->subs[0];
  const int nd = static_cast<int>(m->subs.size());
  for (uwb_ctx* s : m->subs)
    if (!s->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  const int n = lead->prep->n;
  cudaSetDevice(lead->device);
  cudaEventRecord(m->ev_done, lead_st);  // the caller's PSD is ready on the lead
  for (int d = 1; d < nd; ++d) {
    uwb_ctx* s = m->subs[d];
    cudaSetDevice(s->device);
    reset_xfer(s);
    if (psd_dev) {
      cudaStreamWaitEvent(s->stream, m->ev_done, 0);
      cudaMemcpyPeerAsync(s->prep->d_psd, s->device, psd_dev, lead->device, n * sizeof(double),
                          s->stream);
    }
    int rc = run_noise(s, nullptr, s->stream);
    if (rc) return rc;
    cudaEventRecord(s->ev_done, s->stream);
  }
  cudaSetDevice(lead->device);
  int rc = run_noise(lead, psd_dev, lead_st);
  if (rc) return rc;
  int launches = lead->last_launches;
  double* eta = lead->prep->F.eta;
  for (int d = 1; d < nd; ++d) {
    uwb_ctx* s = m->subs[d];
    launches += s->last_launches;
    const int lo = m->part_lo[d], hi = m->part_lo[d + 1];
    cudaStreamWaitEvent(lead_st, s->ev_done, 0);
    if (hi > lo)
      cudaMemcpyPeerAsync(eta + lo, lead->device, s->prep->F.eta + lo, s->device,
                          (hi - lo) * sizeof(double), lead_st);
  }
  rc = run_report(lead, lead_st);
  lead->last_launches = launches + 2;
  if (rc) return rc;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? UWB_OK : cuda_fail(e, "multi-GPU evaluation");
}

int multi_status(uwb_ctx* m) {
  for (uwb_ctx* s : m->subs) {
    cudaSetDevice(s->device);
    const int rc = check_status(s);
    if (rc) return rc;
  }
  return UWB_OK;
}

int multi_evaluate_link(uwb_ctx* m, const uwb_grid* grid, const uwb_fibre* fibre,
                        const uwb_link_cfg* link, const uwb_nli_cfg* cfg, uwb_link_report* out) {
  int rc = multi_prepare(m, grid, fibre, link, cfg, false);
  if (rc) return rc;
  uwb_ctx* lead = m->subs[0];
  cudaSetDevice(lead->device);
  reset_xfer(lead);
  if ((rc = multi_run(m, nullptr, lead->stream))) return rc;
  uwb_ctx::Prepared* pr = lead->prep;
  const int n = pr->n;
  const int nb = pr->L.n_bands;
  std::vector<double> rep(4 * static_cast<size_t>(n) + 3 + 2 * nb);
  cudaStream_t st = lead->stream;
  xfer(lead, rep.data(), pr->L.out, rep.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (out && out->rho_end)
    xfer(lead, out->rho_end, pr->O.rho_end, n * sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "evaluate_link (multi-GPU)");
  if ((rc = multi_status(m))) return rc;
  if (out) {
    if (out->eta) std::memcpy(out->eta, rep.data(), n * sizeof(double));
    if (out->p_ase) std::memcpy(out->p_ase, rep.data() + n, n * sizeof(double));
    if (out->snr_db) std::memcpy(out->snr_db, rep.data() + 2 * n, n * sizeof(double));
    if (out->capacity) std::memcpy(out->capacity, rep.data() + 3 * n, n * sizeof(double));
    out->loss_value = rep[4 * n];
    out->total_capacity = rep[4 * n + 1];
    out->total_power_dbm = rep[4 * n + 2];
    if (out->band_power_dbm) std::memcpy(out->band_power_dbm, rep.data() + 4 * n + 3, nb * 8);
    if (out->band_capacity) std::memcpy(out->band_capacity, rep.data() + 4 * n + 3 + nb, nb * 8);
    // the lead's events bracket its ODE and the gather-gated report: the
    // device time of the whole split evaluation
    float ms = 0.f, oms = 0.f;
    cudaEventElapsedTime(&ms, lead->ev0, lead->ev1);
    if (pr->P.n_probes > 0) cudaEventElapsedTime(&oms, lead->ev0, lead->evk0);
    out->elapsed_seconds = ms * 1e-3;
    out->ode_seconds = oms * 1e-3;
  }
  refresh_cost(m);
  return UWB_OK;
}

int multi_resident(uwb_ctx* m, const double* psd_dev, double* report_dev, void* stream) {
  uwb_ctx* lead = m->subs[0];
  if (!lead->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  cudaSetDevice(lead->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : lead->stream;
  reset_xfer(lead);
  int rc = multi_run(m, psd_dev, st);
  if (rc) return rc;
  if (report_dev) {
    uwb_ctx::Prepared* pr = lead->prep;
    const size_t cnt = 4 * static_cast<size_t>(pr->n) + 3 + 2 * pr->L.n_bands;
    xfer(lead, report_dev, pr->L.out, cnt * sizeof(double), cudaMemcpyDeviceToDevice, st);
  }
  return UWB_OK;
}

int multi_many(uwb_ctx* m, int n_eval, const double* psd_host, double* loss_host,
               double* report_host) {
  const int nd = static_cast<int>(m->bsubs.size());
  for (uwb_ctx* s : m->bsubs)
    if (!s->prep) return fail(UWB_CONFIG_ERROR, "uwb_evaluate_link_prepare not called");
  if (n_eval < 0 || (n_eval > 0 && !psd_host)) return fail(UWB_CONFIG_ERROR, "bad batch");
  const int n = m->bsubs[0]->prep->n;
  int rl = 0;
  uwb_report_len(m->bsubs[0], &rl);
  const int per = (n_eval + nd - 1) / std::max(nd, 1);
  return for_each_sub(m->bsubs, [&](size_t d) {
    const int b = static_cast<int>(d) * per, e = std::min(n_eval, b + per);
    if (b >= e) return static_cast<int>(UWB_OK);
    return uwb_evaluate_link_many(m->bsubs[d], e - b, psd_host + static_cast<size_t>(b) * n,
                                  loss_host ? loss_host + b : nullptr,
                                  report_host ? report_host + static_cast<size_t>(b) * rl : nullptr);
  });
}

}  // namespace uwb

using namespace uwb;

extern "C" {

int uwb_ctx_create_multi(const int* devices, int n_devices, uwb_ctx** out) {
  if (!out) return fail(UWB_CONFIG_ERROR, "null output");
  *out = nullptr;
  if (n_devices < 1 || !devices) return fail(UWB_CONFIG_ERROR, "need at least one device");
  auto* m = new uwb_ctx();
  m->device = devices[0];
  for (int k = 0; k < n_devices; ++k) {
    uwb_ctx* s = nullptr, *b = nullptr;
    int rc = uwb_ctx_create(devices[k], &s);
    if (rc == UWB_OK) {
      m->subs.push_back(s);
      rc = uwb_ctx_create(devices[k], &b);
      if (rc == UWB_OK) m->bsubs.push_back(b);
    }
    if (rc != UWB_OK) {
      const std::string msg = uwb_last_error();
      uwb_ctx_destroy(m);
      return fail(rc, msg);
    }
    cudaSetDevice(devices[k]);
    cudaEventCreateWithFlags(&s->ev_done, cudaEventDisableTiming);
  }
  // NVLink / NVSwitch peer access lead <-> others (the eta gather, the PSD
  // broadcast); without it cudaMemcpyPeerAsync still works, staged
  for (int k = 1; k < n_devices; ++k) {
    if (devices[k] == devices[0]) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, devices[0], devices[k]);
    if (ok) {
      cudaSetDevice(devices[0]);
      cudaDeviceEnablePeerAccess(devices[k], 0);
      cudaSetDevice(devices[k]);
      cudaDeviceEnablePeerAccess(devices[0], 0);
    }
  }
  cudaGetLastError();  // "already enabled" is not an error here
  cudaSetDevice(devices[0]);
  cudaEventCreateWithFlags(&m->ev_done, cudaEventDisableTiming);
  m->sm_count = m->subs[0]->sm_count;
  m->cc_major = m->subs[0]->cc_major;
  m->cc_minor = m->subs[0]->cc_minor;
  *out = m;
  return UWB_OK;
}

int uwb_ctx_width(uwb_ctx* c, int* n) {
  if (!c || !n) return fail(UWB_CONFIG_ERROR, "null argument");
  *n = c->multi() ? static_cast<int>(c->subs.size()) : 1;
  return UWB_OK;
}

int uwb_last_channel_work(uwb_ctx* c, int n_ch, double* work) {
  if (!c || !work) return fail(UWB_CONFIG_ERROR, "null argument");
  std::vector<double> cost;
  if (c->multi()) {
    for (uwb_ctx* s : c->subs) add_channel_work(s, &cost);
  } else {
    add_channel_work(c, &cost);
  }
  for (int ch = 0; ch < n_ch; ++ch) work[ch] = ch < static_cast<int>(cost.size()) ? cost[ch] : 0.0;
  return UWB_OK;
}

int uwb_last_partition_stats(uwb_ctx* c, int n, double* nli_ms, double* ode_ms, int* first_ch) {
  if (!c) return fail(UWB_CONFIG_ERROR, "null context");
  const std::vector<uwb_ctx*> one{c};
  const std::vector<uwb_ctx*>& subs = c->multi() ? c->subs : one;
  for (int d = 0; d < n && d < static_cast<int>(subs.size()); ++d) {
    uwb_ctx* s = subs[d];
    cudaSetDevice(s->device);
    float k = 0.f, o = 0.f;
    if (s->nli_events_valid && cudaEventSynchronize(s->evk1) == cudaSuccess) {
      cudaEventElapsedTime(&k, s->evk0, s->evk1);
      cudaEventElapsedTime(&o, s->ev0, s->evk0);
    }
    if (nli_ms) nli_ms[d] = k;
    if (ode_ms) ode_ms[d] = o;
    if (first_ch) first_ch[d] = c->multi() && d < static_cast<int>(c->part_lo.size()) ? c->part_lo[d] : 0;
  }
  return UWB_OK;
}

}  // extern "C"
