// uwblink_b200/gn_integral.hpp — C++ drop-in for the reference's hot path.
//
// Header-only shim over the C-ABI in uwb_nli.h (libuwbnli.so).  A reference
// user includes this next to the reference headers and calls
// uwblink::b200::<fn> with exactly the reference's signatures and types:
//
//   uwblink::b200::nli_psd_at             <- uwblink::nli_psd_at             gn_integral.hpp:218-222
//   uwblink::b200::channel_nli            <- uwblink::channel_nli            gn_integral.hpp:316-320
//   uwblink::b200::all_channels_nli       <- uwblink::all_channels_nli       gn_integral.hpp:334-338
//   uwblink::b200::solve_power_evolution  <- uwblink::solve_power_evolution  raman_power.hpp:52-55
//   uwblink::b200::solve_link_noise       <- uwblink::solve_link_noise       link_optimizer.hpp:181-190
//   uwblink::b200::evaluate_link          <- uwblink::evaluate_link          link_optimizer.hpp:241-245
//   uwblink::b200::optimise_launch_powers <- uwblink::optimise_launch_powers link_optimizer.hpp:257-324
//       (the reference's own L-BFGS-B, minimize_bounded lbfgsb.hpp:78, drives
//        device-resident evaluations; each forward-difference gradient is ONE
//        batch per GPU, its n_vars evaluations dealt across all visible GPUs)
//
// Errors are rethrown as the reference's own uwblink::ConfigError /
// uwblink::SolverError (units.hpp:16-24), so CLI exit codes 2/3 are kept
// (tools/uwblink_main.cpp:286-296); a missing or unusable B200 throws
// uwblink::b200::DeviceError (there is no CPU fallback).  INTEGRATION.md shows
// the one-line switch that routes the reference's own entry points here.
//
// Requires: the reference include path (uwblink/...), this repo's include/,
// and linking libuwbnli.so.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "uwb_nli.h"
#include "uwblink/gn_integral.hpp"
#include "uwblink/link_optimizer.hpp"

namespace uwblink::b200 {

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == UWB_OK) return;
  const std::string msg = uwb_last_error();
  if (rc == UWB_CONFIG_ERROR) throw ConfigError(msg);
  if (rc == UWB_SOLVER_ERROR) throw SolverError(msg);
  throw DeviceError(msg);
}

// One device context (device buffers stay resident in HBM across calls).
// Contexts are not shared between threads: the reference is reentrant, so
// each calling thread gets its own Engine from engine().
class Engine {
 public:
  explicit Engine(int device = 0) { check(uwb_ctx_create(device, &ctx_)); }
  // Multi-GPU context over `devices` (uwb_ctx_create_multi): the channels of
  // interest are split over the GPUs, bit-identical to one GPU.
  explicit Engine(const std::vector<int>& devices) {
    check(uwb_ctx_create_multi(devices.data(), static_cast<int>(devices.size()), &ctx_));
  }
  ~Engine() { uwb_ctx_destroy(ctx_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  uwb_ctx* get() const { return ctx_; }

 private:
  uwb_ctx* ctx_ = nullptr;
};

// The GPUs the drop-in may use: UWB_DEVICES="0,2,..." or every visible one.
inline std::vector<int> visible_devices() {
  std::vector<int> d;
  if (const char* e = std::getenv("UWB_DEVICES")) {
    const std::string s(e);
    std::size_t p = 0;
    while (p < s.size()) {
      const std::size_t q = s.find(',', p);
      d.push_back(std::stoi(s.substr(p, q == std::string::npos ? std::string::npos : q - p)));
      if (q == std::string::npos) break;
      p = q + 1;
    }
    if (!d.empty()) return d;
  }
  int n = 0;
  check(uwb_device_count(&n));
  for (int k = 0; k < n; ++k) d.push_back(k);
  return d;
}

// The engine for the reference's worker count (GnSolverConfig::workers,
// gn_integral.hpp:22): the workers of parallel_for_batches (parallel.hpp:
// 12-16, 0 = every hardware thread) are GPUs here -- 0 = every GPU of
// visible_devices(), k = the first min(k, n) of them.  One context per
// calling thread (the reference is reentrant) and per width.
inline Engine& engine(int workers = 1) {
  thread_local std::vector<std::unique_ptr<Engine>> cache;
  const std::vector<int> all = visible_devices();
  int w = workers <= 0 ? static_cast<int>(all.size()) : std::min<int>(workers, static_cast<int>(all.size()));
  w = std::max(1, w);
  if (cache.size() < static_cast<std::size_t>(w) + 1) cache.resize(w + 1);
  if (!cache[w]) {
    if (w == 1) cache[w] = std::make_unique<Engine>(all.empty() ? 0 : all[0]);
    else cache[w] = std::make_unique<Engine>(std::vector<int>(all.begin(), all.begin() + w));
  }
  return *cache[w];
}

namespace detail {

inline uwb_grid grid_view(const ChannelGrid& g) {
  uwb_grid v{};
  v.n_ch = static_cast<int>(g.size());
  v.freq = g.freq.data();
  v.psd = g.psd.data();
  v.guard = g.guard.data();
  v.spacing = g.spacing;
  v.bch = g.bch;
  v.centre = g.centre;
  v.half_band = g.half_band;
  return v;
}

inline std::vector<uwb_span> span_views(const std::vector<PowerEvolution>& spans) {
  std::vector<uwb_span> v(spans.size());
  for (std::size_t k = 0; k < spans.size(); ++k) {
    const PowerEvolution& e = spans[k];
    v[k].steps = static_cast<int>(e.steps());
    v[k].log_rho = e.log_rho.data();
    v[k].edge = e.grid.edge.data();
    v[k].mid = e.grid.mid.data();
    v[k].width = e.grid.width.data();
    v[k].length = e.grid.length;
  }
  return v;
}

inline uwb_nli_cfg cfg_view(const GnSolverConfig& c) {
  uwb_nli_cfg v{};
  v.n_r = c.n_r;
  v.u1_uniform = c.u1_sampling == GnSolverConfig::U1Sampling::kUniform ? 1 : 0;
  v.u1_min_ratio = c.u1_min_ratio;
  v.simpson = c.simpson_channel_average ? 1 : 0;
  v.mirror_q4 = c.mirror_q4 ? 1 : 0;
  return v;
}

inline void validate_spans(const ChannelGrid& grid, const std::vector<PowerEvolution>& spans,
                           const char* who) {
  if (spans.empty()) throw ConfigError(std::string(who) + ": need at least one span");
  for (const PowerEvolution& e : spans)
    if (e.channels() != grid.size())
      throw ConfigError(std::string(who) + ": span evolution does not match the channel grid");
}

// Per-channel fibre samples with the reference's own fibre model.
struct FibreSamples {
  std::vector<double> alpha, aeff, gamma;
  uwb_fibre f{};
};

inline FibreSamples fibre_samples(const FibreSpec& fibre, const ChannelGrid& grid) {
  FibreSamples s;
  const std::size_t n = grid.size();
  s.alpha.resize(n);
  s.aeff.resize(n);
  s.gamma.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    const double lam = freq_to_lambda(grid.freq[i]);
    s.alpha[i] = attenuation_at(fibre, lam);   // fibre_model.hpp:256
    s.aeff[i] = aeff_at(fibre, lam);           // :260
    s.gamma[i] = gamma_at(fibre, lam);         // :264
  }
  s.f.alpha = s.alpha.data();
  s.f.aeff = s.aeff.data();
  s.f.gamma = s.gamma.data();
  s.f.raman_n = static_cast<int>(fibre.raman.gain.x.size());
  s.f.raman_x = fibre.raman.gain.x.data();
  s.f.raman_y = fibre.raman.gain.y.data();
  s.f.raman_aeff_ref = fibre.raman.aeff_ref;
  const BetaCoefficients b = beta_from_dispersion(fibre.dispersion, freq_to_lambda(grid.centre));
  s.f.beta[0] = b.beta2;
  s.f.beta[1] = b.beta3;
  s.f.beta[2] = b.beta4;
  s.f.length_m = fibre.length_m;
  s.f.span_count = fibre.span_count;
  return s;
}

}  // namespace detail

// nli_psd_at (gn_integral.hpp:218-313).
[[nodiscard]] inline double nli_psd_at(const ChannelGrid& grid,
                                       const std::vector<PowerEvolution>& spans,
                                       const BetaCoefficients& betas, double gamma_probe,
                                       const GnSolverConfig& cfg, double nu_probe,
                                       std::array<double, 4>* quadrant_diag = nullptr) {
  detail::validate_spans(grid, spans, "nli_psd_at");
  const uwb_grid g = detail::grid_view(grid);
  const std::vector<uwb_span> sv = detail::span_views(spans);
  const uwb_nli_cfg c = detail::cfg_view(cfg);
  const double beta[3] = {betas.beta2, betas.beta3, betas.beta4};
  double out = 0.0;
  std::array<double, 4> q{};
  check(uwb_nli_psd_at(engine().get(), &g, static_cast<int>(sv.size()), sv.data(), beta, &c, 1,
                       &nu_probe, &gamma_probe, &out, q.data()));
  if (quadrant_diag) *quadrant_diag = q;
  return out;
}

// channel_nli (gn_integral.hpp:316-329): centre probe, Simpson when asked.
[[nodiscard]] inline double channel_nli(const ChannelGrid& grid,
                                        const std::vector<PowerEvolution>& spans,
                                        const BetaCoefficients& betas, double gamma_ch,
                                        const GnSolverConfig& cfg, std::size_t ch,
                                        std::array<double, 4>* quadrant_diag = nullptr) {
  detail::validate_spans(grid, spans, "nli_psd_at");
  const uwb_grid g = detail::grid_view(grid);
  const std::vector<uwb_span> sv = detail::span_views(spans);
  const uwb_nli_cfg c = detail::cfg_view(cfg);
  const double beta[3] = {betas.beta2, betas.beta3, betas.beta4};
  double out = 0.0;
  std::array<double, 4> q{};
  check(uwb_channel_nli(engine().get(), &g, static_cast<int>(sv.size()), sv.data(), beta,
                        gamma_ch, &c, static_cast<int>(ch), &out, q.data()));
  if (quadrant_diag) *quadrant_diag = q;
  return out;
}

// all_channels_nli (gn_integral.hpp:334-363).  cfg.workers picks the GPUs
// (engine(workers): 0 = all); results are identical for any value.
[[nodiscard]] inline NliResult all_channels_nli(const ChannelGrid& grid,
                                                const std::vector<PowerEvolution>& spans,
                                                const BetaCoefficients& betas,
                                                const FibreSpec& fibre,
                                                const GnSolverConfig& cfg) {
  detail::validate_spans(grid, spans, "nli_psd_at");
  const std::size_t n = grid.size();
  std::vector<double> gamma(n, 0.0);
  for (std::size_t ch = 0; ch < n; ++ch)
    if (!grid.guard[ch] && grid.psd[ch] > 0.0)
      gamma[ch] = gamma_at(fibre, freq_to_lambda(grid.freq[ch]));  // :353
  const uwb_grid g = detail::grid_view(grid);
  const std::vector<uwb_span> sv = detail::span_views(spans);
  const uwb_nli_cfg c = detail::cfg_view(cfg);
  const double beta[3] = {betas.beta2, betas.beta3, betas.beta4};
  NliResult r;
  r.eta.assign(n, 0.0);
  r.nli_psd.assign(n, 0.0);
  r.nli_power.assign(n, 0.0);
  r.quadrant.assign(n, {0.0, 0.0, 0.0, 0.0});
  r.skipped.assign(n, 0);
  std::vector<double> quad(4 * n, 0.0);
  uwb_nli_result o{};
  o.eta = r.eta.data();
  o.nli_psd = r.nli_psd.data();
  o.nli_power = r.nli_power.data();
  o.quadrant = quad.data();
  o.skipped = r.skipped.data();
  check(uwb_all_channels_nli(engine(cfg.workers).get(), &g, static_cast<int>(sv.size()), sv.data(),
                             beta, gamma.data(), &c, &o));
  for (std::size_t ch = 0; ch < n; ++ch)
    for (int q = 0; q < 4; ++q) r.quadrant[ch][q] = quad[4 * ch + q];
  r.elapsed_seconds = o.elapsed_seconds;
  return r;
}

// solve_power_evolution (raman_power.hpp:52-122) on the device.
[[nodiscard]] inline PowerEvolution solve_power_evolution(const FibreSpec& fibre,
                                                          const ChannelGrid& grid,
                                                          const DistanceGrid& zgrid,
                                                          const RamanSolveOptions& opt = {}) {
  grid.validate();
  const std::size_t n = grid.size();
  const std::size_t nm = zgrid.steps();
  PowerEvolution evo;
  evo.grid = zgrid;
  evo.freq = grid.freq;
  evo.spacing = grid.spacing;
  evo.launch.resize(n);
  for (std::size_t i = 0; i < n; ++i) evo.launch[i] = grid.channel_power(i);
  evo.log_rho.assign(n * nm, 0.0);
  evo.rho_end.assign(n, 1.0);
  detail::FibreSamples fs = detail::fibre_samples(fibre, grid);
  const uwb_grid g = detail::grid_view(grid);
  uwb_link_cfg lk{};
  lk.include_raman = opt.include_raman ? 1 : 0;
  lk.rtol = opt.rtol;
  lk.atol = opt.atol;
  lk.density = zgrid.density;
  check(uwb_power_evolution(engine().get(), &g, &fs.f, &lk, static_cast<int>(nm),
                            zgrid.mid.data(), evo.log_rho.data(), evo.rho_end.data()));
  return evo;
}

// evaluate_link (link_optimizer.hpp:241-245) = solve_link_noise (:181-190) +
// assemble_link_report (:194-237), all on the device.
[[nodiscard]] inline LinkReport evaluate_link(const FibreSpec& fibre, const ChannelGrid& grid,
                                              const BandPlan& plan, const LinkConfig& cfg,
                                              const GnSolverConfig& gn) {
  grid.validate();
  const std::size_t n = grid.size();
  detail::FibreSamples fs = detail::fibre_samples(fibre, grid);
  std::vector<double> nf(n, 5.0);
  std::vector<int> band(n, -1);
  for (std::size_t i = 0; i < n; ++i) {
    band[i] = plan.band_of_lambda(freq_to_lambda(grid.freq[i]));
    if (band[i] >= 0) nf[i] = plan.bands[static_cast<std::size_t>(band[i])].nf_db;
  }
  uwb_link_cfg lk{};
  lk.include_raman = cfg.raman.include_raman ? 1 : 0;
  lk.rtol = cfg.raman.rtol;
  lk.atol = cfg.raman.atol;
  lk.density = gn.mean_step_density;
  lk.nf_db = nf.data();
  lk.band = band.data();
  lk.n_bands = static_cast<int>(plan.bands.size());
  lk.use_snr_trx = cfg.use_snr_trx ? 1 : 0;
  lk.snr_trx_db = cfg.snr_trx_db;
  const uwb_grid g = detail::grid_view(grid);
  const uwb_nli_cfg c = detail::cfg_view(gn);
  std::vector<double> eta(n), pase(n), snr(n), cap(n), rho_end(n);
  std::vector<double> bpow(plan.bands.size()), bcap(plan.bands.size());
  uwb_link_report o{};
  o.eta = eta.data();
  o.p_ase = pase.data();
  o.snr_db = snr.data();
  o.capacity = cap.data();
  o.rho_end = rho_end.data();
  o.band_power_dbm = bpow.data();
  o.band_capacity = bcap.data();
  check(uwb_evaluate_link(engine(gn.workers).get(), &g, &fs.f, &lk, &c, &o));
  LinkReport rep;
  rep.channels.resize(n);
  for (std::size_t i = 0; i < n; ++i) {
    ChannelReport& r = rep.channels[i];
    r.freq = grid.freq[i];
    r.guard = grid.guard[i] != 0;
    r.band = band[i];
    if (r.guard || grid.psd[i] <= 0.0) continue;
    r.launch_dbm = watt_to_dbm(grid.channel_power(i));
    r.eta = eta[i];
    r.p_ase = pase[i];
    r.snr_db = snr[i];
    r.capacity = cap[i];
  }
  rep.band_power_dbm = bpow;
  rep.band_capacity = bcap;
  rep.total_power_dbm = o.total_power_dbm;
  rep.total_capacity = o.total_capacity;
  rep.loss_value = o.loss_value;
  return rep;
}

// solve_link_noise (link_optimizer.hpp:181-190): eta + span-end rho.
[[nodiscard]] inline LinkNoise solve_link_noise(const FibreSpec& fibre, const ChannelGrid& grid,
                                                const LinkConfig& cfg, const GnSolverConfig& gn) {
  grid.validate();
  const std::size_t n = grid.size();
  detail::FibreSamples fs = detail::fibre_samples(fibre, grid);
  std::vector<double> nf(n, 5.0);
  uwb_link_cfg lk{};
  lk.include_raman = cfg.raman.include_raman ? 1 : 0;
  lk.rtol = cfg.raman.rtol;
  lk.atol = cfg.raman.atol;
  lk.density = gn.mean_step_density;
  lk.nf_db = nf.data();
  const uwb_grid g = detail::grid_view(grid);
  const uwb_nli_cfg c = detail::cfg_view(gn);
  LinkNoise out;
  out.eta.assign(n, 0.0);
  out.rho_end.assign(n, 1.0);
  uwb_link_report o{};
  o.eta = out.eta.data();
  o.rho_end = out.rho_end.data();
  check(uwb_evaluate_link(engine(gn.workers).get(), &g, &fs.f, &lk, &c, &o));
  return out;
}

namespace detail {

// Everything uwb_evaluate_link_prepare needs for (fibre, grid, plan, cfg, gn).
struct LinkSetup {
  FibreSamples fs;
  std::vector<double> nf;
  std::vector<int> band;
  uwb_link_cfg lk{};
  uwb_nli_cfg c{};
  LinkSetup(const FibreSpec& fibre, const ChannelGrid& grid, const BandPlan& plan,
            const LinkConfig& cfg, const GnSolverConfig& gn)
      : fs(fibre_samples(fibre, grid)), nf(grid.size(), 5.0), band(grid.size(), -1) {
    for (std::size_t i = 0; i < grid.size(); ++i) {
      band[i] = plan.band_of_lambda(freq_to_lambda(grid.freq[i]));
      if (band[i] >= 0) nf[i] = plan.bands[static_cast<std::size_t>(band[i])].nf_db;
    }
    lk.include_raman = cfg.raman.include_raman ? 1 : 0;
    lk.rtol = cfg.raman.rtol;
    lk.atol = cfg.raman.atol;
    lk.density = gn.mean_step_density;
    lk.nf_db = nf.data();
    lk.band = band.data();
    lk.n_bands = static_cast<int>(plan.bands.size());
    lk.use_snr_trx = cfg.use_snr_trx ? 1 : 0;
    lk.snr_trx_db = cfg.snr_trx_db;
    c = cfg_view(gn);
  }
};

}  // namespace detail

struct OptimiseOptions {
  int n_devices = 0;               // GPUs for the gradient batches; 0 = all visible
  long long* cost_evals = nullptr;  // out (optional): full SNR evaluations issued
};

// optimise_launch_powers (link_optimizer.hpp:257-324) with the reference's
// own profile helpers and L-BFGS-B; the cost calls run on the device.
[[nodiscard]] inline OptimiseOutcome optimise_launch_powers(const FibreSpec& fibre,
                                                            const ChannelGrid& grid0,
                                                            const BandPlan& plan,
                                                            const LinkConfig& cfg,
                                                            double initial_dbm,
                                                            const OptimiseOptions& opt) {
  SegmentProfile prof = make_segment_profile(grid0, plan);
  prof.set_all(initial_dbm);
  const std::size_t n_vars = cfg.uniform_mode ? 1 : prof.variable_count();
  std::vector<double> x0(n_vars, initial_dbm);
  const std::vector<double> lo(n_vars, cfg.bound_lo_dbm);
  const std::vector<double> hi(n_vars, cfg.bound_hi_dbm);
  std::vector<GnSolverConfig> phases = cfg.phases;
  if (phases.empty()) phases.push_back(cfg.gn);

  int n_dev = opt.n_devices;
  if (n_dev <= 0) check(uwb_device_count(&n_dev));
  n_dev = std::max(1, n_dev);
  std::vector<std::unique_ptr<Engine>> eng;
  eng.reserve(static_cast<std::size_t>(n_dev));
  for (int d = 0; d < n_dev; ++d) eng.push_back(std::make_unique<Engine>(d));

  OptimiseOutcome out;
  auto to_profile = [&](const std::vector<double>& v) {
    if (cfg.uniform_mode) {
      prof.set_all(v[0]);
    } else {
      prof.unflatten(v);
    }
  };
  auto psd_of = [&](const std::vector<double>& v) {
    to_profile(v);
    ChannelGrid g = grid0;
    apply_profile(g, prof, plan);
    return g;
  };

  BoundedLbfgsResult best;
  for (const GnSolverConfig& phase_gn : phases) {
    ChannelGrid g0 = psd_of(x0);
    grid0.validate();
    const detail::LinkSetup setup(fibre, g0, plan, cfg, phase_gn);
    const uwb_grid gv = detail::grid_view(g0);
    for (auto& e : eng) check(uwb_evaluate_link_prepare(e->get(), &gv, &setup.fs.f, &setup.lk, &setup.c));
    std::optional<LinkNoise> frozen;
    if (cfg.freeze_eta) frozen = b200::solve_link_noise(fibre, g0, cfg, phase_gn);
    const std::size_t n = grid0.size();
    // losses of a batch of launch-power vectors, dealt over the GPUs
    auto losses = [&](const std::vector<std::vector<double>>& vs) {
      std::vector<double> f(vs.size(), 0.0);
      if (opt.cost_evals) *opt.cost_evals += static_cast<long long>(vs.size());
      if (frozen) {
        for (std::size_t k = 0; k < vs.size(); ++k)
          f[k] = assemble_link_report(fibre, psd_of(vs[k]), plan, cfg, *frozen).loss_value;
        return f;
      }
      std::vector<double> psd(vs.size() * n);
      for (std::size_t k = 0; k < vs.size(); ++k) {
        const ChannelGrid g = psd_of(vs[k]);
        std::copy(g.psd.begin(), g.psd.end(), psd.begin() + k * n);
      }
      const std::size_t per = (vs.size() + eng.size() - 1) / eng.size();
      std::vector<int> rc(eng.size(), UWB_OK);
      std::vector<std::string> msg(eng.size());
      std::vector<std::thread> th;
      for (std::size_t d = 0; d < eng.size(); ++d) {
        const std::size_t b = d * per, e = std::min(vs.size(), b + per);
        if (b >= e) break;
        th.emplace_back([&, d, b, e] {
          rc[d] = uwb_evaluate_link_many(eng[d]->get(), static_cast<int>(e - b), psd.data() + b * n,
                                         f.data() + b, nullptr);
          if (rc[d]) msg[d] = uwb_last_error();
        });
      }
      for (auto& t : th) t.join();
      for (std::size_t d = 0; d < eng.size(); ++d) {
        if (rc[d] == UWB_CONFIG_ERROR) throw ConfigError(msg[d]);
        if (rc[d] == UWB_SOLVER_ERROR) throw SolverError(msg[d]);
        if (rc[d]) throw DeviceError(msg[d]);
      }
      return f;
    };
    auto value = [&](const std::vector<double>& v) { return losses({v})[0]; };
    auto gradient = [&](const std::vector<double>& v, double f0) {
      std::vector<std::vector<double>> vs(v.size(), v);
      for (std::size_t i = 0; i < v.size(); ++i) vs[i][i] += cfg.fd_step_db;
      const std::vector<double> f = losses(vs);
      std::vector<double> g(v.size());
      for (std::size_t i = 0; i < v.size(); ++i) g[i] = (f[i] - f0) / cfg.fd_step_db;
      return g;
    };
    best = minimize_bounded(value, gradient, x0, lo, hi, cfg.lbfgs);
    out.phase_objectives.push_back(best.f);
    x0 = best.x;
  }
  to_profile(best.x);
  out.profile = prof;
  out.solver = best;
  ChannelGrid g = grid0;
  apply_profile(g, prof, plan);
  out.report = b200::evaluate_link(fibre, g, plan, cfg, phases.back());
  return out;
}

[[nodiscard]] inline OptimiseOutcome optimise_launch_powers(const FibreSpec& fibre,
                                                            const ChannelGrid& grid0,
                                                            const BandPlan& plan,
                                                            const LinkConfig& cfg,
                                                            double initial_dbm = 0.0) {
  return optimise_launch_powers(fibre, grid0, plan, cfg, initial_dbm, OptimiseOptions{});
}

}  // namespace uwblink::b200
