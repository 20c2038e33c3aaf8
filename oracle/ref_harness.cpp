// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// C-ABI harness over the UNMODIFIED reference headers (uwblink, header-only
// C++20, /root/reference/proj/include).  Built by oracle/Makefile into
// oracle/_ref/libuwbref.so (git-ignored; travels to the GPU box prebuilt).
// Used only by tests/ (golden generation, oracle pinning), bench.py's
// cpu_baseline leg and `bench.py --impl reference`.  Nothing here is copied from
// the reference: every function below just fills the reference's own structs
// and calls the reference's own entry points:
//   build_distance_grid       distance_grid.hpp:23
//   default_fibre             fibre_model.hpp:287
//   make_uniform_grid         channel_grid.hpp:64
//   make_default_uwb_grid     channel_grid.hpp:133
//   solve_power_evolution     raman_power.hpp:52
//   beta_from_dispersion      fibre_model.hpp:76
//   gamma_at                  fibre_model.hpp:264
//   all_channels_nli          gn_integral.hpp:334
//   nli_psd_at                gn_integral.hpp:218
//   assemble_link_report      link_optimizer.hpp:194
//   optimise_launch_powers    link_optimizer.hpp:257
//   cartesian_nli_psd         tests/support/test_helpers.hpp:43
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "support/test_helpers.hpp"
#include "uwblink/gn_closed_form.hpp"
#include "uwblink/gn_integral.hpp"
#include "uwblink/link_optimizer.hpp"

using namespace uwblink;

extern "C" {

// Flat description of one reference case.  Mirrors uwtest::flat_fibre /
// toy_grid / make_default_uwb_grid choices used by the reference tests.
typedef struct RefCase {
  int fibre_kind;           // 0 = default_fibre(), 1 = flat_fibre(flat_alpha_db_km)
  double flat_alpha_db_km;
  double length_m;
  int span_count;
  int raman;                // RamanSolveOptions::include_raman
  int uwb_default;          // 1 = make_default_uwb_grid(default_band_plan()) (ignores n_ch..centre)
  int n_ch;
  double spacing, bch, centre;
  const double* launch_w;   // per-channel launch power (W) or NULL => uniform_w on every slot
  double uniform_w;
  const uint8_t* guard;     // optional guard override (NULL => grid's own)
  int n_r;
  double density;
  int workers;
  int u1_uniform;
  double u1_min_ratio;
  int simpson;
  int mirror_q4;
  int betas_explicit;       // 0 => beta_from_dispersion(fibre.dispersion, lambda(centre))
  double beta2, beta3, beta4;
} RefCase;

}  // extern "C"

namespace {

thread_local std::string g_err;

FibreSpec make_fibre(const RefCase& c) {
  FibreSpec f = c.fibre_kind == 1 ? uwtest::flat_fibre(c.flat_alpha_db_km, c.length_m, c.span_count)
                                  : default_fibre();
  f.length_m = c.length_m;
  f.span_count = c.span_count;
  return f;
}

ChannelGrid make_grid(const RefCase& c) {
  ChannelGrid g = c.uwb_default ? make_default_uwb_grid(default_band_plan())
                                : make_uniform_grid(static_cast<std::size_t>(c.n_ch), c.spacing,
                                                    c.bch, c.centre);
  if (c.guard) {
    for (std::size_t i = 0; i < g.size(); ++i) g.guard[i] = c.guard[i];
  }
  for (std::size_t i = 0; i < g.size(); ++i) {
    g.set_channel_power(i, c.launch_w ? c.launch_w[i] : c.uniform_w);
  }
  return g;
}

GnSolverConfig make_cfg(const RefCase& c) {
  GnSolverConfig cfg;
  cfg.n_r = c.n_r;
  cfg.mean_step_density = c.density;
  cfg.workers = c.workers;
  cfg.u1_sampling = c.u1_uniform ? GnSolverConfig::U1Sampling::kUniform
                                 : GnSolverConfig::U1Sampling::kLog;
  cfg.u1_min_ratio = c.u1_min_ratio;
  cfg.simpson_channel_average = c.simpson != 0;
  cfg.mirror_q4 = c.mirror_q4 != 0;
  return cfg;
}

BetaCoefficients make_betas(const RefCase& c, const FibreSpec& f, const ChannelGrid& g) {
  if (c.betas_explicit) return BetaCoefficients{c.beta2, c.beta3, c.beta4};
  return beta_from_dispersion(f.dispersion, freq_to_lambda(g.centre));
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Channel grid arrays + scalars {spacing, bch, centre, half_band}.
int ref_grid(const RefCase* c, double* freq, double* psd, uint8_t* guard, double* scalars,
             int* n_out) {
  return guarded([&] {
    const ChannelGrid g = make_grid(*c);
    *n_out = static_cast<int>(g.size());
    if (freq) std::memcpy(freq, g.freq.data(), g.size() * sizeof(double));
    if (psd) std::memcpy(psd, g.psd.data(), g.size() * sizeof(double));
    if (guard) std::memcpy(guard, g.guard.data(), g.size());
    if (scalars) {
      scalars[0] = g.spacing;
      scalars[1] = g.bch;
      scalars[2] = g.centre;
      scalars[3] = g.half_band;
    }
  });
}

int ref_distance_grid(double length_m, double density, int cap, double* edge, double* mid,
                      double* width, int* steps_out) {
  return guarded([&] {
    const DistanceGrid g = build_distance_grid(length_m, density);
    *steps_out = static_cast<int>(g.steps());
    if (static_cast<int>(g.steps()) > cap) return;
    std::memcpy(edge, g.edge.data(), g.edge.size() * sizeof(double));
    std::memcpy(mid, g.mid.data(), g.mid.size() * sizeof(double));
    std::memcpy(width, g.width.data(), g.width.size() * sizeof(double));
  });
}

// log_rho [n_ch * steps] (reference layout ch*steps+m) and rho_end [n_ch].
int ref_power_evolution(const RefCase* c, int cap, double* log_rho, double* rho_end,
                        int* steps_out, double* seconds) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    RamanSolveOptions opt;
    opt.include_raman = c->raman != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const PowerEvolution evo = solve_power_evolution(f, g, zg, opt);
    if (seconds) *seconds = secs(t0);
    *steps_out = static_cast<int>(evo.steps());
    if (static_cast<int>(evo.log_rho.size()) > cap) return;
    std::memcpy(log_rho, evo.log_rho.data(), evo.log_rho.size() * sizeof(double));
    std::memcpy(rho_end, evo.rho_end.data(), evo.rho_end.size() * sizeof(double));
  });
}

// Per-channel fibre quantities used on the path: alpha [1/m], aeff [m^2],
// gamma [1/(W m)] at each grid frequency; betas at the grid centre.
int ref_fibre_at(const RefCase* c, int n, const double* freq, double* alpha, double* aeff,
                 double* gamma, double* betas3) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    for (int i = 0; i < n; ++i) {
      const double lam = freq_to_lambda(freq[i]);
      if (alpha) alpha[i] = attenuation_at(f, lam);
      if (aeff) aeff[i] = aeff_at(f, lam);
      if (gamma) gamma[i] = gamma_at(f, lam);
    }
    if (betas3) {
      const ChannelGrid g = make_grid(*c);
      const BetaCoefficients b = make_betas(*c, f, g);
      betas3[0] = b.beta2;
      betas3[1] = b.beta3;
      betas3[2] = b.beta4;
    }
  });
}

// Full reference sweep: power evolution (timed separately) + all_channels_nli.
int ref_all_channels_nli(const RefCase* c, double* eta, double* nli_psd, double* nli_power,
                         double* quad4, uint8_t* skipped, double* nli_seconds,
                         double* ode_seconds) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    RamanSolveOptions opt;
    opt.include_raman = c->raman != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const PowerEvolution evo = solve_power_evolution(f, g, zg, opt);
    if (ode_seconds) *ode_seconds = secs(t0);
    const std::vector<PowerEvolution> spans(static_cast<std::size_t>(f.span_count), evo);
    const NliResult r = all_channels_nli(g, spans, make_betas(*c, f, g), f, make_cfg(*c));
    const std::size_t n = g.size();
    if (eta) std::memcpy(eta, r.eta.data(), n * sizeof(double));
    if (nli_psd) std::memcpy(nli_psd, r.nli_psd.data(), n * sizeof(double));
    if (nli_power) std::memcpy(nli_power, r.nli_power.data(), n * sizeof(double));
    if (quad4) std::memcpy(quad4, r.quadrant.data(), n * 4 * sizeof(double));
    if (skipped) std::memcpy(skipped, r.skipped.data(), n);
    if (nli_seconds) *nli_seconds = r.elapsed_seconds;
  });
}

// Closed-form model: power evolution + cfm_all_channels_nli (gn_closed_form.hpp:70).
int ref_cfm_all_channels_nli(const RefCase* c, double* eta, double* nli_psd, double* nli_power,
                             uint8_t* skipped, double* seconds) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    RamanSolveOptions opt;
    opt.include_raman = c->raman != 0;
    const PowerEvolution evo = solve_power_evolution(f, g, zg, opt);
    const std::vector<PowerEvolution> spans(static_cast<std::size_t>(f.span_count), evo);
    const auto t0 = std::chrono::steady_clock::now();
    const NliResult r = cfm_all_channels_nli(g, spans, make_betas(*c, f, g), f);
    if (seconds) *seconds = secs(t0);
    const std::size_t n = g.size();
    if (eta) std::memcpy(eta, r.eta.data(), n * sizeof(double));
    if (nli_psd) std::memcpy(nli_psd, r.nli_psd.data(), n * sizeof(double));
    if (nli_power) std::memcpy(nli_power, r.nli_power.data(), n * sizeof(double));
    if (skipped) std::memcpy(skipped, r.skipped.data(), n);
  });
}

// Single probe (nli_psd_at) with an explicit gamma.
int ref_nli_psd_at(const RefCase* c, double gamma, double nu, double* quad4, double* out) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    RamanSolveOptions opt;
    opt.include_raman = c->raman != 0;
    const std::vector<PowerEvolution> spans(static_cast<std::size_t>(f.span_count),
                                            solve_power_evolution(f, g, zg, opt));
    std::array<double, 4> q{};
    *out = nli_psd_at(g, spans, make_betas(*c, f, g), gamma, make_cfg(*c), nu, &q);
    if (quad4) std::memcpy(quad4, q.data(), sizeof(q));
  });
}

// Brute-force Cartesian midpoint quadrature of the test suite (the
// reference's independent oracle for the hyperbolic transform).
int ref_cartesian_nli_psd(const RefCase* c, double gamma, double nu, int n_cells, double* out) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    RamanSolveOptions opt;
    opt.include_raman = c->raman != 0;
    const std::vector<PowerEvolution> spans(static_cast<std::size_t>(f.span_count),
                                            solve_power_evolution(f, g, zg, opt));
    *out = uwtest::cartesian_nli_psd(g, spans, make_betas(*c, f, g), gamma, nu, n_cells);
  });
}

double ref_phase_mismatch(double f1, double f2, double fi, double b2, double b3, double b4) {
  return phase_mismatch(f1, f2, fi, BetaCoefficients{b2, b3, b4});
}

int ref_quadrant_limits(int q, double half_band, double f, double* out5) {
  return guarded([&] {
    const QuadrantSpec s = quadrant_limits(q, half_band, f);
    out5[0] = s.b1;
    out5[1] = s.b2;
    out5[2] = s.s1;
    out5[3] = s.s2;
    out5[4] = s.u1_max;
  });
}

// Full SNR evaluation (evaluate_link, link_optimizer.hpp:241) on the
// default band plan: ODE + NLI + assemble_link_report.  Per-channel outputs
// plus {loss, total_capacity, total_power_dbm} and the three stage timings.
int ref_evaluate_link(const RefCase* c, double* eta, double* p_ase, double* snr_db,
                      double* capacity, double* totals3, double* t_ode_nli_asm) {
  return guarded([&] {
    const FibreSpec f = make_fibre(*c);
    const ChannelGrid g = make_grid(*c);
    const BandPlan plan = default_band_plan();
    LinkConfig lc;
    lc.gn = make_cfg(*c);
    lc.raman.include_raman = c->raman != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const DistanceGrid zg = build_distance_grid(f.length_m, c->density);
    PowerEvolution evo = solve_power_evolution(f, g, zg, lc.raman);
    const double t_ode = secs(t0);
    const auto t1 = std::chrono::steady_clock::now();
    std::vector<PowerEvolution> spans(static_cast<std::size_t>(f.span_count), evo);
    NliResult nli = all_channels_nli(
        g, spans, beta_from_dispersion(f.dispersion, freq_to_lambda(g.centre)), f, lc.gn);
    const double t_nli = secs(t1);
    const auto t2 = std::chrono::steady_clock::now();
    const LinkNoise noise{std::move(nli.eta), std::move(evo.rho_end)};
    const LinkReport rep = assemble_link_report(f, g, plan, lc, noise);
    const double t_asm = secs(t2);
    for (std::size_t i = 0; i < g.size(); ++i) {
      if (eta) eta[i] = rep.channels[i].eta;
      if (p_ase) p_ase[i] = rep.channels[i].p_ase;
      if (snr_db) snr_db[i] = rep.channels[i].snr_db;
      if (capacity) capacity[i] = rep.channels[i].capacity;
    }
    if (totals3) {
      totals3[0] = rep.loss_value;
      totals3[1] = rep.total_capacity;
      totals3[2] = rep.total_power_dbm;
    }
    if (t_ode_nli_asm) {
      t_ode_nli_asm[0] = t_ode;
      t_ode_nli_asm[1] = t_nli;
      t_ode_nli_asm[2] = t_asm;
    }
  });
}

}  // extern "C"
