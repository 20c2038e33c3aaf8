// Drop-in proof for the C++ shim include/uwblink_b200/gn_integral.hpp.
//
// Compiled against the UNMODIFIED reference headers (/root/reference/proj/
// include, tests/support) by oracle/Makefile target `shim` into
// oracle/_ref/shim_parity (test infrastructure; run on the GPU box by
// tests/test_cxx_shim.py).  Each check restates a reference Catch2 assertion
// (file:line cited) with uwblink::b200::* in place of uwblink::*, and
// additionally compares the B200 result with the reference's own CPU result
// on the same inputs.  Prints one PASS/FAIL line per check; exit code = number
// of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "support/test_helpers.hpp"
#include "uwblink_b200/gn_closed_form.hpp"
#include "uwblink_b200/gn_integral.hpp"

using namespace uwblink;
namespace b2 = uwblink::b200;

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, const std::string& detail) {
  std::printf("%s %s %s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  if (!ok) ++g_fail;
}

void run(const std::string& name, const std::function<std::string()>& fn) {
  try {
    const std::string d = fn();
    report(name, d.rfind("FAIL:", 0) != 0, d);
  } catch (const std::exception& e) {
    report(name, false, std::string("exception: ") + e.what());
  }
}

double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double den = b[i] == 0.0 ? 1.0 : std::abs(b[i]);
    m = std::max(m, std::abs(a[i] - b[i]) / den);
  }
  return m;
}

std::string verdict(bool ok, const char* fmt, double v) {
  char buf[160];
  std::snprintf(buf, sizeof buf, fmt, v);
  return ok ? std::string(buf) : std::string("FAIL: ") + buf;
}

// test_gn_integral.cpp:16-29
struct ToyCase {
  FibreSpec fibre = uwtest::flat_fibre(0.2, 80e3);
  ChannelGrid grid = uwtest::toy_grid(3);
  BetaCoefficients betas{-21e-27, 0.0, 0.0};
  double gamma = 1.3e-3;
  std::vector<PowerEvolution> spans;
  explicit ToyCase(double density = 0.95) {
    RamanSolveOptions opt;
    opt.include_raman = false;
    spans.push_back(
        solve_power_evolution(fibre, grid, build_distance_grid(fibre.length_m, density), opt));
  }
};

// BASELINE config 1/2: 11 x 96 GBd at lambda_c, default fibre, Raman on.
struct Band11 {
  FibreSpec fibre = default_fibre();
  ChannelGrid grid;
  std::vector<PowerEvolution> spans;
  BetaCoefficients betas;
  Band11(double lambda_nm, double dbm) {
    grid = make_uniform_grid(11, 100e9, 96e9, kSpeedOfLight / (lambda_nm * 1e-9));
    set_uniform_launch(grid, dbm_to_watt(dbm));
    spans.push_back(solve_power_evolution(fibre, grid, build_distance_grid(fibre.length_m, 1.4)));
    betas = beta_from_dispersion(fibre.dispersion, freq_to_lambda(grid.centre));
  }
};

}  // namespace

// test_closed_form.cpp:104-121
struct CBandComb {
  FibreSpec fibre = default_fibre();
  ChannelGrid grid;
  BetaCoefficients betas;
  std::vector<PowerEvolution> spans;
  explicit CBandComb(std::size_t n_channels, double centre_lambda = 1550e-9,
                     double power_dbm = 0.0, bool raman = false) {
    grid = make_uniform_grid(n_channels, 100e9, 96e9, lambda_to_freq(centre_lambda));
    set_uniform_launch(grid, dbm_to_watt(power_dbm));
    betas = beta_from_dispersion(fibre.dispersion, centre_lambda);
    RamanSolveOptions opt;
    opt.include_raman = raman;
    spans.push_back(
        solve_power_evolution(fibre, grid, build_distance_grid(fibre.length_m, 1.4), opt));
  }
};

void closed_form_checks() {
  run("cfm_tracks_integral_away_from_zdw", [] {  // test_closed_form.cpp:125-136
    CBandComb comb(9);
    GnSolverConfig gn;
    gn.n_r = 200;
    const NliResult full = b2::all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre, gn);
    const NliResult cfm = b2::cfm_all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre);
    const NliResult ref = cfm_all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre);
    bool ok = true;
    for (std::size_t ch = 0; ch < comb.grid.size(); ++ch)
      ok = ok && cfm.eta[ch] > 0.0 && std::abs(uwtest::to_db(cfm.eta[ch] / full.eta[ch])) < 1.0;
    const double rel = max_rel(cfm.eta, ref.eta);
    return verdict(ok && rel < 1e-9, "rel vs reference %.3e", rel);
  });
  run("cfm_edge_handling", [] {  // :158-180
    CBandComb comb(5);
    ChannelGrid gg = comb.grid;
    gg.guard[2] = 1;
    gg.psd[2] = 0.0;
    const NliResult r = b2::cfm_all_channels_nli(gg, comb.spans, comb.betas, comb.fibre);
    bool ok = r.skipped[2] == 1 && r.eta[2] == 0.0 && r.eta[1] > 0.0;
    int thrown = 0;
    try {
      (void)b2::cfm_all_channels_nli(comb.grid, {}, comb.betas, comb.fibre);
    } catch (const ConfigError&) {
      ++thrown;
    }
    CBandComb other(7);
    try {
      (void)b2::cfm_all_channels_nli(comb.grid, other.spans, comb.betas, comb.fibre);
    } catch (const ConfigError&) {
      ++thrown;
    }
    ok = ok && thrown == 2;
    return verdict(ok, "%g", ok ? 1.0 : 0.0);
  });
  run("cfm_undershoots_near_zdw", [] {  // :182-207
    CBandComb comb(5, 1302.3e-9, 2.0, true);
    GnSolverConfig gn;
    gn.n_r = 150;
    const NliResult full = b2::all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre, gn);
    const NliResult cfm = b2::cfm_all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre);
    const NliResult ref = cfm_all_channels_nli(comb.grid, comb.spans, comb.betas, comb.fibre);
    std::size_t worst = 0;
    double gap_w = 0.0;
    for (std::size_t ch = 0; ch < comb.grid.size(); ++ch) {
      const double gap = std::abs(uwtest::to_db(cfm.eta[ch] / full.eta[ch]));
      if (gap > gap_w) {
        gap_w = gap;
        worst = ch;
      }
    }
    const double rel = max_rel(cfm.eta, ref.eta);
    return verdict(cfm.eta[worst] < full.eta[worst] && rel < 1e-9, "rel vs reference %.3e", rel);
  });
}

int main() {
  closed_form_checks();
  // --- hyperbolic vs Cartesian, test_gn_integral.cpp:226-235 (+ B200 == CPU)
  run("toy3_nli_psd_at_vs_reference_and_cartesian", [] {
    ToyCase toy;
    GnSolverConfig cfg;
    cfg.n_r = 150;
    const double nu = toy.grid.centre;
    const double hyp = b2::nli_psd_at(toy.grid, toy.spans, toy.betas, toy.gamma, cfg, nu);
    const double ref = nli_psd_at(toy.grid, toy.spans, toy.betas, toy.gamma, cfg, nu);
    const double cart =
        uwtest::cartesian_nli_psd(toy.grid, toy.spans, toy.betas, toy.gamma, nu, 600);
    const double rel = std::abs(hyp / ref - 1.0);
    const bool ok = rel < 1e-9 && std::abs(uwtest::to_db(hyp / cart)) < 0.1;
    return verdict(ok, "rel vs reference %.3e", rel);
  });

  // --- Q4 mirror == direct Q4, test_gn_integral.cpp:250-263
  run("toy3_mirror_q4", [] {
    ToyCase toy;
    GnSolverConfig mirrored, direct;
    mirrored.n_r = direct.n_r = 100;
    direct.mirror_q4 = false;
    const double nu = toy.grid.freq[0];
    std::array<double, 4> qa{}, qb{};
    const double a = b2::nli_psd_at(toy.grid, toy.spans, toy.betas, toy.gamma, mirrored, nu, &qa);
    const double b = b2::nli_psd_at(toy.grid, toy.spans, toy.betas, toy.gamma, direct, nu, &qb);
    const double rel = std::abs(a / b - 1.0);
    return verdict(rel < 1e-12 && std::abs(qb[1] / qb[3] - 1.0) < 1e-12, "rel %.3e", rel);
  });

  // --- whole-grid sweep, test_gn_integral.cpp:265-346
  const FibreSpec fibre = uwtest::flat_fibre(0.2, 80e3);
  ChannelGrid grid = uwtest::toy_grid(5);
  const BetaCoefficients betas{-21e-27, 0.0, 0.0};
  RamanSolveOptions opt;
  opt.include_raman = false;
  std::vector<PowerEvolution> spans{
      solve_power_evolution(fibre, grid, build_distance_grid(fibre.length_m, 0.95), opt)};
  GnSolverConfig cfg;
  cfg.n_r = 64;
  cfg.workers = 1;

  run("toy5_sweep_vs_reference", [&] {
    const NliResult g = b2::all_channels_nli(grid, spans, betas, fibre, cfg);
    const NliResult r = all_channels_nli(grid, spans, betas, fibre, cfg);
    const double rel = max_rel(g.eta, r.eta);
    return verdict(rel < 1e-9 && g.skipped == r.skipped, "max rel eta %.3e", rel);
  });

  run("toy5_cubic_scaling", [&] {  // :277-289
    const NliResult base = b2::all_channels_nli(grid, spans, betas, fibre, cfg);
    ChannelGrid louder = grid;
    set_uniform_launch(louder, 2e-3);
    std::vector<PowerEvolution> spans2{
        b2::solve_power_evolution(fibre, louder, build_distance_grid(fibre.length_m, 0.95), opt)};
    const NliResult loud = b2::all_channels_nli(louder, spans2, betas, fibre, cfg);
    double worst = 0.0;
    bool pos = true;
    for (std::size_t ch = 0; ch < grid.size(); ++ch) {
      pos = pos && base.eta[ch] > 0.0;
      worst = std::max(worst, std::abs(loud.nli_power[ch] / (8.0 * base.nli_power[ch]) - 1.0));
      worst = std::max(worst, std::abs(loud.eta[ch] / base.eta[ch] - 1.0));
    }
    return verdict(pos && worst < 1e-9, "worst %.3e", worst);
  });

  run("toy5_workers_bit_identical", [&] {  // :291-300
    const NliResult one = b2::all_channels_nli(grid, spans, betas, fibre, cfg);
    GnSolverConfig four = cfg;
    four.workers = 4;
    const NliResult par = b2::all_channels_nli(grid, spans, betas, fibre, four);
    return verdict(one.eta == par.eta && one.nli_psd == par.nli_psd, "identical=%g",
                   one.eta == par.eta ? 1.0 : 0.0);
  });

  run("toy5_guard_skipped", [&] {  // :302-311
    ChannelGrid gg = grid;
    gg.guard[2] = 1;
    gg.psd[2] = 0.0;
    const NliResult r = b2::all_channels_nli(gg, spans, betas, fibre, cfg);
    const bool ok = r.skipped[2] == 1 && r.eta[2] == 0.0 && r.eta[1] > 0.0 && r.eta[3] > 0.0;
    return verdict(ok, "eta[2]=%g", r.eta[2]);
  });

  run("toy5_dark_grid", [&] {  // :313-324
    ChannelGrid dark = grid;
    for (std::size_t i = 0; i < dark.size(); ++i) {
      dark.psd[i] = 0.0;
      dark.guard[i] = 1;
    }
    const NliResult r = b2::all_channels_nli(dark, spans, betas, fibre, cfg);
    bool ok = true;
    for (std::size_t i = 0; i < dark.size(); ++i) ok = ok && r.skipped[i] == 1 && r.eta[i] == 0.0;
    return verdict(ok, "%g", ok ? 1.0 : 0.0);
  });

  run("toy5_simpson", [&] {  // :326-337
    GnSolverConfig simpson = cfg;
    simpson.simpson_channel_average = true;
    const NliResult c = b2::all_channels_nli(grid, spans, betas, fibre, cfg);
    const NliResult a = b2::all_channels_nli(grid, spans, betas, fibre, simpson);
    const NliResult ra = all_channels_nli(grid, spans, betas, fibre, simpson);
    double worst = 0.0;
    for (std::size_t ch = 0; ch < grid.size(); ++ch)
      worst = std::max(worst, std::abs(uwtest::to_db(a.eta[ch] / c.eta[ch])));
    const double rel = max_rel(a.eta, ra.eta);
    return verdict(worst < 0.6 && rel < 1e-9, "rel vs reference %.3e", rel);
  });

  run("config_errors", [&] {  // :339-346
    int thrown = 0;
    GnSolverConfig bad = cfg;
    bad.n_r = 1;
    try {
      (void)b2::nli_psd_at(grid, spans, betas, 1e-3, bad, grid.centre);
    } catch (const ConfigError&) {
      ++thrown;
    }
    try {
      (void)b2::nli_psd_at(grid, {}, betas, 1e-3, cfg, grid.centre);
    } catch (const ConfigError&) {
      ++thrown;
    }
    ChannelGrid other = uwtest::toy_grid(4);
    try {
      (void)b2::nli_psd_at(other, spans, betas, 1e-3, cfg, other.centre);
    } catch (const ConfigError&) {
      ++thrown;
    }
    return verdict(thrown == 3, "ConfigError thrown %g/3", thrown);
  });

  // --- BASELINE configs 1 and 2 (default fibre, Raman on), vs the reference
  run("cband11_all_channels_nli", [] {
    Band11 c(1550.0, 0.0);
    GnSolverConfig gc;
    const NliResult g = b2::all_channels_nli(c.grid, c.spans, c.betas, c.fibre, gc);
    const NliResult r = all_channels_nli(c.grid, c.spans, c.betas, c.fibre, gc);
    const double rel = max_rel(g.eta, r.eta);
    return verdict(rel < 1e-9, "max rel eta %.3e", rel);
  });

  run("oband11_simpson_all_channels_nli", [] {
    Band11 c(1302.3, 2.0);
    GnSolverConfig gc;
    gc.simpson_channel_average = true;
    const NliResult g = b2::all_channels_nli(c.grid, c.spans, c.betas, c.fibre, gc);
    const NliResult r = all_channels_nli(c.grid, c.spans, c.betas, c.fibre, gc);
    const double rel = max_rel(g.eta, r.eta);
    return verdict(rel < 1e-9, "max rel eta %.3e", rel);
  });

  run("cband11_power_evolution", [] {
    Band11 c(1550.0, 0.0);
    const DistanceGrid z = build_distance_grid(c.fibre.length_m, 1.4);
    const PowerEvolution g = b2::solve_power_evolution(c.fibre, c.grid, z);
    const PowerEvolution& r = c.spans[0];
    double worst = 0.0;
    for (std::size_t i = 0; i < r.log_rho.size(); ++i)
      worst = std::max(worst, std::abs(g.log_rho[i] - r.log_rho[i]));
    return verdict(worst < 1e-9 && max_rel(g.rho_end, r.rho_end) < 1e-9, "max |dlog rho| %.3e",
                   worst);
  });

  // --- full SNR evaluation of the 589-channel plan (BASELINE config 3, paper-speed setting)
  run("uwb589_evaluate_link", [] {
    const BandPlan plan = default_band_plan();
    ChannelGrid g = make_default_uwb_grid(plan);
    set_uniform_launch(g, 1e-3);
    const FibreSpec f = default_fibre();
    LinkConfig lc;
    GnSolverConfig gn;
    gn.n_r = 75;
    gn.mean_step_density = 0.95;
    const LinkReport b = b2::evaluate_link(f, g, plan, lc, gn);
    const LinkReport r = evaluate_link(f, g, plan, lc, gn);
    double deta = 0.0, dsnr = 0.0;
    for (std::size_t i = 0; i < g.size(); ++i) {
      if (r.channels[i].eta <= 0.0) continue;
      deta = std::max(deta, std::abs(b.channels[i].eta / r.channels[i].eta - 1.0));
      dsnr = std::max(dsnr, std::abs(b.channels[i].snr_db - r.channels[i].snr_db));
    }
    const bool ok = deta < 1e-6 && dsnr < 0.01 &&
                    std::abs(b.loss_value / r.loss_value - 1.0) < 1e-9;
    char buf[160];
    std::snprintf(buf, sizeof buf, "max rel eta %.3e, max dSNR %.3e dB", deta, dsnr);
    return ok ? std::string(buf) : "FAIL: " + std::string(buf);
  });

  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
