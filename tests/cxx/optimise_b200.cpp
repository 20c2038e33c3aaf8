// BASELINE config 5 (launch-power optimisation loop) through the C++ drop-in:
// uwblink::b200::optimise_launch_powers = the reference's own segment profile
// + L-BFGS-B (link_optimizer.hpp:257-324, lbfgsb.hpp:78) with every cost call
// on the device, forward-difference gradients batched and dealt over the
// visible GPUs.  Compiled against the UNMODIFIED reference headers by
// oracle/Makefile target `shim` (test/measurement infrastructure).
//
//   optimise_b200 [--iters K] [--n-r N] [--density D] [--devices G]
//                 [--reference-iters K2]      (also run the reference CPU path)
//                 [--uniform 1]               (one shared launch power)
// Prints one JSON line.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "uwblink_b200/gn_integral.hpp"

using namespace uwblink;

int main(int argc, char** argv) {
  int iters = 5, n_r = 75, devices = 0, ref_iters = 0, uniform = 0;
  double density = 0.95;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i];
    if (a == "--iters") iters = std::atoi(argv[i + 1]);
    else if (a == "--n-r") n_r = std::atoi(argv[i + 1]);
    else if (a == "--density") density = std::atof(argv[i + 1]);
    else if (a == "--devices") devices = std::atoi(argv[i + 1]);
    else if (a == "--reference-iters") ref_iters = std::atoi(argv[i + 1]);
    else if (a == "--uniform") uniform = std::atoi(argv[i + 1]);
  }
  const BandPlan plan = default_band_plan();
  ChannelGrid grid = make_default_uwb_grid(plan);
  set_uniform_launch(grid, 1e-3);
  const FibreSpec fibre = default_fibre();
  LinkConfig lc;  // segmented mode, bounds [-5, 5] dBm, fd step 1e-3 dB (link_optimizer.hpp:159-171)
  lc.gn.n_r = n_r;
  lc.gn.mean_step_density = density;
  lc.lbfgs.max_iterations = iters;
  lc.uniform_mode = uniform != 0;
  long long evals = 0;
  b200::OptimiseOptions opt;
  opt.n_devices = devices;
  opt.cost_evals = &evals;
  int n_dev = devices;
  if (n_dev <= 0) b200::check(uwb_device_count(&n_dev));
  // device/context initialisation outside the timed loop
  for (int d = 0; d < n_dev; ++d) b200::Engine warm(d);
  const auto t0 = std::chrono::steady_clock::now();
  const OptimiseOutcome o = b200::optimise_launch_powers(fibre, grid, plan, lc, 0.0, opt);
  const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"config\": \"589ch O-U optimise_launch_powers %s, n_r %d, density %.2f\", "
              "\"devices\": %d, \"lbfgs_iterations\": %d, \"cost_evals\": %lld, \"wall_s\": %.4f, "
              "\"evals_per_s\": %.3f, \"objective\": %.17g, \"total_capacity_tbps\": %.6f, "
              "\"total_power_dbm\": %.6f, \"x0\": %.10g",
              uniform ? "uniform" : "segmented", n_r, density, n_dev, o.solver.iterations, evals, dt, evals / dt, o.solver.f,
              o.report.total_capacity / 1e12, o.report.total_power_dbm, o.solver.x[0]);
  if (ref_iters > 0) {
    LinkConfig lr = lc;
    lr.lbfgs.max_iterations = ref_iters;
    lr.gn.workers = 0;
    const auto r0 = std::chrono::steady_clock::now();
    const OptimiseOutcome r = optimise_launch_powers(fibre, grid, plan, lr, 0.0);
    const double rt = std::chrono::duration<double>(std::chrono::steady_clock::now() - r0).count();
    double dx = 0.0;
    for (std::size_t i = 0; i < r.solver.x.size(); ++i)
      dx = std::max(dx, std::abs(r.solver.x[i] - o.solver.x[i]));
    std::printf(", \"reference\": {\"lbfgs_iterations\": %d, \"wall_s\": %.4f, \"objective\": %.17g, "
                "\"max_abs_dx_db\": %.3e, \"rel_dobjective\": %.3e}",
                r.solver.iterations, rt, r.solver.f, dx, std::abs(o.solver.f / r.solver.f - 1.0));
  }
  std::printf("}\n");
  return 0;
}
