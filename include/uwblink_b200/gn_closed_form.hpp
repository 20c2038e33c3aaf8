// uwblink_b200/gn_closed_form.hpp — C++ drop-in for the closed-form model.
//
//   uwblink::b200::cfm_all_channels_nli <- uwblink::cfm_all_channels_nli
//                                          gn_closed_form.hpp:70-144
//
// Same signature and types as the reference; the SPM + pairwise XPM sums
// run on the device (uwb_cfm_all_channels_nli, libuwbnli.so).  Errors are the
// reference's ConfigError; a missing B200 throws b200::DeviceError.
#pragma once

#include <cstddef>
#include <vector>

#include "uwblink/gn_closed_form.hpp"
#include "uwblink_b200/gn_integral.hpp"

namespace uwblink::b200 {

[[nodiscard]] inline NliResult cfm_all_channels_nli(const ChannelGrid& grid,
                                                    const std::vector<PowerEvolution>& spans,
                                                    const BetaCoefficients& betas,
                                                    const FibreSpec& fibre) {
  const std::size_t n = grid.size();
  if (spans.empty()) throw ConfigError("cfm: need at least one span");  // :80
  for (const auto& evo : spans)
    if (evo.channels() != n) throw ConfigError("cfm: span evolution does not match the grid");
  std::vector<double> gamma(n);
  for (std::size_t i = 0; i < n; ++i) gamma[i] = gamma_at(fibre, freq_to_lambda(grid.freq[i]));
  const uwb_grid g = detail::grid_view(grid);
  const std::vector<uwb_span> sv = detail::span_views(spans);
  const double beta[3] = {betas.beta2, betas.beta3, betas.beta4};
  NliResult r;
  r.eta.assign(n, 0.0);
  r.nli_psd.assign(n, 0.0);
  r.nli_power.assign(n, 0.0);
  r.quadrant.assign(n, {0.0, 0.0, 0.0, 0.0});
  r.skipped.assign(n, 0);
  uwb_nli_result o{};
  o.eta = r.eta.data();
  o.nli_psd = r.nli_psd.data();
  o.nli_power = r.nli_power.data();
  o.skipped = r.skipped.data();
  check(uwb_cfm_all_channels_nli(engine().get(), &g, static_cast<int>(sv.size()), sv.data(), beta,
                                 gamma.data(), &o));
  r.elapsed_seconds = o.elapsed_seconds;
  return r;
}

}  // namespace uwblink::b200
