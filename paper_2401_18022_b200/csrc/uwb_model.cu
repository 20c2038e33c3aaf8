// Host-side scenario builders: the data formats either side of the path.
// They let a caller (bench.py, the Python mirror, a C program) assemble the
// BASELINE workloads without the reference tree: the built-in fibre model
// (fibre_model.hpp:287-351), the 589-channel band plan (channel_grid.hpp:
// 118-143) and the distance grid (distance_grid.hpp:23-73).  Host code only;
// everything here runs once per scenario, off the hot path.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/uwb_model.h"
#include "../../include/uwb_nli.h"
#include "uwb_capi_internal.cuh"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kC0 = 299792458.0;

struct Table {
  std::vector<double> x, y;
  // TabulatedProfile::at (fibre_model.hpp:34-41)
  double at(double xq) const {
    if (xq <= x.front()) return y.front();
    if (xq >= x.back()) return y.back();
    const size_t i = static_cast<size_t>(std::upper_bound(x.begin(), x.end(), xq) - x.begin());
    const double t = (xq - x[i - 1]) / (x[i] - x[i - 1]);
    return y[i - 1] + t * (y[i] - y[i - 1]);
  }
};

struct Fibre {
  double lambda_c = 0, d = 0, s = 0, sdot = 0;
  int order = 2;
  Table d_table, alpha_db_km, aeff, raman;
  double n2_intercept = 0, n2_slope = 0, lambda_ref = 0, n2_scale = 1, aeff_ref = 80e-12;

  double gamma_at(double lam) const {  // fibre_model.hpp:264-267
    const double n2 = n2_scale * (n2_intercept + n2_slope * (lam - lambda_ref));
    return 2.0 * kPi * n2 / (lam * aeff.at(lam));
  }
  double alpha_at(double lam) const {  // :256-258 via db_per_km_to_per_m units.hpp:32-34
    return alpha_db_km.at(lam) * std::log(10.0) / 10.0 / 1000.0;
  }
};

// Least-squares quadratic D(lambda) about lambda_c (fit_dispersion :93-152).
void fit_dispersion(Fibre* f, double lambda_c, int order) {
  const int m = order + 1;
  double a[3][3] = {}, rhs[3] = {}, sol[3] = {};
  for (size_t k = 0; k < f->d_table.x.size(); ++k) {
    const double dl = f->d_table.x[k] - lambda_c;
    const double basis[3] = {1.0, dl, 0.5 * dl * dl};
    for (int i = 0; i < m; ++i) {
      rhs[i] += basis[i] * f->d_table.y[k];
      for (int j = 0; j < m; ++j) a[i][j] += basis[i] * basis[j];
    }
  }
  for (int col = 0; col < m; ++col) {
    int piv = col;
    for (int r = col + 1; r < m; ++r)
      if (std::abs(a[r][col]) > std::abs(a[piv][col])) piv = r;
    for (int c = 0; c < 3; ++c) std::swap(a[col][c], a[piv][c]);
    std::swap(rhs[col], rhs[piv]);
    for (int r = col + 1; r < m; ++r) {
      const double fr = a[r][col] / a[col][col];
      for (int c = col; c < m; ++c) a[r][c] -= fr * a[col][c];
      rhs[r] -= fr * rhs[col];
    }
  }
  for (int r = m - 1; r >= 0; --r) {
    double acc = rhs[r];
    for (int c = r + 1; c < m; ++c) acc -= a[r][c] * sol[c];
    acc /= a[r][r];
    sol[r] = acc;
  }
  f->lambda_c = lambda_c;
  f->d = sol[0];
  f->s = sol[1];
  f->sdot = order >= 2 ? sol[2] : 0.0;
  f->order = order;
}

// default_fibre (fibre_model.hpp:287-351).
Fibre default_fibre() {
  Fibre f;
  std::vector<double> grid;
  for (int i = 0; i <= 83; ++i) grid.push_back((1260.0 + 5.0 * i) * 1e-9);
  const double a = -4.837314933693081e-5, r1 = 1302.3, r2 = 2986.799283154149;
  for (double l : grid) {
    const double lnm = l * 1e9;
    f.d_table.x.push_back(l);
    f.d_table.y.push_back(a * (lnm - r1) * (lnm - r2) * 1e-6);
  }
  fit_dispersion(&f, 1438e-9, 2);
  const double cr = 0.9421437757062556, air = 1.0264019670371897e12, lir = 48.48;
  for (double l : grid) {
    const double lum = l * 1e6;
    f.alpha_db_km.x.push_back(l);
    f.alpha_db_km.y.push_back(cr / (lum * lum * lum * lum) + air * std::exp(-lir / lum));
  }
  const double a_core = 4.1e-6, n_clad = 1.444;
  const double n_core = n_clad / std::sqrt(1.0 - 2.0 * 0.0036);
  const double na = std::sqrt(n_core * n_core - n_clad * n_clad);
  for (double l : grid) {
    const double v = 2.0 * kPi * a_core * na / l;
    const double w = a_core * (0.65 + 1.619 * std::pow(v, -1.5) + 2.879 * std::pow(v, -6.0));
    f.aeff.x.push_back(l);
    f.aeff.y.push_back(kPi * w * w);
  }
  f.lambda_ref = 1302.3e-9;
  f.n2_intercept = 2.6040013328848567e-20;
  f.n2_slope = -4.5e-15;
  f.n2_scale = 1.0;
  f.n2_scale = 2.0e-3 / f.gamma_at(1302.3e-9);
  f.aeff_ref = 80e-12;
  f.raman.x = {0.0, 13.2e12, 30e12, 100e12};
  f.raman.y = {0.0, 0.39e-3, 0.0, 0.0};
  return f;
}

// beta_from_dispersion (fibre_model.hpp:76-89).
std::array<double, 3> betas_at(const Fibre& f, double l) {
  const double dl = l - f.lambda_c;
  double d = f.d + f.s * dl;
  if (f.order >= 2) d += 0.5 * f.sdot * dl * dl;
  double s = f.s;
  if (f.order >= 2) s += f.sdot * (l - f.lambda_c);
  const double sd = f.order >= 2 ? f.sdot : 0.0;
  const double tp = 2.0 * kPi * kC0;
  return {-d * l * l / tp, l * l * l / (tp * tp) * (2.0 * d + s * l),
          -l * l * l * l / (tp * tp * tp) * (6.0 * d + 6.0 * s * l + sd * l * l)};
}

// default_band_plan (channel_grid.hpp:118-129).
struct Band {
  double lo, hi, nf;
};
constexpr Band kBands[6] = {{1260e-9, 1360e-9, 7.0}, {1360e-9, 1460e-9, 7.0},
                            {1460e-9, 1530e-9, 7.0}, {1530e-9, 1565e-9, 5.0},
                            {1565e-9, 1625e-9, 6.0}, {1625e-9, 1675e-9, 8.0}};

}  // namespace

extern "C" {

int uwb_model_fibre(int kind, double flat_alpha_db_km, int n, const double* freq,
                    double lambda_beta, uwb_fibre_sample* out) {
  if (!out || (n > 0 && !freq)) return uwb::fail(UWB_CONFIG_ERROR, "null argument");
  if (!(lambda_beta > 0.0))
    return uwb::fail(UWB_CONFIG_ERROR, "beta_from_dispersion: wavelength must be > 0");
  Fibre f = default_fibre();
  if (kind == 1) {  // uwtest::flat_fibre (tests/support/test_helpers.hpp:22-29)
    f.alpha_db_km.x = {1.0e-6, 2.0e-6};
    f.alpha_db_km.y = {flat_alpha_db_km, flat_alpha_db_km};
  }
  for (int i = 0; i < n; ++i) {
    const double lam = kC0 / freq[i];
    if (out->alpha) out->alpha[i] = f.alpha_at(lam);
    if (out->aeff) out->aeff[i] = f.aeff.at(lam);
    if (out->gamma) out->gamma[i] = f.gamma_at(lam);
  }
  const auto b = betas_at(f, lambda_beta);
  std::copy(b.begin(), b.end(), out->beta);
  out->raman_n = static_cast<int>(f.raman.x.size());
  for (int i = 0; i < out->raman_n && i < 16; ++i) {
    out->raman_x[i] = f.raman.x[i];
    out->raman_y[i] = f.raman.y[i];
  }
  out->raman_aeff_ref = f.aeff_ref;
  out->dispersion[0] = f.lambda_c;
  out->dispersion[1] = f.d;
  out->dispersion[2] = f.s;
  out->dispersion[3] = f.sdot;
  return UWB_OK;
}

int uwb_model_grid(int uwb_default, int n, double spacing, double bch, double centre,
                   double* freq, uint8_t* guard, int* band, double* nf_db, double* half_band) {
  if (uwb_default) {  // make_default_uwb_grid (channel_grid.hpp:133-143)
    n = 589;
    spacing = 100e9;
    bch = 96e9;
    centre = kC0 / 1438e-9;
  }
  if (n <= 0) return uwb::fail(UWB_CONFIG_ERROR, "need at least one channel");
  const double mid = 0.5 * static_cast<double>(n - 1);
  for (int i = 0; i < n; ++i) {
    const double f = centre + (static_cast<double>(i) - mid) * spacing;  // :74-77
    const double lam = kC0 / f;
    if (freq) freq[i] = f;
    int b = -1;
    for (int k = 0; k < 6; ++k)
      if (lam >= kBands[k].lo && lam < kBands[k].hi) {
        b = k;
        break;
      }
    if (band) band[i] = b;
    if (nf_db) nf_db[i] = b >= 0 ? kBands[b].nf : 5.0;
    if (guard) {
      uint8_t gd = 0;
      if (uwb_default)
        for (int k = 0; k + 1 < 6; ++k)
          if (std::abs(lam - kBands[k].hi) <= 2.5e-9) gd = 1;  // in_guard_zone :110-115
      guard[i] = gd;
    }
  }
  if (half_band) *half_band = (static_cast<double>(n - 1) * 0.5) * spacing + 0.5 * bch;
  return UWB_OK;
}

int uwb_model_distance_grid(double length_m, double density, int cap, double* edge, double* mid,
                            double* width, int* steps) {
  std::vector<double> e, m, w;
  const int rc = uwb::distance_grid_host(length_m, density, &e, &m, &w);
  if (rc) return rc;
  if (steps) *steps = static_cast<int>(m.size());
  if (static_cast<int>(m.size()) > cap) return UWB_OK;
  if (edge) std::memcpy(edge, e.data(), e.size() * sizeof(double));
  if (mid) std::memcpy(mid, m.data(), m.size() * sizeof(double));
  if (width) std::memcpy(width, w.data(), w.size() * sizeof(double));
  return UWB_OK;
}

}  // extern "C"
