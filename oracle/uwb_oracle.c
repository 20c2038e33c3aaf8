/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  See uwb_oracle.h.
 *
 * Plain-C restatement of the reference algorithm.  Every function cites the
 * reference file:line (paths relative to /root/reference/proj/include/uwblink)
 * whose arithmetic it restates.  Operation order follows the reference so
 * that, compiled with -ffp-contract=off against the same libm, results are
 * bit-identical to the reference; tests/test_oracle_golden.py pins that.
 */
#define _GNU_SOURCE
#include "uwb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static const double kPi = 3.14159265358979323846;      /* units.hpp:11 */
static const double kC0 = 299792458.0;                 /* units.hpp:9 */
static const double kH = 6.62607015e-34;               /* units.hpp:10 */

static __thread char g_err[256];

const char* or_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

static double lam_of(double f) { return kC0 / f; }          /* units.hpp:37 */
static double db_km_to_m(double a) { return a * log(10.0) / 10.0 / 1000.0; } /* units.hpp:32-34 */

/* ===================== fibre_model.hpp ===================== */

/* TabulatedProfile::at, fibre_model.hpp:34-41 (upper_bound + linear). */
double or_table_at(const OrTable* t, double xq) {
  if (xq <= t->x[0]) return t->y[0];
  if (xq >= t->x[t->n - 1]) return t->y[t->n - 1];
  int i = 0; /* first index with x[i] > xq */
  while (i < t->n && !(t->x[i] > xq)) ++i;
  const double u = (xq - t->x[i - 1]) / (t->x[i] - t->x[i - 1]);
  return t->y[i - 1] + u * (t->y[i] - t->y[i - 1]);
}

/* fit_dispersion, fibre_model.hpp:93-152: normal equations on (1, dl, dl^2/2)
 * solved by Gaussian elimination with partial pivoting. */
static void fit_dispersion(OrFibre* f, double lambda_c, int order) {
  const int m = order + 1;
  double a[3][3] = {{0}}, rhs[3] = {0}, sol[3] = {0};
  for (int k = 0; k < f->d_table.n; ++k) {
    const double dl = f->d_table.x[k] - lambda_c;
    const double phi[3] = {1.0, dl, 0.5 * dl * dl};
    for (int i = 0; i < m; ++i) {
      rhs[i] += phi[i] * f->d_table.y[k];
      for (int j = 0; j < m; ++j) a[i][j] += phi[i] * phi[j];
    }
  }
  for (int col = 0; col < m; ++col) {
    int piv = col;
    for (int r = col + 1; r < m; ++r)
      if (fabs(a[r][col]) > fabs(a[piv][col])) piv = r;
    for (int c = 0; c < 3; ++c) {
      const double t = a[col][c];
      a[col][c] = a[piv][c];
      a[piv][c] = t;
    }
    { const double t = rhs[col]; rhs[col] = rhs[piv]; rhs[piv] = t; }
    const double diag = a[col][col];
    for (int r = col + 1; r < m; ++r) {
      const double fr = a[r][col] / diag;
      for (int c2 = col; c2 < m; ++c2) a[r][c2] -= fr * a[col][c2];
      rhs[r] -= fr * rhs[col];
    }
  }
  for (int r = m - 1; r >= 0; --r) {
    double acc = rhs[r];
    for (int c2 = r + 1; c2 < m; ++c2) acc -= a[r][c2] * sol[c2];
    acc /= a[r][r];
    sol[r] = acc;
  }
  f->lambda_c = lambda_c;
  f->d = sol[0];
  f->s = sol[1];
  f->sdot = order >= 2 ? sol[2] : 0.0;
  f->order = order;
}

double or_attenuation_at(const OrFibre* f, double lambda_m) {
  return db_km_to_m(or_table_at(&f->alpha_db_km, lambda_m)); /* :196-198, :256-258 */
}

double or_aeff_at(const OrFibre* f, double lambda_m) { return or_table_at(&f->aeff, lambda_m); }

/* gamma_at fibre_model.hpp:264-267 with n2_at :208-210 */
double or_gamma_at(const OrFibre* f, double lambda_m) {
  const double n2 = f->n2_scale * (f->n2_intercept + f->n2_slope * (lambda_m - f->lambda_ref));
  return 2.0 * kPi * n2 / (lambda_m * or_aeff_at(f, lambda_m));
}

/* beta_from_dispersion fibre_model.hpp:76-89 (dispersion_at :61-66, slope :68-72) */
int or_beta_from_dispersion(const OrFibre* f, double lambda_m, double b[3]) {
  if (!(lambda_m > 0.0)) return fail(OR_CONFIG_ERROR, "beta_from_dispersion: wavelength must be > 0");
  const double dl = lambda_m - f->lambda_c;
  double d = f->d + f->s * dl;
  if (f->order >= 2) d += 0.5 * f->sdot * dl * dl;
  double s = f->s;
  if (f->order >= 2) s += f->sdot * (lambda_m - f->lambda_c);
  const double sd = f->order >= 2 ? f->sdot : 0.0;
  const double tp = 2.0 * kPi * kC0;
  const double l = lambda_m;
  b[0] = -d * l * l / tp;
  b[1] = l * l * l / (tp * tp) * (2.0 * d + s * l);
  b[2] = -l * l * l * l / (tp * tp * tp) * (6.0 * d + 6.0 * s * l + sd * l * l);
  return OR_OK;
}

/* raman_gain_between fibre_model.hpp:221-227 */
double or_raman_gain_between(const OrFibre* f, double df_hz, double aeff_signal) {
  const double df = fabs(df_hz);
  if (df >= f->raman_gain.x[f->raman_gain.n - 1]) return 0.0;
  return or_table_at(&f->raman_gain, df) * f->aeff_ref / aeff_signal;
}

/* default_fibre fibre_model.hpp:287-351 */
void or_default_fibre(OrFibre* f) {
  memset(f, 0, sizeof *f);
  const int n = 84; /* detail::default_lambda_grid :272-276 */
  double grid[84];
  for (int i = 0; i <= 83; ++i) grid[i] = (1260.0 + 5.0 * i) * 1e-9;
  {
    const double a = -4.837314933693081e-5;
    const double r1 = 1302.3, r2 = 2986.799283154149;
    f->d_table.n = n;
    for (int i = 0; i < n; ++i) {
      const double lnm = grid[i] * 1e9;
      f->d_table.x[i] = grid[i];
      f->d_table.y[i] = a * (lnm - r1) * (lnm - r2) * 1e-6;
    }
  }
  fit_dispersion(f, 1438e-9, 2);
  {
    const double cr = 0.9421437757062556, air = 1.0264019670371897e12, lir = 48.48;
    f->alpha_db_km.n = n;
    for (int i = 0; i < n; ++i) {
      const double lum = grid[i] * 1e6;
      f->alpha_db_km.x[i] = grid[i];
      f->alpha_db_km.y[i] = cr / (lum * lum * lum * lum) + air * exp(-lir / lum);
    }
  }
  {
    const double a_core = 4.1e-6, n_clad = 1.444;
    const double n_core = n_clad / sqrt(1.0 - 2.0 * 0.0036);
    const double na = sqrt(n_core * n_core - n_clad * n_clad);
    f->aeff.n = n;
    for (int i = 0; i < n; ++i) {
      const double v = 2.0 * kPi * a_core * na / grid[i];
      const double w = a_core * (0.65 + 1.619 * pow(v, -1.5) + 2.879 * pow(v, -6.0));
      f->aeff.x[i] = grid[i];
      f->aeff.y[i] = kPi * w * w;
    }
  }
  f->lambda_ref = 1302.3e-9;
  f->n2_intercept = 2.6040013328848567e-20;
  f->n2_slope = -4.5e-15;
  f->n2_scale = 1.0;
  f->n2_scale = 2.0e-3 / or_gamma_at(f, 1302.3e-9);
  f->aeff_ref = 80e-12;
  f->raman_gain.n = 4;
  const double rx[4] = {0.0, 13.2e12, 30e12, 100e12}, ry[4] = {0.0, 0.39e-3, 0.0, 0.0};
  memcpy(f->raman_gain.x, rx, sizeof rx);
  memcpy(f->raman_gain.y, ry, sizeof ry);
  f->length_m = 80e3;
  f->span_count = 1;
}

/* uwtest::flat_fibre tests/support/test_helpers.hpp:22-29 */
void or_flat_fibre(OrFibre* f, double alpha_db_km, double length_m, int spans) {
  or_default_fibre(f);
  f->alpha_db_km.n = 2;
  f->alpha_db_km.x[0] = 1.0e-6;
  f->alpha_db_km.x[1] = 2.0e-6;
  f->alpha_db_km.y[0] = alpha_db_km;
  f->alpha_db_km.y[1] = alpha_db_km;
  f->length_m = length_m;
  f->span_count = spans;
}

/* ===================== channel_grid.hpp ===================== */

static int grid_alloc(OrGrid* g, int n) {
  g->n = n;
  g->freq = (double*)calloc((size_t)n, sizeof(double));
  g->psd = (double*)calloc((size_t)n, sizeof(double));
  g->guard = (uint8_t*)calloc((size_t)n, 1);
  return (g->freq && g->psd && g->guard) ? OR_OK : fail(1, "out of memory");
}

void or_grid_free(OrGrid* g) {
  free(g->freq);
  free(g->psd);
  free(g->guard);
  memset(g, 0, sizeof *g);
}

/* make_uniform_grid channel_grid.hpp:64-81 */
int or_make_uniform_grid(OrGrid* g, int n, double spacing, double bch, double centre) {
  if (n <= 0) return fail(OR_CONFIG_ERROR, "need at least one channel");
  if (grid_alloc(g, n)) return 1;
  g->spacing = spacing;
  g->bch = bch;
  g->centre = centre;
  const double mid = 0.5 * (double)(n - 1);
  for (int i = 0; i < n; ++i) g->freq[i] = centre + ((double)i - mid) * spacing;
  g->half_band = ((double)(n - 1) * 0.5) * spacing + 0.5 * bch;
  return OR_OK;
}

/* default_band_plan channel_grid.hpp:118-129 */
static const double kBandLo[6] = {1260e-9, 1360e-9, 1460e-9, 1530e-9, 1565e-9, 1625e-9};
static const double kBandHi[6] = {1360e-9, 1460e-9, 1530e-9, 1565e-9, 1625e-9, 1675e-9};
static const double kBandNf[6] = {7.0, 7.0, 7.0, 5.0, 6.0, 8.0};

int or_band_of_lambda(double lambda_m) { /* :101-108 */
  for (int b = 0; b < 6; ++b)
    if (lambda_m >= kBandLo[b] && lambda_m < kBandHi[b]) return b;
  return -1;
}

double or_band_nf_db(int band) { return band >= 0 && band < 6 ? kBandNf[band] : 5.0; }

/* make_default_uwb_grid channel_grid.hpp:133-143 with in_guard_zone :110-115 */
int or_make_default_uwb_grid(OrGrid* g) {
  int rc = or_make_uniform_grid(g, 589, 100e9, 96e9, kC0 / 1438e-9);
  if (rc) return rc;
  for (int i = 0; i < g->n; ++i) {
    const double lam = lam_of(g->freq[i]);
    int guard = 0;
    for (int b = 0; b + 1 < 6; ++b)
      if (fabs(lam - kBandHi[b]) <= 2.5e-9) guard = 1;
    g->guard[i] = (uint8_t)guard;
  }
  return OR_OK;
}

void or_set_channel_power(OrGrid* g, int i, double watts) { /* :30-32 */
  g->psd[i] = g->guard[i] ? 0.0 : watts / g->bch;
}

/* ChannelGrid::psd_at channel_grid.hpp:35-42 */
double or_psd_at(const OrGrid* g, double nu) {
  const double pos = (nu - g->freq[0]) / g->spacing;
  const long i = lround(pos);
  if (i < 0 || i >= (long)g->n) return 0.0;
  if (fabs(nu - g->freq[i]) > 0.5 * g->bch) return 0.0;
  return g->psd[i];
}

/* ===================== distance_grid.hpp:23-73 ===================== */

int or_distance_grid(double length_m, double density, int cap, double* edge, double* mid,
                     double* width, int* steps) {
  if (!(length_m > 0.0)) return fail(OR_CONFIG_ERROR, "build_distance_grid: length must be > 0");
  if (!(density > 0.0)) return fail(OR_CONFIG_ERROR, "build_distance_grid: density must be > 0");
  long n_edges = lround(density * length_m / 1e3) + 1;
  if (n_edges < 2) n_edges = 2;
  const int n = (int)n_edges;
  *steps = n - 1;
  if (n - 1 > cap) return OR_OK;
  const double n_steps = (double)(n - 1);
  const double uniform_step = length_m / n_steps;
  const double first_target = 1e3 / (10.0 * density);
  if (first_target >= uniform_step * 0.999) {
    for (int i = 0; i < n; ++i) edge[i] = length_m * (double)i / n_steps;
  } else {
    double lo = length_m * 1e-12, hi = length_m * 1e12;
    for (int it = 0; it < 200; ++it) {
      const double m = sqrt(lo * hi);
      const double t = log1p(length_m / m);
      if (m * expm1(t / n_steps) < first_target) lo = m; else hi = m;
    }
    const double z0 = sqrt(lo * hi);
    const double t = log1p(length_m / z0);
    for (int i = 0; i < n; ++i) edge[i] = z0 * expm1(t * (double)i / n_steps);
  }
  edge[0] = 0.0;
  edge[n - 1] = length_m;
  for (int i = 0; i + 1 < n; ++i) {
    mid[i] = 0.5 * (edge[i] + edge[i + 1]);
    width[i] = edge[i + 1] - edge[i];
  }
  return OR_OK;
}

/* ===================== rk45.hpp + raman_power.hpp ===================== */

/* Dormand-Prince tableau rk45.hpp:79-95 */
static const double kRkC[7] = {0.0, 1.0 / 5, 3.0 / 10, 4.0 / 5, 8.0 / 9, 1.0, 1.0};
static const double kRkA[7][6] = {
    {0},
    {1.0 / 5},
    {3.0 / 40, 9.0 / 40},
    {44.0 / 45, -56.0 / 15, 32.0 / 9},
    {19372.0 / 6561, -25360.0 / 2187, 64448.0 / 6561, -212.0 / 729},
    {9017.0 / 3168, -355.0 / 33, 46732.0 / 5247, 49.0 / 176, -5103.0 / 18656},
    {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84},
};
static const double kRkB5[7] = {35.0 / 384, 0.0, 500.0 / 1113, 125.0 / 192, -2187.0 / 6784, 11.0 / 84, 0.0};
static const double kRkB4[7] = {5179.0 / 57600, 0.0, 7571.0 / 16695, 393.0 / 640,
                                -92097.0 / 339200, 187.0 / 2100, 1.0 / 40};

typedef struct {
  int n;
  const double* alpha;
  const double* m; /* n*n or NULL */
  long evals;
} OdeSys;

/* RHS raman_power.hpp:90-101 */
static void ode_rhs(OdeSys* sys, const double* rho, double* drho) {
  const int n = sys->n;
  ++sys->evals;
  for (int i = 0; i < n; ++i) {
    double acc = -sys->alpha[i];
    if (sys->m) {
      const double* row = sys->m + (size_t)i * n;
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += row[j] * rho[j];
      acc += s;
    }
    drho[i] = rho[i] * acc;
  }
}

/* Rk45::integrate rk45.hpp:28-70 (rtol/atol from RamanSolveOptions :39-43,
 * initial step (z1-z0)/100, max_steps 2e6). */
static int rk45_integrate(OdeSys* sys, double z0, double z1, double* y, double* k[7],
                          double* ytmp, double* ynew, double rtol, double atol) {
  const int n = sys->n;
  double kE[7];
  for (int j = 0; j < 7; ++j) kE[j] = kRkB5[j] - kRkB4[j];
  double z = z0;
  double h = (z1 - z0) / 100.0;
  long steps = 0;
  ode_rhs(sys, y, k[0]);
  while (z < z1) {
    if (++steps > 2000000) return fail(OR_SOLVER_ERROR, "rk45: step budget exhausted");
    if (h > z1 - z) h = z1 - z;
    for (int s = 1; s < 7; ++s) {
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = 0; j < s; ++j) acc += kRkA[s][j] * k[j][i];
        ytmp[i] = y[i] + h * acc;
      }
      ode_rhs(sys, ytmp, k[s]);
    }
    double err = 0.0;
    for (int i = 0; i < n; ++i) {
      double y5 = 0.0, e = 0.0;
      for (int j = 0; j < 7; ++j) {
        y5 += kRkB5[j] * k[j][i];
        e += kE[j] * k[j][i];
      }
      ynew[i] = y[i] + h * y5;
      const double ay = fabs(y[i]), an = fabs(ynew[i]);
      const double sc = atol + rtol * (ay > an ? ay : an);
      const double r = h * e / sc;
      err += r * r;
    }
    err = sqrt(err / (double)n);
    if (err <= 1.0) {
      z += h;
      memcpy(y, ynew, (size_t)n * sizeof(double));
      double* t = k[0];
      k[0] = k[6];
      k[6] = t;
    }
    const double fac = err > 0.0 ? 0.9 * pow(err, -0.2) : 5.0;
    const double cl = fac < 0.2 ? 0.2 : fac;
    h *= (cl < 5.0 ? cl : 5.0);
    if (!(h > 0.0) || !isfinite(h)) return fail(OR_SOLVER_ERROR, "rk45: step size underflow");
  }
  return OR_OK;
}

/* solve_power_evolution raman_power.hpp:52-122 */
int or_power_evolution(const OrFibre* f, const OrGrid* g, const double* mid, int steps,
                       double length_m, int include_raman, double* log_rho, double* rho_end,
                       long* rhs_evals) {
  const int n = g->n;
  double* launch = (double*)malloc(sizeof(double) * n);
  double* alpha = (double*)malloc(sizeof(double) * n);
  double* m = include_raman ? (double*)calloc((size_t)n * n, sizeof(double)) : NULL;
  double* buf = (double*)malloc(sizeof(double) * n * 10);
  int rc = OR_OK;
  for (int i = 0; i < n; ++i) launch[i] = g->psd[i] * g->bch;
  for (int i = 0; i < n; ++i) alpha[i] = or_attenuation_at(f, lam_of(g->freq[i]));
  if (m) {
    for (int lo = 0; lo < n; ++lo) {
      const double aeff_lo = or_aeff_at(f, lam_of(g->freq[lo]));
      for (int hi = lo + 1; hi < n; ++hi) {
        const double gg = or_raman_gain_between(f, g->freq[hi] - g->freq[lo], aeff_lo);
        if (gg == 0.0) continue;
        const double ratio = g->freq[lo] / g->freq[hi];
        m[(size_t)lo * n + hi] = ratio * gg * launch[hi];
        m[(size_t)hi * n + lo] = -gg * launch[lo];
      }
    }
  }
  OdeSys sys = {n, alpha, m, 0};
  double* k[7];
  for (int s = 0; s < 7; ++s) k[s] = buf + (size_t)s * n;
  double* ytmp = buf + 7 * (size_t)n;
  double* ynew = buf + 8 * (size_t)n;
  double* rho = buf + 9 * (size_t)n;
  for (int i = 0; i < n; ++i) rho[i] = 1.0;
  double z = 0.0;
  for (int s = 0; s < steps && rc == OR_OK; ++s) {
    rc = rk45_integrate(&sys, z, mid[s], rho, k, ytmp, ynew, 1e-9, 1e-16);
    z = mid[s];
    for (int i = 0; i < n && rc == OR_OK; ++i) {
      if (!(rho[i] > 0.0)) rc = fail(OR_SOLVER_ERROR, "power evolution: non-positive rho");
      else log_rho[(size_t)i * steps + s] = log(rho[i]);
    }
  }
  if (rc == OR_OK) rc = rk45_integrate(&sys, z, length_m, rho, k, ytmp, ynew, 1e-9, 1e-16);
  if (rc == OR_OK) memcpy(rho_end, rho, sizeof(double) * n);
  if (rhs_evals) *rhs_evals = sys.evals;
  free(launch);
  free(alpha);
  free(m);
  free(buf);
  return rc;
}

/* ===================== gn_integral.hpp ===================== */

/* phase_mismatch gn_integral.hpp:43-50 */
double or_phase_mismatch(double f1, double f2, double fi, const double b[3]) {
  const double quartic = (f1 * f1 + f2 * f2) + 1.5 * (f1 * f2) + 3.0 * fi * (f1 + f2) + 3.0 * (fi * fi);
  const double bracket = b[0] + kPi * b[1] * ((f1 + f2) + 2.0 * fi) + (2.0 * kPi * kPi / 3.0) * b[2] * quartic;
  return -4.0 * kPi * kPi * (f1 * f2) * bracket;
}

/* quadrant_limits gn_integral.hpp:63-79 -> {b1, b2, s1, s2, u1_max} */
int or_quadrant_limits(int q, double half_band, double f, double o[5]) {
  if (fabs(f) > half_band) return fail(OR_CONFIG_ERROR, "quadrant_limits: channel offset must lie inside the half band");
  const double bm = half_band - f, bp = half_band + f;
  switch (q) {
    case 1: o[0] = bm; o[1] = bm; o[2] = +1.0; o[3] = +1.0; break;
    case 2: o[0] = bp; o[1] = bm; o[2] = -1.0; o[3] = +1.0; break;
    case 3: o[0] = bp; o[1] = bp; o[2] = -1.0; o[3] = -1.0; break;
    case 4: o[0] = bm; o[1] = bp; o[2] = +1.0; o[3] = -1.0; break;
    default: return fail(OR_CONFIG_ERROR, "quadrant_limits: quadrant index must be 1..4");
  }
  o[4] = o[0] * o[1];
  return OR_OK;
}

typedef struct { int i0, i1; double hw0, hw1; } Stencil;

/* stencil_for gn_integral.hpp:110-129 */
static Stencil stencil_for(const OrGrid* g, double nu) {
  Stencil s = {0, 0, 0.5, 0.0};
  const int n = g->n;
  if (n == 1) return s;
  const double pos = (nu - g->freq[0]) / g->spacing;
  if (pos <= 0.0) return s;
  if (pos >= (double)(n - 1)) {
    s.i0 = s.i1 = n - 1;
    return s;
  }
  const size_t k = (size_t)pos;
  const double t = pos - (double)k;
  s.i0 = (int)k;
  s.i1 = (int)k + 1;
  s.hw0 = 0.5 * (1.0 - t);
  s.hw1 = 0.5 * t;
  return s;
}

/* detail::kernel_abs2 gn_integral.hpp:136-191 */
static double kernel_abs2(const OrGrid* g, const OrSpan* spans, int n_spans,
                          const double* z_base, Stencil s1, Stencil s2, Stencil s3,
                          double* const* hl, double phi) {
  double re = 0.0, im = 0.0;
  for (int k = 0; k < n_spans; ++k) {
    const OrSpan* sv = &spans[k];
    const int nm = sv->steps;
    const double* c1a = sv->log_rho + (size_t)s1.i0 * nm;
    const double* c1b = sv->log_rho + (size_t)s1.i1 * nm;
    const double* c2a = sv->log_rho + (size_t)s2.i0 * nm;
    const double* c2b = sv->log_rho + (size_t)s2.i1 * nm;
    const double* c3a = sv->log_rho + (size_t)s3.i0 * nm;
    const double* c3b = sv->log_rho + (size_t)s3.i1 * nm;
    const double* hl4 = hl[k];
    const int fast = fabs(phi) * sv->width[nm - 1] > 1e-4;
    if (fast) {
      double pc = cos(phi * (z_base[k] + sv->edge[0]));
      double ps = sin(phi * (z_base[k] + sv->edge[0]));
      double sre = 0.0, sim = 0.0;
      for (int m = 0; m < nm; ++m) {
        const double lg = s1.hw0 * c1a[m] + s1.hw1 * c1b[m] + s2.hw0 * c2a[m] + s2.hw1 * c2b[m] +
                          s3.hw0 * c3a[m] + s3.hw1 * c3b[m] - hl4[m];
        const double p = exp(lg);
        const double ang = phi * (z_base[k] + sv->edge[m + 1]);
        const double nc = cos(ang), ns = sin(ang);
        sre += p * (nc - pc);
        sim += p * (ns - ps);
        pc = nc;
        ps = ns;
      }
      re += sim / phi;
      im += -sre / phi;
    } else {
      for (int m = 0; m < nm; ++m) {
        const double lg = s1.hw0 * c1a[m] + s1.hw1 * c1b[m] + s2.hw0 * c2a[m] + s2.hw1 * c2b[m] +
                          s3.hw0 * c3a[m] + s3.hw1 * c3b[m] - hl4[m];
        const double p = exp(lg);
        const double x = 0.5 * phi * sv->width[m];
        const double sinc = fabs(x) < 1e-8 ? 1.0 : sin(x) / x;
        const double ang = phi * (z_base[k] + sv->mid[m]);
        const double w = p * sv->width[m] * sinc;
        re += w * cos(ang);
        im += w * sin(ang);
      }
    }
  }
  (void)g;
  return re * re + im * im;
}

/* log_rho_at / p_k_factor raman_power.hpp:133-170 */
static double log_rho_at(const OrGrid* g, const OrSpan* sp, double nu, int m) {
  const int n = g->n;
  int i0 = 0, i1 = 0;
  double w0 = 1.0, w1 = 0.0;
  if (!(n == 1 || nu <= g->freq[0])) {
    if (nu >= g->freq[n - 1]) {
      i0 = i1 = n - 1;
    } else {
      const double pos = (nu - g->freq[0]) / g->spacing;
      const size_t k = (size_t)pos;
      i0 = (int)k;
      i1 = (int)k + 1;
      w1 = pos - (double)k;
      w0 = 1.0 - w1;
    }
  }
  return w0 * sp->log_rho[(size_t)i0 * sp->steps + m] + w1 * sp->log_rho[(size_t)i1 * sp->steps + m];
}

/* distance_kernel_abs2_reference gn_integral.hpp:198-214 */
double or_kernel_abs2_reference(const OrGrid* g, const OrSpan* spans, int n_spans, double nu1,
                                double nu2, double nu_ch, double phi) {
  double are = 0.0, aim = 0.0, z_base = 0.0;
  for (int k = 0; k < n_spans; ++k) {
    const OrSpan* sp = &spans[k];
    for (int m = 0; m < sp->steps; ++m) {
      const double l1 = log_rho_at(g, sp, nu1, m), l2 = log_rho_at(g, sp, nu2, m);
      const double l3 = log_rho_at(g, sp, nu1 + nu2 - nu_ch, m), l4 = log_rho_at(g, sp, nu_ch, m);
      const double p = exp(0.5 * (l1 + l2 + l3 - l4));
      const double dz = sp->width[m];
      const double x = 0.5 * phi * dz;
      const double sinc = fabs(x) < 1e-8 ? 1.0 : sin(x) / x;
      const double ang = phi * (z_base + sp->mid[m]);
      const double a = p * dz * sinc;
      are += a * cos(ang);
      aim += a * sin(ang);
    }
    z_base += sp->length;
  }
  return are * are + aim * aim;
}

/* nli_psd_at gn_integral.hpp:218-313 */
int or_nli_psd_at(const OrGrid* g, const OrSpan* spans, int n_spans, const double b[3],
                  double gamma, const OrNliCfg* cfg, double nu, double quad4[4], double* out) {
  if (n_spans <= 0) return fail(OR_CONFIG_ERROR, "nli_psd_at: need at least one span");
  const int n_r = cfg->n_r;
  if (n_r < 2) return fail(OR_CONFIG_ERROR, "nli_psd_at: n_r must be >= 2");
  const double f = nu - g->centre;
  const double b_hull = g->half_band;
  double z_base[64];
  double* hl[64];
  if (n_spans > 64) return fail(OR_CONFIG_ERROR, "oracle: at most 64 spans");
  const Stencil sc = stencil_for(g, nu);
  double zb = 0.0;
  for (int k = 0; k < n_spans; ++k) {
    z_base[k] = zb;
    zb += spans[k].length;
    const int nm = spans[k].steps;
    hl[k] = (double*)malloc(sizeof(double) * (size_t)nm);
    const double* ca = spans[k].log_rho + (size_t)sc.i0 * nm;
    const double* cb = spans[k].log_rho + (size_t)sc.i1 * nm;
    for (int m = 0; m < nm; ++m) hl[k][m] = sc.hw0 * ca[m] + sc.hw1 * cb[m];
  }
  double quad[4] = {0.0, 0.0, 0.0, 0.0};
  const int last_q = cfg->mirror_q4 ? 3 : 4;
  double* edges = (double*)malloc(sizeof(double) * (size_t)(n_r + 1));
  int rc = OR_OK;
  for (int q = 1; q <= last_q && rc == OR_OK; ++q) {
    double spec[5];
    rc = or_quadrant_limits(q, b_hull, f, spec);
    if (rc) break;
    if (!(spec[4] > 0.0)) continue;
    double sum = 0.0, comp = 0.0; /* detail::KahanSum :83-92 */
    const double u1_max = spec[4];
    if (cfg->u1_uniform) {
      for (int i = 0; i <= n_r; ++i) edges[i] = u1_max * (double)i / n_r;
    } else {
      edges[0] = 0.0;
      const double ln_min = log(cfg->u1_min_ratio);
      for (int i = 1; i <= n_r; ++i) edges[i] = u1_max * exp(ln_min * (double)(n_r - i) / (n_r - 1));
    }
    for (int i = 0; i < n_r; ++i) {
      const double e0 = edges[i], e1 = edges[i + 1];
      const double du1 = e1 - e0;
      const double u1 = (e0 == 0.0 || cfg->u1_uniform) ? 0.5 * (e0 + e1) : sqrt(e0 * e1);
      const double su = sqrt(u1);
      const double hi = log(spec[0] / su);
      const double lo = -log(spec[1] / su);
      if (!(hi > lo)) continue;
      const double du2 = (hi - lo) / n_r;
      double row = 0.0;
      for (int j = 0; j < n_r; ++j) {
        const double u2 = lo + ((double)j + 0.5) * du2;
        const double g1 = su * exp(u2);
        const double g2 = u1 / g1;
        const double f1 = spec[2] * g1;
        const double f2 = spec[3] * g2;
        const double p1 = or_psd_at(g, nu + f1);
        if (p1 == 0.0) continue;
        const double p2 = or_psd_at(g, nu + f2);
        if (p2 == 0.0) continue;
        const double p3 = or_psd_at(g, nu + f1 + f2);
        if (p3 == 0.0) continue;
        const Stencil s1 = stencil_for(g, nu + f1);
        const Stencil s2 = stencil_for(g, nu + f2);
        const Stencil s3 = stencil_for(g, nu + f1 + f2);
        const double phi = or_phase_mismatch(f1, f2, f, b);
        row += p1 * p2 * p3 * kernel_abs2(g, spans, n_spans, z_base, s1, s2, s3, hl, phi);
      }
      const double x = row * du1 * du2;
      const double y = x - comp;
      const double t = sum + y;
      comp = (t - sum) - y;
      sum = t;
    }
    quad[q - 1] = sum;
  }
  free(edges);
  for (int k = 0; k < n_spans; ++k) free(hl[k]);
  if (rc) return rc;
  if (cfg->mirror_q4) quad[3] = quad[1];
  if (quad4) memcpy(quad4, quad, sizeof quad);
  *out = (16.0 / 27.0) * gamma * gamma * (quad[0] + quad[1] + quad[2] + quad[3]);
  return OR_OK;
}

/* channel_nli gn_integral.hpp:316-329 */
static int channel_nli(const OrGrid* g, const OrSpan* spans, int n_spans, const double b[3],
                       double gamma, const OrNliCfg* cfg, int ch, double quad4[4], double* out) {
  const double nu = g->freq[ch];
  double psd_c;
  int rc = or_nli_psd_at(g, spans, n_spans, b, gamma, cfg, nu, quad4, &psd_c);
  if (rc) return rc;
  if (cfg->simpson) {
    double g_lo, g_hi;
    rc = or_nli_psd_at(g, spans, n_spans, b, gamma, cfg, nu - 0.5 * g->bch, NULL, &g_lo);
    if (rc) return rc;
    rc = or_nli_psd_at(g, spans, n_spans, b, gamma, cfg, nu + 0.5 * g->bch, NULL, &g_hi);
    if (rc) return rc;
    psd_c = (g_lo + 4.0 * psd_c + g_hi) / 6.0;
  }
  *out = psd_c;
  return OR_OK;
}

typedef struct {
  const OrGrid* g;
  const OrSpan* spans;
  int n_spans;
  const double* b;
  const double* gamma;
  const OrNliCfg* cfg;
  double *eta, *nli_psd, *nli_power, *quad4;
  uint8_t* skipped;
  int begin, end, rc;
  char err[256];
} Batch;

/* body of all_channels_nli gn_integral.hpp:348-359 over one contiguous batch
 * (parallel_for_batches parallel.hpp:21-47). */
static void* run_batch(void* arg) {
  Batch* bt = (Batch*)arg;
  for (int ch = bt->begin; ch < bt->end && bt->rc == OR_OK; ++ch) {
    const OrGrid* g = bt->g;
    if (g->guard[ch] || g->psd[ch] <= 0.0) {
      bt->skipped[ch] = 1;
      continue;
    }
    double psd;
    double* q4 = bt->quad4 ? bt->quad4 + 4 * (size_t)ch : NULL;
    double tmpq[4];
    bt->rc = channel_nli(g, bt->spans, bt->n_spans, bt->b, bt->gamma[ch], bt->cfg, ch,
                         q4 ? q4 : tmpq, &psd);
    if (bt->rc) {
      snprintf(bt->err, sizeof bt->err, "%s", g_err);
      break;
    }
    const double p = g->psd[ch] * g->bch;
    bt->nli_psd[ch] = psd;
    bt->nli_power[ch] = psd * g->bch;
    bt->eta[ch] = bt->nli_power[ch] / (p * p * p);
  }
  return NULL;
}

/* all_channels_nli gn_integral.hpp:334-363 (gamma supplied per channel,
 * = gamma_at(fibre, lambda(ch)) in the reference :353). */
int or_all_channels_nli(const OrGrid* g, const OrSpan* spans, int n_spans, const double b[3],
                        const double* gamma_per_ch, const OrNliCfg* cfg, double* eta,
                        double* nli_psd, double* nli_power, double* quad4, uint8_t* skipped) {
  const int n = g->n;
  for (int i = 0; i < n; ++i) {
    eta[i] = nli_psd[i] = nli_power[i] = 0.0;
    skipped[i] = 0;
    if (quad4) quad4[4 * i] = quad4[4 * i + 1] = quad4[4 * i + 2] = quad4[4 * i + 3] = 0.0;
  }
  int w = cfg->workers > 0 ? cfg->workers : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (w < 1) w = 1;
  if (w > n) w = n;
  Batch* bs = (Batch*)calloc((size_t)w, sizeof(Batch));
  pthread_t* th = (pthread_t*)calloc((size_t)w, sizeof(pthread_t));
  for (int k = 0; k < w; ++k) {
    Batch* bt = &bs[k];
    bt->g = g; bt->spans = spans; bt->n_spans = n_spans; bt->b = b; bt->gamma = gamma_per_ch;
    bt->cfg = cfg; bt->eta = eta; bt->nli_psd = nli_psd; bt->nli_power = nli_power;
    bt->quad4 = quad4; bt->skipped = skipped;
    bt->begin = (int)((long)n * k / w);
    bt->end = (int)((long)n * (k + 1) / w);
    if (w == 1) run_batch(bt);
    else pthread_create(&th[k], NULL, run_batch, bt);
  }
  int rc = OR_OK;
  for (int k = 0; k < w; ++k) {
    if (w > 1) pthread_join(th[k], NULL);
    if (rc == OR_OK && bs[k].rc) {
      rc = bs[k].rc;
      snprintf(g_err, sizeof g_err, "%s", bs[k].err);
    }
  }
  free(bs);
  free(th);
  return rc;
}

/* uwtest::cartesian_nli_psd tests/support/test_helpers.hpp:43-70 */
int or_cartesian_nli_psd(const OrGrid* g, const OrSpan* spans, int n_spans, const double b[3],
                         double gamma, double nu, int n_cells, double* out) {
  const double f = nu - g->centre;
  const double lo = -(g->half_band + f);
  const double hi = g->half_band - f;
  const double d = (hi - lo) / n_cells;
  double total = 0.0;
  for (int i = 0; i < n_cells; ++i) {
    const double f1 = lo + (i + 0.5) * d;
    const double p1 = or_psd_at(g, nu + f1);
    if (p1 == 0.0) continue;
    double row = 0.0;
    for (int j = 0; j < n_cells; ++j) {
      const double f2 = lo + (j + 0.5) * d;
      const double p2 = or_psd_at(g, nu + f2);
      if (p2 == 0.0) continue;
      const double p3 = or_psd_at(g, nu + f1 + f2);
      if (p3 == 0.0) continue;
      const double phi = or_phase_mismatch(f1, f2, f, b);
      row += p1 * p2 * p3 * or_kernel_abs2_reference(g, spans, n_spans, nu + f1, nu + f2, nu, phi);
    }
    total += row * d * d;
  }
  *out = (16.0 / 27.0) * gamma * gamma * total;
  return OR_OK;
}

/* ===================== link_optimizer.hpp ===================== */

/* ase_power link_optimizer.hpp:22-26 */
double or_ase_power(double nf_db, double gain, double f, double bch) {
  const double n_sp = 0.5 * pow(10.0, nf_db / 10.0);
  return 2.0 * n_sp * kH * f * (gain - 1.0) * bch;
}

/* assemble_link_report link_optimizer.hpp:194-237 on the default band plan */
int or_assemble_link_report(const OrGrid* g, int span_count, const double* eta,
                            const double* rho_end, int use_snr_trx, double snr_trx_db,
                            double* p_ase, double* snr_db, double* capacity, double totals3[3]) {
  double total_w = 0.0, loss = 0.0, total_cap = 0.0;
  const double snr_trx = use_snr_trx ? pow(10.0, snr_trx_db / 10.0) : 0.0;
  for (int i = 0; i < g->n; ++i) {
    p_ase[i] = snr_db[i] = capacity[i] = 0.0;
    const int band = or_band_of_lambda(lam_of(g->freq[i]));
    if (g->guard[i] || g->psd[i] <= 0.0) continue;
    const double p = g->psd[i] * g->bch;
    const double gain = 1.0 / rho_end[i];
    const double nf = band >= 0 ? kBandNf[band] : 5.0;
    if ((gain > 1.0 ? gain : 1.0) < 1.0) return fail(OR_CONFIG_ERROR, "ase_power: gain below 1");
    p_ase[i] = (double)span_count * or_ase_power(nf, gain > 1.0 ? gain : 1.0, g->freq[i], g->bch);
    double denom = eta[i] * p * p * p + p_ase[i];
    if (use_snr_trx) denom += p / snr_trx;
    const double snr = p / denom;
    snr_db[i] = 10.0 * log10(snr);
    capacity[i] = 2.0 * g->bch * log2(1.0 + snr);
    loss -= log2(1.0 + snr);
    total_cap += capacity[i];
    total_w += p;
  }
  totals3[0] = loss;
  totals3[1] = total_cap;
  totals3[2] = total_w > 0.0 ? 10.0 * log10(total_w / 1e-3) : -300.0;
  return OR_OK;
}

/* ---- closed-form model (gn_closed_form.hpp) ---------------------------- */

/* phi_xpm gn_closed_form.hpp:23-27 */
double or_phi_xpm(double f_i, double f_k, const double b[3]) {
  const double bracket = b[0] + kPi * b[1] * (f_i + f_k) +
                         (2.0 * kPi * kPi / 3.0) * b[2] * (f_i * f_i + f_i * f_k + f_k * f_k);
  return -4.0 * kPi * kPi * bracket * (f_k - f_i);
}

/* phi_spm :30-33 */
double or_phi_spm(double f_i, const double b[3]) {
  return -4.0 * kPi * kPi *
         (b[0] + 2.0 * kPi * b[1] * f_i + 2.0 * kPi * kPi * b[2] * f_i * f_i);
}

/* effective_alpha :37-47 (bisection, 200 iterations) */
double or_effective_alpha(double l_eff, double length) {
  if (l_eff >= length) return 1e-12;
  double lo = 1e-12, hi = 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double val = (1.0 - exp(-mid * length)) / mid;
    if (val > l_eff) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

/* detail::xpm_island :53-59 */
double or_xpm_island(double phi_abs, double bch, double alpha) {
  const double x = phi_abs * bch / (2.0 * alpha);
  if (x < 1e-3) return (0.75 - (5.0 / 24.0) * x * x) * bch * bch / (alpha * alpha);
  return 2.0 * bch / (alpha * phi_abs) * atan(x) - log1p(x * x) / (phi_abs * phi_abs);
}

/* cfm_all_channels_nli :70-144 (kCfmSpmCalibration / kCfmXpmCalibration :67-68) */
int or_cfm_all_channels_nli(const OrGrid* g, const OrSpan* spans, int n_spans, const double b[3],
                            const double* gamma_ch, double* eta, double* nli_psd,
                            double* nli_power, uint8_t* skipped) {
  const int n = g->n;
  const double spm_cal = 1.9641, xpm_cal = 1.0571;
  for (int i = 0; i < n; ++i) {
    eta[i] = nli_psd[i] = nli_power[i] = 0.0;
    skipped[i] = 0;
  }
  if (n_spans < 1) return fail(OR_CONFIG_ERROR, "cfm: need at least one span");
  double* alpha_eff = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int s = 0; s < n_spans; ++s) {
    const OrSpan* ev = &spans[s];
    const double span_len = ev->length;
    for (int i = 0; i < n; ++i) {
      alpha_eff[i] = 1e-12;
      double l_eff = 0.0;
      for (int m = 0; m < ev->steps; ++m)
        l_eff += exp(ev->log_rho[(size_t)i * ev->steps + m]) * ev->width[m];
      if (l_eff > 0.0) alpha_eff[i] = or_effective_alpha(l_eff < span_len ? l_eff : span_len, span_len);
    }
    for (int i = 0; i < n; ++i) {
      if (g->guard[i] || g->psd[i] <= 0.0) {
        skipped[i] = 1;
        continue;
      }
      const double p_i = g->psd[i] * g->bch;
      const double f_i = g->freq[i] - g->centre;
      double eta_i = 0.0;
      const double phi_i = fabs(or_phi_spm(f_i, b));
      const double a_i = alpha_eff[i];
      const double spm_arg = phi_i * g->bch * g->bch / (8.0 * a_i);
      double spm;
      if (spm_arg < 1e-3)
        spm = (kPi / (a_i * (phi_i > 1e-300 ? phi_i : 1e-300))) * spm_arg;
      else
        spm = (kPi / (a_i * phi_i)) * asinh(spm_arg);
      eta_i += spm_cal * (16.0 / 27.0) * (gamma_ch[i] * gamma_ch[i] / (g->bch * g->bch)) * spm;
      for (int k = 0; k < n; ++k) {
        if (k == i || g->guard[k] || g->psd[k] <= 0.0) continue;
        const double p_k = g->psd[k] * g->bch;
        const double phik = fabs(or_phi_xpm(f_i, g->freq[k] - g->centre, b));
        const double island = or_xpm_island(phik, g->bch, alpha_eff[k]);
        const double ratio = p_k / p_i;
        eta_i += xpm_cal * (32.0 / 27.0) * (gamma_ch[i] * gamma_ch[k] / (g->bch * g->bch)) *
                 ratio * ratio * island;
      }
      eta[i] += eta_i;
    }
  }
  free(alpha_eff);
  for (int i = 0; i < n; ++i) {
    if (skipped[i]) continue;
    const double p = g->psd[i] * g->bch;
    nli_power[i] = eta[i] * p * p * p;
    nli_psd[i] = nli_power[i] / g->bch;
  }
  return OR_OK;
}
