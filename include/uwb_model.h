/*
 * uwb_model.h — host-side scenario builders exported by libuwbnli.so.
 *
 * Not part of the hot path: they restate the reference's input builders so
 * that the BASELINE workloads can be assembled on a machine without the
 * reference tree (the GPU box).  A reference user keeps calling the
 * reference's own builders and passes their outputs to include/uwb_nli.h.
 *
 *   uwb_model_fibre          <- default_fibre + attenuation_at/aeff_at/gamma_at
 *                               + beta_from_dispersion (fibre_model.hpp:76-351);
 *                               kind 1 = uwtest::flat_fibre (test_helpers.hpp:22)
 *   uwb_model_grid           <- make_uniform_grid / make_default_uwb_grid +
 *                               default_band_plan (channel_grid.hpp:64-143)
 *   uwb_model_distance_grid  <- build_distance_grid (distance_grid.hpp:23-73)
 */
#ifndef UWB_MODEL_H
#define UWB_MODEL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double* alpha;         /* [n] 1/m   (may be NULL) */
  double* aeff;          /* [n] m^2   (may be NULL) */
  double* gamma;         /* [n] 1/(W m) (may be NULL) */
  double beta[3];        /* at lambda_beta */
  int raman_n;
  double raman_x[16];
  double raman_y[16];
  double raman_aeff_ref;
  double dispersion[4];  /* lambda_c, d, s, sdot of the quadratic fit */
} uwb_fibre_sample;

int uwb_model_fibre(int kind, double flat_alpha_db_km, int n, const double* freq,
                    double lambda_beta, uwb_fibre_sample* out);

/* uwb_default != 0 ignores n/spacing/bch/centre and builds the 589-channel
 * O->U plan with guard slots.  band/nf_db follow default_band_plan(). */
int uwb_model_grid(int uwb_default, int n, double spacing, double bch, double centre,
                   double* freq, uint8_t* guard, int* band, double* nf_db, double* half_band);

int uwb_model_distance_grid(double length_m, double density, int cap, double* edge, double* mid,
                            double* width, int* steps);

#ifdef __cplusplus
}
#endif
#endif
