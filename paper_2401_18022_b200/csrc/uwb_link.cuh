// Prepared (device-resident) full SNR evaluation: the state uwb_link.cu keeps
// between calls and the stage functions the single- and multi-device entry
// points share (uwb_link.cu, uwb_multi.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/uwb_nli.h"
#include "nli_kernel.cuh"
#include "raman_ode.cuh"
#include "uwb_ctx.cuh"

namespace uwb {

// assemble_link_report's device view (link_optimizer.hpp:194-237).
struct LinkDev {
  int n;
  const double* freq;
  const double* psd;
  const uint8_t* guard;
  double bch;
  const double* eta;
  const double* rho_end;
  const double* nf_db;
  const int* band;
  int n_bands;
  int span_count;
  int use_snr_trx;
  double snr_trx;
  double* out;  // [4n] eta | p_ase | snr_db | capacity, then [3] totals, then [2*n_bands]
  double* tmp;  // [3n] per-channel p, capacity, log2(1+snr) for the ordered sums
};

}  // namespace uwb

// Everything evaluate_link keeps resident between calls.
struct uwb_ctx::Prepared {
  int n = 0;
  int steps = 0;
  int span_count = 1;
  int include_raman = 1;
  double rtol = 1e-9, atol = 1e-16, length = 0.0;
  uwb_nli_cfg cfg{};
  uwb::NliParams P{};
  uwb::FinalizeParams F{};
  uwb::OdeParams O{};
  uwb::LinkDev L{};
  int raman_n = 0;
  double aeff_ref = 0.0;
  const double* d_aeff = nullptr;
  int* d_status = nullptr;
  long long* d_rhs = nullptr;
  double* d_psd = nullptr;  // the NLI/ODE/link read launch PSD from here
  int grid_ctas = 0;
  int setup_ctas = 0;      // split evaluation: the setup pass's grid (0: fused kernel)
  int list_ctas = 0;       // and the list pass's
  size_t split_bytes = 0;  // its point lists, allocated by the first single evaluation
  int launches = 0;
};

namespace uwb {

// evaluate_link's stages on a prepared context (uwb_link.cu).
// sync = false only when everything that reads the prepared state runs on the
// context's own stream (uwb_evaluate_link); the public prepare synchronises so
// resident calls may use any stream.
int prepare(uwb_ctx* c, const uwb_grid* g, const uwb_fibre* fb, const uwb_link_cfg* lk,
            const uwb_nli_cfg* cfg, bool sync = true);
// solve_link_noise (link_optimizer.hpp:181-190): Raman ODE + NLI of the
// context's channels; psd_dev = launch PSD on the device, or null for the
// prepared one.
int run_noise(uwb_ctx* c, const double* psd_dev, cudaStream_t st, bool reset_status = true);
// assemble_link_report (link_optimizer.hpp:194-237) from the context's eta.
int run_report(uwb_ctx* c, cudaStream_t st, const LinkDev* Lp = nullptr);
int run_prepared(uwb_ctx* c, const double* psd_dev, cudaStream_t st, bool reset_status = true);
// SolverError from the device status word (synchronises the context stream).
int check_status(uwb_ctx* c);
// SolverError for a status word already on the host (0 = OK).
int status_error(int status);

}  // namespace uwb
