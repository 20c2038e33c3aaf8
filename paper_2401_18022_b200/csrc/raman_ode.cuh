// Device ISRS power-evolution solve: launch interface (raman_ode.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace uwb {

struct OdeParams {
  int n;                 // channels
  const double* alpha;   // [n] 1/m
  const double* M;       // [n*n] coupling premultiplied by launch power, or null (Raman off)
  const int* row_lo;     // [n] first nonzero column of row i
  const int* row_hi;     // [n] one past the last nonzero column
  int steps;             // distance-grid steps (midpoints)
  int col_stride;        // row stride of log2rho / log_rho (>= steps)
  const double* mid;     // [steps]
  double length;
  double rtol, atol;
  double* log2rho;       // [n*steps] out: log2(rho) in the NLI layout
  double* log_rho;       // [n*steps] out: ln(rho) (may be null)
  double* rho_end;       // [n] out
  int* status;           // out: 0 ok, 1 non-positive rho, 2 step budget, 3 step underflow
  long long* rhs_evals;  // out (may be null)
  int rows_per_cta;      // set by launch_raman_ode
  int slab_in_smem;      // set by launch_raman_ode
};

// Builds M (if P.M != null) from the grid/fibre arrays and runs the cluster
// ODE kernel.  Returns kernel launches issued, or < 0 on a launch failure.
int launch_raman_ode(OdeParams P, const double* freq, const double* psd, double bch,
                     const double* aeff, const double* rx, const double* ry, int rn,
                     double aeff_ref, double* M, int* row_lo, int* row_hi, cudaStream_t st);

size_t ode_smem_bytes(int n, int rpc, bool slab);

}  // namespace uwb
