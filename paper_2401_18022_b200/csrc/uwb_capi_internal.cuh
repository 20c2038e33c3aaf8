// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/uwb_nli.h"
#include "nli_kernel.cuh"
#include "uwb_ctx.cuh"

namespace uwb {

int fail(int code, const std::string& msg);

// cudaMemcpy(Async) that accounts host<->device bytes on the context
// (uwb_last_transfer_bytes: the e2e bench reports them per step).
inline cudaError_t xfer(uwb_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                        cudaStream_t st) {
  if (kind == cudaMemcpyHostToDevice) c->h2d_bytes += bytes;
  if (kind == cudaMemcpyDeviceToHost) c->d2h_bytes += bytes;
  return cudaMemcpyAsync(dst, src, bytes, kind, st);
}
inline cudaError_t xfer_sync(uwb_ctx* c, void* dst, const void* src, size_t bytes,
                             cudaMemcpyKind kind) {
  cudaError_t e = xfer(c, dst, src, bytes, kind, c->stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(c->stream);
}
inline void reset_xfer(uwb_ctx* c) { c->h2d_bytes = c->d2h_bytes = 0; }
int cuda_fail(cudaError_t e, const char* what);
int validate_grid(const uwb_grid* g);
int validate_grid_full(const uwb_grid* g);
int set_cfg(const uwb_nli_cfg* cfg, NliParams* P, int precision);
int run_probes(uwb_ctx* c, NliParams& P, const uwb_nli_cfg* cfg, const std::vector<double>& nu,
               const std::vector<double>& gam, const std::vector<int>* chan_probe0,
               bool sync_stats);
void channel_probes(const uwb_grid* g, const double* gamma, const uwb_nli_cfg* cfg,
                    const std::vector<int>& subset, std::vector<double>* nu,
                    std::vector<double>* gam, std::vector<int>* chan_probe0,
                    bool include_dark = false, std::vector<int>* probe_chan = nullptr);
int launch_finalize_channels_only(const FinalizeParams& f, cudaStream_t st);
void release_link_state(uwb_ctx* c);
int distance_grid_host(double length_m, double density, std::vector<double>* edge,
                       std::vector<double>* mid, std::vector<double>* width);

}  // namespace uwb
