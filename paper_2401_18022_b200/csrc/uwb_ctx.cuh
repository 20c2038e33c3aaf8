// Context object behind the C-ABI: device, stream, and the HBM-resident
// buffers that persist across calls.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "nli_kernel.cuh"

namespace uwb {

// Grow-only device allocation.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    const size_t bytes = n * sizeof(T) + 16;
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
  template <class T>
  T* ptr() const {
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct Error {
  int code;
  std::string msg;
};

}  // namespace uwb

struct uwb_ctx {
  int device = 0;
  int sm_count = 0;
  int precision = 0;  // UWB_PRECISION_FP64 / _MIXED (uwb_set_precision)
  int ode_continuous = 0;  // UWB_ODE_RESTART / _CONTINUOUS (uwb_set_ode_stepping)
  int cc_major = 0, cc_minor = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evk0 = nullptr, evk1 = nullptr;
  // channel grid
  uwb::DBuf freq, psd, gamma;
  // spans
  uwb::DBuf log2rho, zedge, zstart, zmid, width, wlast, span_steps;
  // probes + work
  uwb::DBuf probe_work;  // per-probe |K|^2 evaluations of the last NLI
  uwb::DBuf rowcnt;      // per-row work counts (summed per probe by the finalize)
  uwb::DBuf probe_nu, probe_chan, probe_gamma, hl2, rowsum, rowpar, counter, n_eval, probe_g, probe_quad,
      chan_probe0;
  // per-channel results
  uwb::DBuf eta, nli_psd, nli_power, quad, skipped;
  // uwb_evaluate_link_many: the batch's launch profiles and reports
  uwb::DBuf batch_psd, batch_report, batch_ode;
  // closed-form model (uwb_cfm.cu)
  uwb::DBuf cfm_in, cfm_work, cfm_span;
  struct BatchState {  // overlapped uwb_evaluate_link_many (second ODE stream)
    cudaStream_t s_ode = nullptr;
    cudaEvent_t ev_start = nullptr, ev_ode[2] = {nullptr, nullptr}, ev_nli[2] = {nullptr, nullptr};
  };
  BatchState* batch = nullptr;
  // split evaluation (launch_nli_setup beside the Raman ODE): per-row point
  // records and counts, the setup pass's stream and its fork/join events
  uwb::DBuf plist, plist_n;
  cudaStream_t s_setup = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_lists = nullptr;  // the last list pass is done with the point lists
  // link evaluation state (raman ODE + assembly)
  uwb::DBuf alpha, aeff, raman_x, raman_y, nf_db, guard, rho_end, ode_work, ode_gwork, report, mid, edge;
  std::vector<int> subset;
  // stats of the last call
  unsigned long long h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic of the last call
  int last_launches = 0;
  bool nli_events_valid = false;
  double last_total_steps = 0.0;  // distance steps summed over the spans of the last NLI
  double last_kernel_ms = 0.0;
  double last_inner_steps = 0.0;
  double last_points = 0.0;
  double last_active = 0.0;  // active (reference-enumerated) points of the last NLI
  // pinned host staging for small transfers
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  // deferred uploads (evaluate_link prepare): the host arrays are packed into
  // one staging block, copied with ONE host-to-device transfer and scattered to
  // their buffers by one kernel, instead of ~20 pageable cudaMemcpyAsync calls
  struct UpSeg {
    void* dst;
    size_t off, bytes;
  };
  bool up_defer = false;
  std::vector<unsigned char> up_host;
  std::vector<UpSeg> up_segs;
  void* up_pinned = nullptr;
  size_t up_pinned_cap = 0;
  uwb::DBuf up_dev;
  // probes of the last NLI: first probe of each channel (-1: none) and
  // probes per channel (3 with Simpson), for uwb_last_channel_work
  std::vector<int> last_chan_probe0;
  int last_probes_per_chan = 1;
  int last_n_probes = 0;
  // prepared link problem (uwb_evaluate_link_prepare)
  struct Prepared;
  Prepared* prep = nullptr;
  // Multi-device context (uwb_ctx_create_multi): the reference's channel-
  // parallel worker pool (parallel_for_batches, parallel.hpp:21-47) as a
  // partition of the channels over GPUs.  subs[0] is the lead.
  std::vector<uwb_ctx*> subs;   // channel-split evaluation, one per device entry
  std::vector<uwb_ctx*> bsubs;  // whole evaluations of a batch (uwb_evaluate_link_many)
  std::vector<double> chan_cost;  // per-channel work of the last NLI (balances the next split)
  std::vector<int> part_lo;       // channel ranges [part_lo[d], part_lo[d+1]) of the last split
  cudaEvent_t ev_done = nullptr;  // this context's noise stage is complete (multi gather)
  bool multi() const { return !subs.empty(); }
};
