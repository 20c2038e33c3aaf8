/*
 * uwb_nli.h — C-ABI of the B200-native ISRS-GN NLI engine (libuwbnli.so).
 *
 * Drop-in boundary for the reference's hot path (uwblink, header-only C++20,
 * /root/reference/proj/include/uwblink).  The reference has no FFI: its
 * "operator API" is the set of inline C++ free functions below, and the C++
 * shim include/uwblink_b200/gn_integral.hpp re-exposes exactly those
 * signatures over this C-ABI.  Each entry point names
 * the reference interface it replaces.
 *
 *   uwb_all_channels_nli   <- uwblink::all_channels_nli   gn_integral.hpp:334-338
 *   uwb_nli_psd_at         <- uwblink::nli_psd_at         gn_integral.hpp:218-222
 *   uwb_channel_nli        <- uwblink::channel_nli        gn_integral.hpp:316-320
 *   uwb_power_evolution    <- uwblink::solve_power_evolution raman_power.hpp:52-55
 *   uwb_evaluate_link      <- uwblink::evaluate_link      link_optimizer.hpp:241-245
 *   uwb_cfm_all_channels_nli <- uwblink::cfm_all_channels_nli gn_closed_form.hpp:70-74
 *                              (= solve_link_noise :181-190 + assemble_link_report :194-237)
 *
 * Conventions
 *  - Plain pointers + sizes, host memory unless a name says _dev.  The caller
 *    owns every host array; the context owns its device buffers, which stay
 *    resident in HBM across calls (the optimisation loop re-uses them).
 *  - Return value: UWB_OK (0) or an error code; uwb_last_error() returns a
 *    thread-local message.  UWB_CONFIG_ERROR / UWB_SOLVER_ERROR map 1:1 to the
 *    reference's uwblink::ConfigError / uwblink::SolverError (units.hpp:16-24),
 *    which the C++ shim rethrows so CLI exit codes 2/3 are preserved
 *    (tools/uwblink_main.cpp:286-296).
 *  - No CPU fallback: without a usable sm_100 device every compute entry point
 *    returns UWB_CUDA_ERROR.
 *  - Results are deterministic and independent of how channels are split over
 *    GPUs (the reference's bit-identity-across-workers contract,
 *    test_gn_integral.cpp:291-300).
 */
#ifndef UWB_NLI_H
#define UWB_NLI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UWB_ABI_VERSION 1

#define UWB_OK 0
#define UWB_ERROR 1
#define UWB_CONFIG_ERROR 2 /* uwblink::ConfigError */
#define UWB_SOLVER_ERROR 3 /* uwblink::SolverError */
#define UWB_CUDA_ERROR 4   /* no device / CUDA failure (no CPU fallback exists) */

typedef struct uwb_ctx uwb_ctx; /* opaque; one per (process, device) */

/* ChannelGrid, channel_grid.hpp:15-22.  psd = launch PSD W/Hz (0 for guards). */
typedef struct {
  int n_ch;
  const double* freq;    /* [n_ch] Hz, ascending, equally spaced */
  const double* psd;     /* [n_ch] W/Hz */
  const uint8_t* guard;  /* [n_ch] 1 = guard slot */
  double spacing;        /* Hz */
  double bch;            /* Hz */
  double centre;         /* Hz */
  double half_band;      /* Hz */
} uwb_grid;

/* One span: PowerEvolution (raman_power.hpp:19-37) + its DistanceGrid
 * (distance_grid.hpp:13-20).  log_rho keeps the reference layout ch*steps+m. */
typedef struct {
  int steps;                /* N_M = number of distance steps */
  const double* log_rho;    /* [n_ch * steps] */
  const double* edge;       /* [steps + 1] m */
  const double* mid;        /* [steps] m */
  const double* width;      /* [steps] m */
  double length;            /* m */
} uwb_span;

/* GnSolverConfig, gn_integral.hpp:19-28 (workers has no meaning here). */
typedef struct {
  int n_r;
  int u1_uniform;           /* 0 = U1Sampling::kLog (default), 1 = kUniform */
  double u1_min_ratio;
  int simpson;              /* simpson_channel_average */
  int mirror_q4;
} uwb_nli_cfg;

/* NliResult, gn_integral.hpp:30-37.  Any output pointer may be NULL. */
typedef struct {
  double* eta;              /* [n_ch] 1/W^2 */
  double* nli_psd;          /* [n_ch] W/Hz */
  double* nli_power;        /* [n_ch] W */
  double* quadrant;         /* [n_ch * 4] */
  uint8_t* skipped;         /* [n_ch] */
  double elapsed_seconds;   /* device time of the sweep (CUDA events) */
} uwb_nli_result;

/* Fibre quantities the full evaluation needs, sampled by the caller at the
 * grid frequencies with the reference's own fibre model
 * (attenuation_at / aeff_at / gamma_at fibre_model.hpp:256-267, Raman curve
 * :213-227, beta_from_dispersion at lambda(centre) :76-89). */
typedef struct {
  const double* alpha;      /* [n_ch] power attenuation 1/m */
  const double* aeff;       /* [n_ch] m^2 */
  const double* gamma;      /* [n_ch] 1/(W m) */
  int raman_n;              /* Raman gain table rows */
  const double* raman_x;    /* [raman_n] Hz, ascending */
  const double* raman_y;    /* [raman_n] 1/(W m) */
  double raman_aeff_ref;    /* m^2 */
  double beta[3];           /* beta2, beta3, beta4 */
  double length_m;
  int span_count;
} uwb_fibre;

/* LinkConfig pieces used by assemble_link_report (link_optimizer.hpp:159-171). */
typedef struct {
  int include_raman;        /* RamanSolveOptions::include_raman */
  double rtol, atol;        /* RamanSolveOptions rtol/atol (1e-9 / 1e-16) */
  double density;           /* GnSolverConfig::mean_step_density, steps/km */
  const double* nf_db;      /* [n_ch] amplifier NF of each channel's band (BandPlan), 5 dB if none */
  const int* band;          /* [n_ch] band index (BandPlan::band_of_lambda) or -1; may be NULL */
  int n_bands;              /* number of bands (per-band report sums) */
  int use_snr_trx;
  double snr_trx_db;
} uwb_link_cfg;

/* LinkReport, link_optimizer.hpp:139-157 (per-channel arrays; NULL allowed). */
typedef struct {
  double* eta;
  double* p_ase;
  double* snr_db;
  double* capacity;
  double* rho_end;
  double* band_power_dbm;   /* [n_bands] */
  double* band_capacity;    /* [n_bands] */
  double loss_value;
  double total_capacity;
  double total_power_dbm;
  double elapsed_seconds;   /* device time: ODE + NLI + assembly */
  double ode_seconds;
} uwb_link_report;

const char* uwb_last_error(void);
int uwb_abi_version(void);

/* Visible CUDA devices (the multi-GPU optimiser gives each one a context). */
int uwb_device_count(int* n);

/* Context: binds one CUDA device (0-based index within CUDA_VISIBLE_DEVICES). */
int uwb_ctx_create(int device, uwb_ctx** out);
void uwb_ctx_destroy(uwb_ctx* ctx);

/* Multi-GPU context = the reference's worker pool (GnSolverConfig::workers,
 * all_channels_nli's parallel_for_batches, gn_integral.hpp:348 ->
 * parallel.hpp:21-47) with GPUs as the workers.  devices[0..n_devices) are
 * CUDA device indices (repeats allowed, e.g. several contexts on one GPU);
 * devices[0] leads.  Every entry point accepts the returned context:
 *  - uwb_all_channels_nli, uwb_evaluate_link, uwb_evaluate_link_prepare /
 *    _resident split the channels into contiguous ranges balanced by the
 *    per-channel work the previous NLI measured; each GPU runs the Raman ODE
 *    and its range's NLI; eta slices are gathered on the lead
 *    (cudaMemcpyPeerAsync over NVLink), which assembles the report.
 *    _resident's psd_dev / report_dev / stream live on the lead device;
 *  - uwb_evaluate_link_many deals whole evaluations to the GPUs;
 *  - nli_psd_at, channel_nli, power_evolution and the closed form run on the
 *    lead;
 *  - uwb_set_channel_subset and the split _resident_noise / _report /
 *    uwb_link_eta_buffer stages are single-device: ConfigError.
 * Results are bit-identical to one device for any device list. */
int uwb_ctx_create_multi(const int* devices, int n_devices, uwb_ctx** out);
/* Devices behind a context (1 for uwb_ctx_create). */
int uwb_ctx_width(uwb_ctx* ctx, int* n);
/* |K|^2 evaluations per channel of the last NLI ([n_ch]; the multi-GPU
 * split's cost model, measured on the device). */
int uwb_last_channel_work(uwb_ctx* ctx, int n_ch, double* work);
/* Per device of the last split evaluation: integrand and ODE device time
 * (ms) and the first channel of its range ([n] each, any may be NULL). */
int uwb_last_partition_stats(uwb_ctx* ctx, int n, double* nli_ms, double* ode_ms, int* first_ch);
int uwb_device_info(uwb_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);

/* Restrict all_channels_nli / evaluate_link to a subset of channels (multi-GPU
 * partition; the others report skipped=1 and zeros).  n = 0 clears it. */
int uwb_set_channel_subset(uwb_ctx* ctx, int n, const int* channels);

/* all_channels_nli (gn_integral.hpp:334-363): gamma[n_ch] = gamma_at per
 * channel (:353).  Spans must share one step count.  Like the reference, the
 * NLI entry points do not run ChannelGrid::validate (the reference never
 * calls it on this path); they reject only what would make the device's index
 * arithmetic undefined.  uwb_power_evolution / uwb_evaluate_link /
 * uwb_evaluate_link_prepare run the full ChannelGrid::validate
 * (channel_grid.hpp:44-61) as solve_power_evolution does (raman_power.hpp:56). */
int uwb_all_channels_nli(uwb_ctx* ctx, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                         const double beta[3], const double* gamma, const uwb_nli_cfg* cfg,
                         uwb_nli_result* out);

/* cfm_all_channels_nli (gn_closed_form.hpp:70-144): the closed-form SPM +
 * XPM model over the same inputs (gamma[n_ch] = gamma_at per channel, :84-87;
 * spans may differ in step count).  quadrant (if non-NULL) is zeroed like
 * the reference's; elapsed_seconds is device time. */
int uwb_cfm_all_channels_nli(uwb_ctx* ctx, const uwb_grid* grid, int n_spans,
                             const uwb_span* spans, const double beta[3], const double* gamma,
                             uwb_nli_result* out);

/* nli_psd_at (gn_integral.hpp:218-313) for n_probe absolute probe frequencies
 * with per-probe gamma; quadrant4 [n_probe*4] may be NULL. */
int uwb_nli_psd_at(uwb_ctx* ctx, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                   const double beta[3], const uwb_nli_cfg* cfg, int n_probe, const double* nu,
                   const double* gamma, double* out, double* quadrant4);

/* channel_nli (gn_integral.hpp:316-329) for one channel index. */
int uwb_channel_nli(uwb_ctx* ctx, const uwb_grid* grid, int n_spans, const uwb_span* spans,
                    const double beta[3], double gamma_ch, const uwb_nli_cfg* cfg, int ch,
                    double* out, double* quadrant4);

/* solve_power_evolution (raman_power.hpp:52-122) on the device: fills
 * log_rho [n_ch*steps] and rho_end [n_ch] for the given distance grid. */
int uwb_power_evolution(uwb_ctx* ctx, const uwb_grid* grid, const uwb_fibre* fibre,
                        const uwb_link_cfg* link, int steps, const double* mid,
                        double* log_rho, double* rho_end);

/* Full SNR evaluation = evaluate_link (link_optimizer.hpp:241-245): distance
 * grid + device Raman ODE + device NLI + device assemble_link_report.  The
 * grid's psd carries the launch powers.  Host in, host out. */
int uwb_evaluate_link(uwb_ctx* ctx, const uwb_grid* grid, const uwb_fibre* fibre,
                      const uwb_link_cfg* link, const uwb_nli_cfg* cfg, uwb_link_report* out);

/* Device-resident variant used by the optimisation loop and the bench
 * `value` leg: static state (grid layout, fibre, configs) is uploaded by
 * uwb_evaluate_link_prepare once; each uwb_evaluate_link_resident call takes
 * launch powers already in device memory (psd_dev [n_ch], W/Hz) and leaves the
 * report in device memory.  stream: cudaStream_t or NULL for the context's.
 * Calls on one context share its device buffers: issue them on one stream (or
 * order them with events); the context joins its own side stream internally.
 *
 * Report layout (report_dev here, and each row of uwb_evaluate_link_many's
 * report_host), report_len = 4*n_ch + 3 + 2*n_bands doubles:
 *   [0, n_ch)               eta      1/W^2 (0 for skipped channels)
 *   [n_ch, 2 n_ch)          p_ase    W
 *   [2 n_ch, 3 n_ch)        snr_db
 *   [3 n_ch, 4 n_ch)        capacity b/s
 *   [4 n_ch + 0..2]         loss_value, total_capacity, total_power_dbm
 *   [4 n_ch + 3, +n_bands)  band_power_dbm
 *   [.. + n_bands, +n_bands) band_capacity
 * (n_bands = uwb_link_cfg::n_bands of the prepare call; uwb_report_len
 * returns report_len.)
 *
 * The skip set is re-derived from each call's launch profile, like the
 * reference (guard or psd <= 0, gn_integral.hpp:349-352): a channel that was
 * dark at prepare time and is lit in a later call gets its NLI.
 *
 * Memory: single evaluations (uwb_evaluate_link, _resident) run the rows'
 * point setup beside the Raman ODE and keep one 96-byte record slot per
 * (row, column) in HBM, allocated by the first such call on a prepared link:
 * 4 * n_r^2 * 96 bytes per probe (5.1 GB for 589 channels at N_R = 150).
 * Lists over UWB_NLI_SPLIT_MB (default 8192) or a failed allocation fall back
 * to the fused integrand kernel (same results, bit for bit). */
int uwb_evaluate_link_prepare(uwb_ctx* ctx, const uwb_grid* grid, const uwb_fibre* fibre,
                              const uwb_link_cfg* link, const uwb_nli_cfg* cfg);
int uwb_evaluate_link_resident(uwb_ctx* ctx, const double* psd_dev, double* report_dev,
                               void* stream);
/* Doubles per report of the prepared link (see the layout above). */
int uwb_report_len(uwb_ctx* ctx, int* len);
/* n_eval full evaluations of the prepared link back to back on the device
 * (optimise_launch_powers' value + forward-difference gradient calls,
 * link_optimizer.hpp:294-309): psd_host [n_eval][n_ch] launch PSDs (W/Hz) in,
 * loss_host [n_eval] (may be NULL) and report_host [n_eval][report_len] (may
 * be NULL; layout of uwb_evaluate_link_resident) out.  One upload, one
 * download, one synchronisation per batch; the first SolverError of the
 * batch is reported. */
int uwb_evaluate_link_many(uwb_ctx* ctx, int n_eval, const double* psd_host, double* loss_host,
                           double* report_host);
/* Split resident evaluation for multi-GPU runs: the noise stage (Raman ODE +
 * NLI of this context's channel subset) leaves eta in the buffer returned by
 * uwb_link_eta_buffer (zeros outside the subset); the caller all-reduces it
 * across ranks (NCCL), then the report stage assembles SNR from the full eta.
 * uwb_resident_status synchronises and maps the ODE status to SolverError. */
int uwb_evaluate_link_resident_noise(uwb_ctx* ctx, const double* psd_dev, void* stream);
int uwb_evaluate_link_resident_report(uwb_ctx* ctx, double* report_dev, void* stream);
int uwb_link_eta_buffer(uwb_ctx* ctx, double** eta_dev, int* n_ch);
int uwb_resident_status(uwb_ctx* ctx);
/* Active points of the last NLI (every point of the reference's enumeration
 * with three non-zero PSDs); evaluated_points of uwb_last_nli_stats counts
 * the |K|^2 evaluations actually run (symmetric rows share mirrored ones).
 * Call after uwb_last_nli_stats. */
int uwb_last_nli_active(uwb_ctx* ctx, double* active_points);
/* Device time (ms) of the last evaluation's Raman ODE stage and its number
 * of RHS evaluations (prepared/resident path; synchronises). */
int uwb_last_ode_stats(uwb_ctx* ctx, double* ode_ms, long long* rhs_evals);
/* Host<->device bytes moved by the last public call. */
int uwb_last_transfer_bytes(uwb_ctx* ctx, unsigned long long* h2d, unsigned long long* d2h);
/* Bounds-checked builds (-DUWB_BOUNDS_CHECK=1): first source line of the
 * integrand / ODE whose index check failed (0 = none), -1 in normal builds. */
int uwb_debug_bounds(int* nli_line, int* ode_line);
/* Live FP64 FMA-pipe peak of this device, TFLOP/s (roofline denominator). */
int uwb_fp64_peak(uwb_ctx* ctx, double* tflops);
/* Step arithmetic of the NLI integrand for subsequent calls (and for
 * subsequent uwb_evaluate_link_prepare; a prepared link keeps its mode).
 * UWB_PRECISION_FP64 (default): every operation in FP64, the reference's
 * arithmetic.  UWB_PRECISION_MIXED: compensated FP32 -- the log2-rho
 * interpolation, the phase and its reduction, and all sums past a lane stay
 * FP64; 2^x, sin/cos and the lane's partial sums of reduced, well-conditioned
 * arguments run in FP32 (BASELINE config 4, "FP64 vs compensated FP32";
 * accuracy per setting in profiles/r01_config4_sweep.json).  This is an
 * extension: the reference has no precision knob. */
#define UWB_PRECISION_FP64 0
#define UWB_PRECISION_MIXED 1
int uwb_set_precision(uwb_ctx* ctx, int mode);
/* Step-size policy of the device Raman ODE for subsequent calls/prepares.
 * UWB_ODE_RESTART (default): the reference's -- Rk45::integrate restarts at
 * every distance-grid midpoint with h0 = (z1 - z0)/100 (raman_power.hpp:107-
 * 118, rk45.hpp:33).  UWB_ODE_CONTINUOUS: the same Dormand-Prince controller and
 * tolerances, landing exactly on every midpoint, but the step size carries
 * across midpoints instead of restarting (about 3x fewer RHS evaluations).
 * An extension: results differ from the reference by the ODE's own truncation
 * error. */
#define UWB_ODE_RESTART 0
#define UWB_ODE_CONTINUOUS 1
int uwb_set_ode_stepping(uwb_ctx* ctx, int mode);
/* Kernel launches issued by the last call (evidence for bench gpu_launches). */
int uwb_last_launch_count(uwb_ctx* ctx);
/* Device time (ms) of the last NLI integrand kernel and its inner-step count
 * (evaluated points x distance steps x spans) — the roofline inputs. */
int uwb_last_nli_stats(uwb_ctx* ctx, double* kernel_ms, double* inner_steps,
                       double* evaluated_points);

#ifdef __cplusplus
}
#endif
#endif /* UWB_NLI_H */
