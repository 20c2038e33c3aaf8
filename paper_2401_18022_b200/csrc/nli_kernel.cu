// ISRS-GN numerical-integral NLI kernels for sm_100a (FP64).
//
// Reference algorithm: nli_psd_at / kernel_abs2 (gn_integral.hpp:136-313).
// The hyperbolic-coordinate Riemann sum is generated from indices on the
// device; nothing about the (u1, u2) grid is materialised in HBM.
//
// Work decomposition:
//   unit  = one u1-row (probe, quadrant q, row i); a persistent grid of warps
//           pulls rows from an atomic queue.
//   warp  = one row.  Lanes first evaluate the per-point setup for 32 u2
//           columns at a time (coordinates, 3x psd_at, 3 stencils, phi,
//           gn_integral.hpp:288-303), then the two 16-lane half-warps each take
//           one evaluated point and split its distance steps across lanes
//           (step m = lane + 16 k), so the table loads are coalesced, the
//           fast/slow branch (gn_integral.hpp:156) is uniform per half-warp,
//           and every lane does exp2 + sincos per step.
//   reduce= fixed-order xor-shuffle tree per point, points summed into the row
//           in ascending j (reference order), rows Kahan-summed in ascending i
//           by the finalize kernel (gn_integral.hpp:258,306) -> deterministic,
//           independent of grid size, CTA scheduling and GPU partitioning.
//
// Fast branch uses summation by parts of the reference's phasor-difference
// sum:  sum_m p_m (E_{m+1} - E_m) = -p_0 E_0 + sum_{e>=1} (p_{e-1} - p_e) E_e
// (p_N = 0), so each step needs ONE sincos (at its end edge) and one shuffle.
//
// This file is compiled with -fmad=false: all setup arithmetic rounds exactly
// like the reference (no contraction); the hot loop uses explicit fma().
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "nli_kernel.cuh"
#include "uwb_devmath.cuh"

namespace uwb {

namespace {

// Bounds-checked build (-DUWB_BOUNDS_CHECK=1, tools/build_variant.py): every
// table, record and row index the integrand forms is checked against its
// allocation; the first failing source line is kept for uwb_debug_bounds.
// (compute-sanitizer is not available on the GPU pool; this is its stand-in.)
#if UWB_BOUNDS_CHECK
__device__ int g_nli_bounds_fail;
#define UWB_BOUND(cond)                                          \
  do {                                                           \
    if (!(cond)) atomicCAS(&g_nli_bounds_fail, 0, __LINE__);     \
  } while (0)
#else
#define UWB_BOUND(cond) \
  do {                  \
  } while (0)
#endif

#ifndef UWB_Z_SMEM
#define UWB_Z_SMEM 1  // HOIST: z edges from shared memory (broadcast LDS) instead of registers
#endif
#ifndef UWB_NLI_WARPS
#define UWB_NLI_WARPS 8  // hoisted FP64 kernels (8-lane segments): x 2 CTAs, 128 registers
#endif                   // (8.48 ms on the bench workload; 10 x 2 at 96 registers: 8.52)
#ifndef UWB_NLI_WARPS_OTHER
#define UWB_NLI_WARPS_OTHER 8  // per-step-load (multi-span / long-span) and mixed kernels
#endif
#ifndef UWB_NLI_MIN_BLOCKS
#define UWB_NLI_MIN_BLOCKS 2
#endif
#ifndef UWB_NLI_MIXED_MIN_BLOCKS
#define UWB_NLI_MIXED_MIN_BLOCKS 3  // 80 registers: 6 warps per SMSP (10.9 -> 10.0 ms)
#endif
// warps per CTA of each integrand instantiation
template <bool HOIST, bool MIXED>
struct WarpsFor {
  static constexpr int value = (HOIST && !MIXED) ? UWB_NLI_WARPS : UWB_NLI_WARPS_OTHER;
};
constexpr unsigned kFull = 0xffffffffu;

__constant__ double c_exp2_tab16[16] = UWB_EXP2_TABLE16;

// ChannelGrid::psd_at (channel_grid.hpp:35-42) fused with stencil_for
// (gn_integral.hpp:110-129): both start from the same `pos`.
struct Stencil {
  int i0, i1;
  double hw0, hw1;
};

__device__ __forceinline__ Stencil psd_and_stencil(const NliParams& P, double nu, double* psd) {
  // the reference divides; a reciprocal multiply moves pos by <= 1 ulp, which
  // only nudges the (continuous) interpolation weight -- the PSD window test
  // below uses nu - freq[i] itself
  const double pos = (nu - P.freq[0]) * P.inv_spacing;
  const long i = lround(pos);
  double v = 0.0;
  if (i >= 0 && i < P.n_ch) {
    if (!(fabs(nu - __ldg(P.freq + i)) > 0.5 * P.bch)) v = __ldg(P.psd + i);
  }
  *psd = v;
  const int n = P.n_ch;
  // stencil_for: clamp below (pos <= 0) / above (pos >= n-1), else linear
  const bool below = n == 1 || pos <= 0.0;
  const bool above = !below && pos >= static_cast<double>(n - 1);
  const int k = (below || above) ? 0 : static_cast<int>(pos);  // truncation == size_t cast
  const double t = pos - static_cast<double>(k);
  Stencil s;
  s.i0 = below ? 0 : (above ? n - 1 : k);
  s.i1 = below ? 0 : (above ? n - 1 : k + 1);
  s.hw0 = (below || above) ? 0.5 : 0.5 * (1.0 - t);
  s.hw1 = (below || above) ? 0.0 : 0.5 * t;
  return s;
}

// phase_mismatch (gn_integral.hpp:43-50), same grouping; -fmad=false keeps
// every product/sum separately rounded like the reference.
__device__ __forceinline__ double phase_mismatch(double f1, double f2, double fi, double b2,
                                                 double b3, double b4) {
  const double quartic =
      (f1 * f1 + f2 * f2) + 1.5 * (f1 * f2) + 3.0 * fi * (f1 + f2) + 3.0 * (fi * fi);
  const double bracket = b2 + kPi * b3 * ((f1 + f2) + 2.0 * fi) +
                         (2.0 * kPi * kPi / 3.0) * b4 * quartic;
  return -4.0 * kPi * kPi * (f1 * f2) * bracket;
}

// Per-warp shared state for one chunk of 32 u2 columns, plus the row's
// parameters (parked here so they are not live in registers across the
// integrand loop).
// One listed point, packed so a 16-lane segment reads it with five broadcast
// 128-bit loads.
struct alignas(16) PointRec {
  double w[6];         // 16 x half weights for columns i0 and i0 + 1 of nu1, nu2, nu3
  double phi8, rphi8;  // phi 8/pi (the fast branch's phase in units of pi/8) and 1/phi8
                       // (0 when phi == 0: no fast span then)
  int col[3];          // element offset (i0 * NS) of each stencil's first column
  int src;             // chunk-local column of the listed point (point_kernel8 path: 1 = fast)
  double phi;          // phase mismatch itself (sinc branch, fast/slow test of later spans)
  double pws;          // point_kernel8 path: p1 p2 p3 of the column plus that of the mirror
                       // column sharing its |K|^2 (0 when none)
};

#ifndef UWB_SEG8
#define UWB_SEG8 1  // hoisted FP64 kernels: 8-lane segments over 2K steps (point_kernel8)
#endif
#if UWB_SEG8 && !UWB_Z_SMEM
#error "UWB_SEG8 reads the z edges from shared memory (UWB_Z_SMEM)"
#endif
struct WarpSmem {
  PointRec pt[36];   // a chunk's listed points, plus up to 3 carried over (point_kernel8 path)
  double kv[32];     // |kernel|^2 of each chunk lane's evaluated point
#if UWB_SEG8
  alignas(16) double h[128];  // the row's probe half-log column (point_kernel8), lane order
#endif
  double nu, f, s1, s2, su, u1, lo, du2;
  int sym;           // row symmetric under u2 -> -u2 (b1 == b2: quadrants 1, 3)
};

// Polynomial coefficients as __constant__ data: ptxas keeps them in uniform
// registers (DFMA R, R, UR, R) instead of re-materialising 64-bit immediates
// with UMOV/IMAD.MOV pairs every step, which cost v1 ~70 issue slots per step.
__constant__ double c_e4[6] = {kE4c1, kE4c2, kE4c3, kE4c4, kE4c5, kE4c6};
#ifndef UWB_FAST_POLY
#define UWB_FAST_POLY 2
#endif
// Step kernels for 2^(r/16), sin and cos on the reduced ranges, shorter than
// the ulp-accurate ones (Chebyshev fits): 2^x degree 4 (max relative error
// 5e-12), sin degree 7 (3.7e-14 absolute), cos degree 6 (1.7e-12 absolute).
// They only enter the per-step phasor sums, not a discrete decision, so the
// row setup keeps the full-accuracy dev_exp2_16 (its coordinates decide the
// active set).  UWB_FAST_POLY selects the sinc branch's dev_sincos kernels
// (2: these fits, 1: cos degree 8, 0: ulp-accurate); the fast branch always
// runs step_exp2_16t / step_sincos8.  eta vs the reference: 3.2e-12 on the
// 589-ch golden, <= 6.2e-13 on the 11-channel goldens (tests: 1e-9).
// The coefficients live in uwb_devmath.cuh (kStep*), where
// tests/test_devmath.py checks them on the host.
__constant__ double c_s3f[3] = {kStepS0, kStepS1, kStepS2};
__constant__ double c_c4f[4] = {-0.4999999999999954, 0.0416666666627131, -0.0013888883764931453,
                                2.478033379585741e-05};
__constant__ double c_e4f[4] = {kStepE0, kStepE1, kStepE2, kStepE3};
__constant__ double c_c3f[3] = {kStepC0, kStepC1, kStepC2};

// 2^(j/16) for dev_exp2_16, filled by each CTA at start.  A file-scope
// __shared__ array (not a generic pointer) so the lookup is one LDS.
__shared__ double s_exp2_tab[16];

// 2^(x/16), x = 16 log2 p (uwb_devmath.cuh exp2_16): 3 DADD + 6 DFMA + 1 DMUL,
// one conflict-free LDS.
__device__ __forceinline__ double dev_exp2_16(double x) {
  const double t = x + kMagic;
  const int k = __double2loint(t);
  const double r = x - (t - kMagic);
  double p = fma(r, c_e4[5], c_e4[4]);
  p = fma(p, r, c_e4[3]);
  p = fma(p, r, c_e4[2]);
  p = fma(p, r, c_e4[1]);
  p = fma(p, r, c_e4[0]);
  p = fma(p, r, 1.0);
  const double s = s_exp2_tab[k & 15] * p;
  return __hiloint2double(__double2hiint(s) + ((k >> 4) << 20), __double2loint(s));
}

// (cos x, sin x) for |x| < 2^50 by a 16-entry full-circle table: x = k pi/8
// + r, |r| <= pi/16, cos/sin(k pi/8) from two 128-byte shared tables (one
// line each: conflict-free for any lane pattern), minimax kernels on r
// (sin: r + r^3 S(r^2), deg 3, |err| 3.3e-18; cos: 1 + r^2 C(r^2), deg 4,
// |err| 1.3e-20; Chebyshev fits in 50-digit arithmetic), then the angle
// addition.  19 FP64 instructions and no quadrant selects / sign fix-ups.
__constant__ double c_red8[3] = {kEightOverPi, -kPio8Hi, -kPio8Lo};
__constant__ double c_s16[4] = {kS16c1, kS16c2, kS16c3, kS16c4};
__constant__ double c_c16[5] = {kC16c0, kC16c1, kC16c2, kC16c3, kC16c4};
__constant__ double c_tab_cos16[16] = UWB_COS_TABLE16;
__constant__ double c_tab_sin16[16] = UWB_SIN_TABLE16;
// (cos, sin)(k pi/8) interleaved: one 128-bit LDS per lookup (the 256-byte
// table costs at most a 2-way conflict, q vs q + 8, i.e. the same wavefronts
// as two 64-bit lookups in two 128-byte tables, with one instruction fewer
// and no second base address)
__shared__ double2 s_cs16[16];

// The hot loop's shared tables (kernel scope, passed by reference):
//   cs16[q]: (cos, sin)(q pi/8)
//   e2c[j]:  2^(j/16) with j << 16 subtracted from its high word, so that adding
//            k << 16 (k = 16 e + j) to it yields 2^(k/16) exactly: the exponent
//            insertion is one shift-add (LEA) instead of shift, mask and add.
// Each table is its own kernel-scope __shared__ array (StepTabs holds their
// addresses), so a lookup is [index + uniform base] with no per-lookup base add.
struct StepTabs {
  double2* cs16;  // [16]
  double* e2c;    // [16]
  double* z;      // [128] the span's end-edge positions (HOIST, K <= 8), lane order
};

// nli_list_kernel's per-warp records: a chunk of kListChunk listed points
// plus up to 3 carried over, and the probe half-log column (no per-lane |K|^2
// or row fields: the fused kernel's WarpSmem is ~40 % larger, and what the
// list kernel does not hold in shared memory the carveout leaves to L1)
#ifndef UWB_LIST_CHUNK
#define UWB_LIST_CHUNK 16
#endif
constexpr int kListChunk = UWB_LIST_CHUNK;
struct ListWarpSmem {
  PointRec pt[kListChunk + 4];
  alignas(16) double h[128];
};
__device__ __forceinline__ double* S_h(ListWarpSmem& S) { return S.h; }
// the fused kernel's records on the point_kernel8 path (WarpSmem without kv)
struct WarpSmemCarry {
  PointRec pt[36];
  alignas(16) double h[128];
  double nu, f, s1, s2, su, u1, lo, du2;
  int sym;
};
__device__ __forceinline__ double* S_h(WarpSmemCarry& S) { return S.h; }

__device__ __forceinline__ double* S_h(WarpSmem& S) {
#if UWB_SEG8
  return S.h;
#else
  return nullptr;  // not reached
#endif
}

template <class T>
__device__ __forceinline__ double TB_z(const T& tb, int i) {
#if UWB_Z_SMEM
  return tb.z[i];
#else
  return 0.0;
#endif
}

__device__ __forceinline__ void init_step_tabs(const StepTabs& T, int i) {
  if (i < 16) {
    T.cs16[i] = make_double2(c_tab_cos16[i], c_tab_sin16[i]);
    const double v = c_exp2_tab16[i];
    T.e2c[i] = __hiloint2double(__double2hiint(v) - (i << 16), __double2loint(v));
  }
}

// 2^(x/16) (uwb_devmath.cuh step_exp2_16; the same value bit for bit: the
// power-of-two scale is applied to the table entry before the product)
#ifndef UWB_EXP2_NOTAB
#define UWB_EXP2_NOTAB 0
#endif
#if UWB_EXP2_NOTAB
// table-free variant (A/B): 2^(x/16) = 2^n 2^f, f in [-1/2, 1/2], degree-8
// fit (relative error 1.1e-12), 2^n inserted into the exponent field
__constant__ double c_e8[9] = {1.0, 0.6931471805465779, 0.24022650699046685,
                               0.055504109391347665, 0.009618128509058098,
                               0.0013333452228655083, 0.00015403873617090126,
                               1.5309699242759908e-05, 1.3171450610841097e-06};
#endif
__device__ __forceinline__ double step_exp2_16t(double x, const StepTabs& T) {
#if UWB_EXP2_NOTAB
  const double t = fma(x, 0.0625, kMagic);
  const int n = __double2loint(t);
  const double f = fma(x, 0.0625, -(t - kMagic));
  double q = fma(f, c_e8[8], c_e8[7]);
  q = fma(q, f, c_e8[6]);
  q = fma(q, f, c_e8[5]);
  q = fma(q, f, c_e8[4]);
  q = fma(q, f, c_e8[3]);
  q = fma(q, f, c_e8[2]);
  q = fma(q, f, c_e8[1]);
  q = fma(q, f, 1.0);
  return __hiloint2double(__double2hiint(q) + (n << 20), __double2loint(q));
#else
  const double t = x + kMagic;
  const int k = __double2loint(t);
  const double r = x - (t - kMagic);
  double p = fma(r, c_e4f[3], c_e4f[2]);
  p = fma(p, r, c_e4f[1]);
  p = fma(p, r, c_e4f[0]);
  p = fma(p, r, 1.0);
  const double v = T.e2c[k & 15];
  return __hiloint2double(__double2hiint(v) + (k << 16), __double2loint(v)) * p;
#endif
}


__device__ __forceinline__ void dev_sincos_table(double x, double* c_out, double* s_out) {
  const double t = fma(x, c_red8[0], kMagic);
  const int q = __double2loint(t) & 15;
  const double kd = t - kMagic;
  double r = fma(kd, c_red8[1], x);
  r = fma(kd, c_red8[2], r);
  const double z = r * r;
  double sr, cr;
  if (UWB_FAST_POLY) {
    double ps = fma(z, c_s3f[2], c_s3f[1]);
    ps = fma(ps, z, c_s3f[0]);
    sr = fma(r * z, ps, r);
#if UWB_FAST_POLY >= 2
    double pc = fma(z, c_c3f[2], c_c3f[1]);
    pc = fma(pc, z, c_c3f[0]);
#else
    double pc = fma(z, c_c4f[3], c_c4f[2]);
    pc = fma(pc, z, c_c4f[1]);
    pc = fma(pc, z, c_c4f[0]);
#endif
    cr = fma(pc, z, 1.0);
  } else {
    double ps = fma(z, c_s16[3], c_s16[2]);
    ps = fma(ps, z, c_s16[1]);
    ps = fma(ps, z, c_s16[0]);
    sr = fma(r * z, ps, r);
    double pc = fma(z, c_c16[4], c_c16[3]);
    pc = fma(pc, z, c_c16[2]);
    pc = fma(pc, z, c_c16[1]);
    pc = fma(pc, z, c_c16[0]);
    cr = fma(pc, z, 1.0);
  }
  const double2 cs = s_cs16[q];
  const double tc = cs.x, ts = cs.y;
  *c_out = fma(tc, cr, -(ts * sr));
  *s_out = fma(ts, cr, tc * sr);
}

__device__ __forceinline__ void dev_sincos(double x, double* c_out, double* s_out) {
  dev_sincos_table(x, c_out, s_out);
}

// Fast-branch phasor (cos, sin)(phi z) / a, a = pi/8, from phi8 = phi 8/pi
// (uwb_devmath.cuh step_sincos8): k = rint(phi8 z), r = phi8 z - k by one FMA
// (|r| <= 1/2, no Cody-Waite constants, no phi z product), kernels with the
// powers of a folded into their coefficients, the 16-entry (cos, sin)(k pi/8)
// table.  15 FP64 instructions where dev_sincos(phi z) took 17.
__constant__ double c_s8[3] = {kStep8S0, kStep8S1, kStep8S2};
__constant__ double c_c8[4] = {kStep8C0, kStep8C1, kStep8C2, kInvPio8};

constexpr double kUnitInv = kInvPio8;  // 1 / (the phase unit pi/8)

#ifndef UWB_SINCOS_NOTAB
#define UWB_SINCOS_NOTAB 1
#endif
#if UWB_SINCOS_NOTAB
// Shipping phasor (uwb_devmath.cuh step_sincos8q, same operation sequence):
// reduction to multiples of pi/2 (k = rint(phi8 z / 4) by a 1.5 * 2^54
// shifter, r = phi8 z - 4k in [-2, 2] pi/8 units), sin degree 9 (2.5e-12) and
// cos degree 10 (1.4e-13) with the powers of pi/8 folded in, then the
// quarter-turn rotation by a swap and two sign flips of the high word: 14 FP64
// instructions and no table (the pi/8 version: 15 FP64 and a bank-conflicted
// LDS.128, 5.5 of the ~26 LSU wavefronts per warp-step; 7.62 -> 7.12 ms).
__constant__ double c_s8q[4] = {kStepQS0, kStepQS1, kStepQS2, kStepQS3};
__constant__ double c_c8q[5] = {kStepQC0, kStepQC1, kStepQC2, kStepQC3, kStepQC4};
#endif
__device__ __forceinline__ void step_sincos8(double phi8, double z, const StepTabs& T,
                                             double* c_out, double* s_out) {
#if UWB_SINCOS_NOTAB
  constexpr double kMagic4 = 4.0 * kMagic;
  const double t4 = fma(phi8, z, kMagic4);
  const int q4 = __double2loint(t4);
  const double kd4 = t4 - kMagic4;
  const double r4 = fma(phi8, z, -kd4);
  const double z4 = r4 * r4;
  double ps4 = fma(z4, c_s8q[3], c_s8q[2]);
  ps4 = fma(ps4, z4, c_s8q[1]);
  ps4 = fma(ps4, z4, c_s8q[0]);
  const double sr4 = fma(r4 * z4, ps4, r4);
  double pc4 = fma(z4, c_c8q[4], c_c8q[3]);
  pc4 = fma(pc4, z4, c_c8q[2]);
  pc4 = fma(pc4, z4, c_c8q[1]);
  pc4 = fma(pc4, z4, c_c8q[0]);
  const double cr4 = fma(pc4, z4, kInvPio8);
  const bool sw = (q4 & 1) != 0;
  const double c4 = sw ? sr4 : cr4, s4 = sw ? cr4 : sr4;
  *c_out = __hiloint2double(__double2hiint(c4) ^ (((q4 + 1) & 2) << 30), __double2loint(c4));
  *s_out = __hiloint2double(__double2hiint(s4) ^ ((q4 & 2) << 30), __double2loint(s4));
#else
  const double t = fma(phi8, z, kMagic);
  const int q = __double2loint(t) & 15;
  const double kd = t - kMagic;
  const double r = fma(phi8, z, -kd);
  const double zz = r * r;
  double ps = fma(zz, c_s8[2], c_s8[1]);
  ps = fma(ps, zz, c_s8[0]);
  const double sr = fma(r * zz, ps, r);
  double pc = fma(zz, c_c8[2], c_c8[1]);
  pc = fma(pc, zz, c_c8[0]);
  const double cr = fma(pc, zz, c_c8[3]);
  const double2 cs = T.cs16[q];
  const double tc = cs.x, ts = cs.y;
  *c_out = fma(tc, cr, -(ts * sr));
  *s_out = fma(ts, cr, tc * sr);
#endif
}

// ---- compensated-FP32 ("mixed") step arithmetic (GnSolverConfig precision
// extension, BASELINE config 4).  What must stay FP64 stays FP64: the log2 rho
// interpolation, the split of 16 log2 p into (k, r), the phase phi z and its
// reduction modulo pi/8, and every sum past the lane.  What is evaluated in
// FP32 is only what is already small and well conditioned: 2^(r/16) on
// |r| <= 1/2, sin/cos on |r| <= pi/16, expm1 of the step-to-step log change,
// and the lane's K-step partial sums.  The summation-by-parts differences
// p_{m-1} - p_m are formed as p_m (2^(d/16) - 1) with d = lg_{m-1} - lg_m
// taken in FP64 first, so they never cancel in FP32.
__shared__ float s_exp2_tabf[16];
__shared__ float s_cos16f[16];
__shared__ float s_sin16f[16];

// 2^(x/16) for x = 16 log2 p in FP64 -> FP32 (relative error ~1e-7).
__device__ __forceinline__ float mixed_exp2_16(double x) {
  const double t = x + kMagic;
  int k = __double2loint(t);
  const float r = __double2float_rn(x - (t - kMagic));  // |r| <= 1/2
  const float y = r * 0.043321698784996581f;            // r ln2 / 16
  float e = fmaf(y, 1.0f / 24.0f, 1.0f / 6.0f);
  e = fmaf(e, y, 0.5f);
  e = fmaf(e, y, 1.0f);
  e = fmaf(e, y, 1.0f);
  k = max(k, -16 * 120);  // p < 2^-120 is far below anything the sum resolves
  const float v = s_exp2_tabf[k & 15] * e;
  return __int_as_float(__float_as_int(v) + ((k >> 4) << 23));
}

// p_m (2^(d/16) - 1) = p_{m-1} - p_m without cancellation: Taylor in
// y = d ln2/16 for |y| < 0.3 (relative error < 1e-8); past that the plain
// difference loses at most two bits.
__device__ __forceinline__ float mixed_dp(float p, float pprev, float d) {
  const float y = d * 0.043321698784996581f;
  float e = fmaf(y, 1.0f / 5040.0f, 1.0f / 720.0f);
  e = fmaf(e, y, 1.0f / 120.0f);
  e = fmaf(e, y, 1.0f / 24.0f);
  e = fmaf(e, y, 1.0f / 6.0f);
  e = fmaf(e, y, 0.5f);
  e = fmaf(e, y, 1.0f);
  return fabsf(y) < 0.3f ? p * (e * y) : pprev - p;
}

// (cos x, sin x) in FP32 with the reduction x = k pi/8 + r done in FP64 (the
// phase reaches 1e5 rad), r rounded to FP32 (|r| <= pi/16), Taylor kernels
// (sin to r^5, cos to r^6: truncation < 3e-9) and the 16-entry tables.
__device__ __forceinline__ void mixed_sincos(double x, float* c_out, float* s_out) {
  const double t = fma(x, c_red8[0], kMagic);
  const int q = __double2loint(t) & 15;
  const double kd = t - kMagic;
  double rd = fma(kd, c_red8[1], x);
  rd = fma(kd, c_red8[2], rd);
  const float r = __double2float_rn(rd);
  const float z = r * r;
  const float ps = fmaf(z, 1.0f / 120.0f, -1.0f / 6.0f);
  const float sr = fmaf(r * z, ps, r);
  float pc = fmaf(z, -1.0f / 720.0f, 1.0f / 24.0f);
  pc = fmaf(pc, z, -0.5f);
  const float cr = fmaf(pc, z, 1.0f);
  const float tc = s_cos16f[q], ts = s_sin16f[q];
  *c_out = fmaf(tc, cr, -(ts * sr));
  *s_out = fmaf(ts, cr, tc * sr);
}

// |sum over spans & steps|^2 for one point, computed by one 16-lane segment.
// Lane sl owns the K consecutive steps m = sl K + b (lane_pos layout, so for
// each b the segment's 16 loads of a column are one 128-byte line).
// Fast branch (gn_integral.hpp:156-175) by summation by parts of the
// reference's phasor-difference sum:
//   sum_m p_m (E_{m+1} - E_m) = -p_0 E_0 + sum_{m} (p_m - p_{m+1}) E_{m+1}
// (p_N = 0): step b adds (p_{b-1} - p_b) E_b of the previous step, the
// lane's last step pairs with the next lane's first p (one shuffle per point),
// so each step costs one exp2 and one sincos and nothing crosses lanes inside
// the step loop.  The phasors are E / a (a = pi/8, step_sincos8); the sum is
// divided by j phi8 = j phi / a, which restores the scale.  Slow branch
// (:176-188) is the direct sinc form.  Lanes with m >= N (only when
// N < 16 K) mask p to 0 and feed sincos z = 0.
// HOIST: the lane's K end-edge positions Zr and probe half-logs Hr live in
// registers for the whole row (single span, K <= 8); the row setup's fast
// flag (span 0's test) and z0 == 0 come in as arguments.
// K = 0: steps per lane known only at run time (spans longer than 512
// steps): the same code with rolled step loops.
// Both half-warps always run this together (warp-uniform point loop), so the
// segment shuffles use the full mask: no run-time convergence checks.
template <int K, bool FULL, bool HOIST, bool TINY>
__device__ __forceinline__ double point_kernel(const NliParams& P, const WarpSmem& S, int idx,
                                               int probe, int sl, bool fast0, bool z0zero,
                                               const StepTabs& TB, const double (&Zr)[K > 0 ? K : 1],
                                               const double (&Hr)[K > 0 ? K : 1]) {
  const int Kr = K > 0 ? K : P.col_stride / 16;
  const int NS = 16 * Kr;
  const PointRec& R = S.pt[idx];
  const double2 wa = *reinterpret_cast<const double2*>(&R.w[0]);
  const double2 wb = *reinterpret_cast<const double2*>(&R.w[2]);
  const double2 wc = *reinterpret_cast<const double2*>(&R.w[4]);
  const double2 ph = *reinterpret_cast<const double2*>(&R.phi8);
  const int4 cl = *reinterpret_cast<const int4*>(&R.col[0]);
  const double phi8 = ph.x;
  const double w0 = wa.x, w1 = wa.y, w2 = wb.x, w3 = wb.y, w4 = wc.x, w5 = wc.y;
  const int oa = cl.x + sl, ob = cl.y + sl, oc = cl.z + sl;
  // columns i0 and i0 + 1 of every stencil inside the [n_ch + 1][NS] table
  UWB_BOUND(cl.x >= 0 && cl.y >= 0 && cl.z >= 0 && max(cl.x, max(cl.y, cl.z)) + 2 * NS <=
                                                       (P.n_ch + 1) * NS);
  UWB_BOUND(idx >= 0 && idx < 32 && probe < P.n_probes);
  double fre = 0.0, fim = 0.0, sre = 0.0, sim = 0.0;
  const int n_spans = HOIST ? 1 : P.n_spans;
  for (int k = 0; k < n_spans; ++k) {
    // this span's own step count (spans may differ, gn_integral.hpp:231-251)
    const int N = (HOIST || !P.span_steps) ? P.steps : __ldg(P.span_steps + k);
    const double* T = P.log2rho + k * P.span_stride;
    const double* ca = T + oa;
    const double* cb = T + ob;
    const double* cc3 = T + oc;
    const double* hl = P.hl2 + (static_cast<size_t>(probe) * P.n_spans + k) * NS + sl;
    const bool fast = HOIST ? fast0 : fabs(R.phi) * __ldg(P.wlast + k) > 1e-4;
    double p0 = 0.0, pp = 0.0, pc = 0.0, ps = 0.0;
    if (fast) {
      const double* ze = P.zedge + static_cast<size_t>(k) * NS + sl;
#pragma unroll(K > 0 ? K : 4)
      for (int b = 0; b < Kr; ++b) {
        const int o = 16 * b;
        const double H = HOIST ? Hr[b] : __ldg(hl + o);
        double Z = HOIST ? (UWB_Z_SMEM ? TB_z(TB, o + sl) : Zr[b]) : __ldg(ze + o);
        double lg = fma(w0, __ldg(ca + o), -H);
        lg = fma(w1, __ldg(ca + NS + o), lg);
        lg = fma(w2, __ldg(cb + o), lg);
        lg = fma(w3, __ldg(cb + NS + o), lg);
        lg = fma(w4, __ldg(cc3 + o), lg);
        lg = fma(w5, __ldg(cc3 + NS + o), lg);
        double p = step_exp2_16t(lg, TB);
        if (!FULL) {
          const bool ok = sl * Kr + b < N;
          p = ok ? p : 0.0;
          Z = ok ? Z : 0.0;
        }
        double cs, sn;
        step_sincos8(phi8, Z, TB, &cs, &sn);
        if (b == 0) {
          p0 = p;
        } else {  // (p_{m-1} - p_m) E_m, E_m = end edge of the previous step
          const double cf = pp - p;
          fre = fma(cf, pc, fre);
          fim = fma(cf, ps, fim);
        }
        pp = p;
        pc = cs;
        ps = sn;
      }
    } else {
      const double phi = R.phi;
      const double* zm = P.zmid + static_cast<size_t>(k) * NS + sl;
      const double* wd = P.width + static_cast<size_t>(k) * NS + sl;
      // fully unrolled like the fast loop (independent steps interleave);
      // lanes past N contribute a zero weight.  A sinc-branch point has
      // |phi| w_last <= 1e-4, so its phases are small: TINY kernels are
      // chosen by the host when 1e-4 z_max / w_last <= 2^-6 (NliParams::
      // slow_tiny, true for single-span grids like the bench's), and there the
      // Taylor kernels to x^6 / x^7 are exact to < 1e-19 and replace the
      // reduction + table sincos (8 FP64 instructions instead of 19).  Each
      // kernel holds one of the two loops (both in one kernel cost 4 %).
#pragma unroll(K > 0 ? K : 4)
      for (int b = 0; b < Kr; ++b) {
        const int o = 16 * b;
        const double H = HOIST ? Hr[b] : __ldg(hl + o);
        double lg = fma(w0, __ldg(ca + o), -H);
        lg = fma(w1, __ldg(ca + NS + o), lg);
        lg = fma(w2, __ldg(cb + o), lg);
        lg = fma(w3, __ldg(cb + NS + o), lg);
        lg = fma(w4, __ldg(cc3 + o), lg);
        lg = fma(w5, __ldg(cc3 + NS + o), lg);
        const double p = step_exp2_16t(lg, TB);
        const double wm = __ldg(wd + o);
        // sinc(x), |x| = |phi| w / 2 <= 5e-5 here: 1 - x^2/6 + x^4/120 is exact
        const double x = 0.5 * phi * wm;
        const double x2 = x * x;
        const double sinc = fma(x2, fma(x2, 1.0 / 120.0, -1.0 / 6.0), 1.0);
        double w = p * wm * sinc;
        if (!FULL) w = (sl * Kr + b < N) ? w : 0.0;
        const double a = phi * __ldg(zm + o);
        double cs, sn;
        if constexpr (TINY) {
          const double a2 = a * a;
          cs = fma(a2, fma(a2, fma(a2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
          sn = fma(a * a2, fma(a2, fma(a2, -1.0 / 5040.0, 1.0 / 120.0), -1.0 / 6.0), a);
        } else {
          dev_sincos(a, &cs, &sn);
        }
        sre = fma(w, cs, sre);
        sim = fma(w, sn, sim);
      }
    }
    // the lane's last step pairs with the next lane's first (p_N = 0); both
    // half-warps reach this shuffle whatever their branch
    double pn = __shfl_down_sync(kFull, p0, 1, 16);
    if (fast) {
      if (sl == 15) pn = 0.0;
      const double cf = pp - pn;
      fre = fma(cf, pc, fre);
      fim = fma(cf, ps, fim);
      // -p_0 E(z_0) / a: E = 1 when the span starts at z = 0
      if (HOIST ? z0zero : __ldg(P.zstart + k) == 0.0) {
        if (sl == 0) fre = fma(-p0, kUnitInv, fre);
      } else {
        double c0v, s0v;
        step_sincos8(phi8, __ldg(P.zstart + k), TB, &c0v, &s0v);
        if (sl == 0) {
          fre = fma(-p0, c0v, fre);
          fim = fma(-p0, s0v, fim);
        }
      }
    }
  }
  // fast spans contribute (sum / (j phi)) = (scaled sum / (j phi8))
  // (gn_integral.hpp:173-175)
  const double rphi8 = ph.y;
  double re = fma(fim, rphi8, sre);
  double im = fma(-fre, rphi8, sim);
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    re += __shfl_xor_sync(kFull, re, o, 16);
    im += __shfl_xor_sync(kFull, im, o, 16);
  }
  return re * re + im * im;
}

// point_kernel for one 8-lane segment (single span, FP64; UWB_SEG8): a warp
// evaluates four points at a time.  Lane s8 takes the steps of the two
// 16-lane-layout lanes 2 s8 and 2 s8 + 1, i.e. the 2K CONTIGUOUS steps
// [2 s8 K, 2 s8 K + 2K): run A = first K, run B = next K.  In the lane-ordered
// table those two lanes' values for a given b sit side by side, so ONE 16-byte
// load serves both runs (three LDG.128 per step pair instead of six LDG.64 per
// step: the same L1 wavefronts, half the load instructions).  Run A's last step
// pairs with run B's first inside the lane; run B's last pairs with the next
// lane's first (one shuffle); the per-point record loads, the boundary shuffle
// and the 3-level reduction tree are amortised over 2K steps instead of K.
// The probe half-logs come from a per-warp shared column (S.h), the z edges
// from the CTA-wide one, both as 16-byte pairs.
template <int K, bool FULL, bool TINY, class WS>
__device__ __forceinline__ double point_kernel8(const NliParams& P, const WS& S, int idx,
                                                int s8, bool z0zero, const StepTabs& TB) {
  constexpr int NS = 16 * K;
  const PointRec& R = S.pt[idx];
  const double2 wa = *reinterpret_cast<const double2*>(&R.w[0]);
  const double2 wb = *reinterpret_cast<const double2*>(&R.w[2]);
  const double2 wc = *reinterpret_cast<const double2*>(&R.w[4]);
  const double2 ph = *reinterpret_cast<const double2*>(&R.phi8);
  const int4 cl = *reinterpret_cast<const int4*>(&R.col[0]);
  const bool fast = cl.w != 0;
  const double phi8 = ph.x;
  const double w0 = wa.x, w1 = wa.y, w2 = wb.x, w3 = wb.y, w4 = wc.x, w5 = wc.y;
  const int l2 = 2 * s8;
  UWB_BOUND(cl.x >= 0 && cl.y >= 0 && cl.z >= 0 && max(cl.x, max(cl.y, cl.z)) + 2 * NS <=
                                                       (P.n_ch + 1) * NS);
  const double2* ca = reinterpret_cast<const double2*>(P.log2rho + cl.x + l2);
  const double2* cb = reinterpret_cast<const double2*>(P.log2rho + cl.y + l2);
  const double2* cc3 = reinterpret_cast<const double2*>(P.log2rho + cl.z + l2);
  const double2* hs = reinterpret_cast<const double2*>(S_h(const_cast<WS&>(S)) + l2);
  const double2* zs = reinterpret_cast<const double2*>(TB.z + l2);
  constexpr int NS2 = NS / 2;  // the column stride in double2 units
  const int N = P.steps;
  const int mA = l2 * K, mB = mA + K;  // first step of run A / run B
  double fre = 0.0, fim = 0.0, sre = 0.0, sim = 0.0;
  double pA0 = 0.0, pB0 = 0.0, ppA = 0.0, ppB = 0.0, pcA = 0.0, psA = 0.0, pcB = 0.0, psB = 0.0;
  if (fast) {
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int o = 8 * b;  // 16 b doubles = 8 b double2
      const double2 H = hs[o];
      double2 Z = zs[o];
      const double2 a0 = __ldg(ca + o), a1 = __ldg(ca + NS2 + o);
      const double2 b0 = __ldg(cb + o), b1 = __ldg(cb + NS2 + o);
      const double2 c0 = __ldg(cc3 + o), c1 = __ldg(cc3 + NS2 + o);
      double lgA = fma(w0, a0.x, -H.x), lgB = fma(w0, a0.y, -H.y);
      lgA = fma(w1, a1.x, lgA), lgB = fma(w1, a1.y, lgB);
      lgA = fma(w2, b0.x, lgA), lgB = fma(w2, b0.y, lgB);
      lgA = fma(w3, b1.x, lgA), lgB = fma(w3, b1.y, lgB);
      lgA = fma(w4, c0.x, lgA), lgB = fma(w4, c0.y, lgB);
      lgA = fma(w5, c1.x, lgA), lgB = fma(w5, c1.y, lgB);
      double pA = step_exp2_16t(lgA, TB), pB = step_exp2_16t(lgB, TB);
      if (!FULL) {
        const bool okA = mA + b < N, okB = mB + b < N;
        pA = okA ? pA : 0.0;
        Z.x = okA ? Z.x : 0.0;
        pB = okB ? pB : 0.0;
        Z.y = okB ? Z.y : 0.0;
      }
      double cA, sA, cB, sB;
      step_sincos8(phi8, Z.x, TB, &cA, &sA);
      step_sincos8(phi8, Z.y, TB, &cB, &sB);
      if (b == 0) {
        pA0 = pA;
        pB0 = pB;
      } else {  // (p_{m-1} - p_m) E_m, E_m = end edge of the previous step
        const double cfA = ppA - pA, cfB = ppB - pB;
        fre = fma(cfA, pcA, fre);
        fim = fma(cfA, psA, fim);
        fre = fma(cfB, pcB, fre);
        fim = fma(cfB, psB, fim);
      }
      ppA = pA, pcA = cA, psA = sA;
      ppB = pB, pcB = cB, psB = sB;
    }
    // run A's last step pairs with run B's first
    const double cf = ppA - pB0;
    fre = fma(cf, pcA, fre);
    fim = fma(cf, psA, fim);
  } else {
    const double phi = R.phi;
    const double2* zm = reinterpret_cast<const double2*>(P.zmid + l2);
    const double2* wd = reinterpret_cast<const double2*>(P.width + l2);
#pragma unroll
    for (int b = 0; b < K; ++b) {
      const int o = 8 * b;
      const double2 H = hs[o];
      const double2 a0 = __ldg(ca + o), a1 = __ldg(ca + NS2 + o);
      const double2 b0 = __ldg(cb + o), b1 = __ldg(cb + NS2 + o);
      const double2 c0 = __ldg(cc3 + o), c1 = __ldg(cc3 + NS2 + o);
      double lgA = fma(w0, a0.x, -H.x), lgB = fma(w0, a0.y, -H.y);
      lgA = fma(w1, a1.x, lgA), lgB = fma(w1, a1.y, lgB);
      lgA = fma(w2, b0.x, lgA), lgB = fma(w2, b0.y, lgB);
      lgA = fma(w3, b1.x, lgA), lgB = fma(w3, b1.y, lgB);
      lgA = fma(w4, c0.x, lgA), lgB = fma(w4, c0.y, lgB);
      lgA = fma(w5, c1.x, lgA), lgB = fma(w5, c1.y, lgB);
      const double pv[2] = {step_exp2_16t(lgA, TB), step_exp2_16t(lgB, TB)};
      const double2 wm2 = __ldg(wd + o), zm2 = __ldg(zm + o);
      const double wmv[2] = {wm2.x, wm2.y}, zmv[2] = {zm2.x, zm2.y};
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        // sinc(x), |x| = |phi| w / 2 <= 5e-5 here: 1 - x^2/6 + x^4/120 is exact
        const double x = 0.5 * phi * wmv[r];
        const double x2 = x * x;
        const double sinc = fma(x2, fma(x2, 1.0 / 120.0, -1.0 / 6.0), 1.0);
        double w = pv[r] * wmv[r] * sinc;
        if (!FULL) w = ((r ? mB : mA) + b < N) ? w : 0.0;
        const double a = phi * zmv[r];
        double cs, sn;
        if constexpr (TINY) {
          const double a2 = a * a;
          cs = fma(a2, fma(a2, fma(a2, -1.0 / 720.0, 1.0 / 24.0), -0.5), 1.0);
          sn = fma(a * a2, fma(a2, fma(a2, -1.0 / 5040.0, 1.0 / 120.0), -1.0 / 6.0), a);
        } else {
          dev_sincos(a, &cs, &sn);
        }
        sre = fma(w, cs, sre);
        sim = fma(w, sn, sim);
      }
    }
  }
  // run B's last step pairs with the next lane's first (p_N = 0); all four
  // segments reach this shuffle whatever their branch
  double pn = __shfl_down_sync(kFull, pA0, 1, 8);
  if (fast) {
    if (s8 == 7) pn = 0.0;
    const double cf = ppB - pn;
    fre = fma(cf, pcB, fre);
    fim = fma(cf, psB, fim);
    // -p_0 E(z_0) / a: E = 1 when the span starts at z = 0
    if (z0zero) {
      if (s8 == 0) fre = fma(-pA0, kUnitInv, fre);
    } else {
      double c0v, s0v;
      step_sincos8(phi8, __ldg(P.zstart), TB, &c0v, &s0v);
      if (s8 == 0) {
        fre = fma(-pA0, c0v, fre);
        fim = fma(-pA0, s0v, fim);
      }
    }
  }
  const double rphi8 = ph.y;
  double re = fma(fim, rphi8, sre);
  double im = fma(-fre, rphi8, sim);
#pragma unroll
  for (int o = 4; o >= 1; o >>= 1) {
    re += __shfl_xor_sync(kFull, re, o, 8);
    im += __shfl_xor_sync(kFull, im, o, 8);
  }
  return re * re + im * im;
}

// point_kernel in compensated FP32 (see mixed_exp2_16 above): same lane
// layout, same summation by parts, same fast/slow split; lane partial sums in
// FP32, everything across lanes in FP64.
template <int K, bool FULL, bool HOIST>
__device__ __forceinline__ double point_kernel_mixed(const NliParams& P, const WarpSmem& S, int idx,
                                                     int probe, int sl,
                                                     const double (&Zr)[K], const double (&Hr)[K]) {
  constexpr int NS = 16 * K;
  const PointRec& R = S.pt[idx];
  const double2 wa = *reinterpret_cast<const double2*>(&R.w[0]);
  const double2 wb = *reinterpret_cast<const double2*>(&R.w[2]);
  const double2 wc = *reinterpret_cast<const double2*>(&R.w[4]);
  const int4 cl = *reinterpret_cast<const int4*>(&R.col[0]);
  const double phi = R.phi;
  const double w0 = wa.x, w1 = wa.y, w2 = wb.x, w3 = wb.y, w4 = wc.x, w5 = wc.y;
  const int oa = cl.x + sl, ob = cl.y + sl, oc = cl.z + sl;
  double fre = 0.0, fim = 0.0, sre = 0.0, sim = 0.0;
  const int n_spans = HOIST ? 1 : P.n_spans;
  for (int k = 0; k < n_spans; ++k) {
    const int N = (HOIST || !P.span_steps) ? P.steps : __ldg(P.span_steps + k);
    const double* T = P.log2rho + k * P.span_stride;
    const double* ca = T + oa;
    const double* cb = T + ob;
    const double* cc3 = T + oc;
    const double* hl = P.hl2 + (static_cast<size_t>(probe) * P.n_spans + k) * NS + sl;
    const bool fast = fabs(phi) * __ldg(P.wlast + k) > 1e-4;
    float lre = 0.0f, lim = 0.0f;  // fast branch: the lane's FP32 partial sums
    float p0 = 0.0f, pp = 0.0f, pc = 0.0f, ps = 0.0f;
    double lg0 = 0.0, lgp = 0.0;
    if (fast) {
      const double* ze = P.zedge + static_cast<size_t>(k) * NS + sl;
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const int o = 16 * b;
        const double H = HOIST ? Hr[b] : __ldg(hl + o);
        const double Z = HOIST ? Zr[b] : __ldg(ze + o);
        double lg = fma(w0, __ldg(ca + o), -H);
        lg = fma(w1, __ldg(ca + NS + o), lg);
        lg = fma(w2, __ldg(cb + o), lg);
        lg = fma(w3, __ldg(cb + NS + o), lg);
        lg = fma(w4, __ldg(cc3 + o), lg);
        lg = fma(w5, __ldg(cc3 + NS + o), lg);
        float p = mixed_exp2_16(lg);
        double ang = phi * Z;
        const bool ok = FULL || sl * K + b < N;
        if (!FULL) {
          p = ok ? p : 0.0f;
          ang = ok ? ang : 0.0;
        }
        float cs, sn;
        mixed_sincos(ang, &cs, &sn);
        if (b == 0) {
          p0 = p;
          lg0 = lg;
        } else {  // (p_{m-1} - p_m) E_m = p_m (2^((lg_{m-1} - lg_m)/16) - 1) E_m
          float cf = mixed_dp(p, pp, __double2float_rn(lgp - lg));
          if (!FULL) cf = ok ? cf : pp;
          lre = fmaf(cf, pc, lre);
          lim = fmaf(cf, ps, lim);
        }
        pp = p;
        lgp = lg;
        pc = cs;
        ps = sn;
      }
    } else {
      const double* zm = P.zmid + static_cast<size_t>(k) * NS + sl;
      const double* wd = P.width + static_cast<size_t>(k) * NS + sl;
      float ure = 0.0f, uim = 0.0f;
      const float phf = static_cast<float>(phi);
#pragma unroll
      for (int b = 0; b < K; ++b) {
        const int o = 16 * b;
        const double H = HOIST ? Hr[b] : __ldg(hl + o);
        double lg = fma(w0, __ldg(ca + o), -H);
        lg = fma(w1, __ldg(ca + NS + o), lg);
        lg = fma(w2, __ldg(cb + o), lg);
        lg = fma(w3, __ldg(cb + NS + o), lg);
        lg = fma(w4, __ldg(cc3 + o), lg);
        lg = fma(w5, __ldg(cc3 + NS + o), lg);
        const float p = mixed_exp2_16(lg);
        const float wm = static_cast<float>(__ldg(wd + o));
        // |x| = |phi| w / 2 <= 5e-5: 1 - x^2/6 is exact in FP32
        const float x = 0.5f * phf * wm;
        const float sinc = fmaf(x * x, -1.0f / 6.0f, 1.0f);
        float w = p * wm * sinc;
        if (!FULL) w = (sl * K + b < N) ? w : 0.0f;
        float cs, sn;
        mixed_sincos(phi * __ldg(zm + o), &cs, &sn);
        ure = fmaf(w, cs, ure);
        uim = fmaf(w, sn, uim);
      }
      sre += static_cast<double>(ure);
      sim += static_cast<double>(uim);
    }
    // the lane's last step pairs with the next lane's first (p_N = 0); both
    // half-warps reach these shuffles whatever their branch
    float pn = __shfl_down_sync(kFull, p0, 1, 16);
    const double lgn = __shfl_down_sync(kFull, lg0, 1, 16);
    if (fast) {
      if (sl == 15) pn = 0.0f;
      const float cf = pn == 0.0f ? pp : mixed_dp(pn, pp, __double2float_rn(lgp - lgn));
      lre = fmaf(cf, pc, lre);
      lim = fmaf(cf, ps, lim);
      fre += static_cast<double>(lre);
      fim += static_cast<double>(lim);
      // -p_0 E(z_0): E = 1 when the span starts at z = 0
      const double z0 = __ldg(P.zstart + k);
      if (z0 == 0.0) {
        if (sl == 0) fre -= p0;
      } else {
        double c0v, s0v;
        dev_sincos(phi * z0, &c0v, &s0v);
        if (sl == 0) {
          fre = fma(-static_cast<double>(p0), c0v, fre);
          fim = fma(-static_cast<double>(p0), s0v, fim);
        }
      }
    }
  }
  // 1/phi = (8/pi) / phi8 = (8/pi) rphi8
  const double invphi = R.rphi8 * kUnitInv;
  double re = fma(fim, invphi, sre);
  double im = fma(-fre, invphi, sim);
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    re += __shfl_xor_sync(kFull, re, o, 16);
    im += __shfl_xor_sync(kFull, im, o, 16);
  }
  return re * re + im * im;
}

template <int K, bool FULL, bool HOIST, bool MIXED, bool TINY>
__global__ void __launch_bounds__(WarpsFor<HOIST, MIXED>::value * 32,
                                  MIXED ? UWB_NLI_MIXED_MIN_BLOCKS : UWB_NLI_MIN_BLOCKS)
    nli_rows_kernel(const NliParams P) {
  constexpr int kWarps = WarpsFor<HOIST, MIXED>::value;
  // the point_kernel8 path keeps no per-lane |K|^2 (kv): its smaller records
  using WS = typename std::conditional<UWB_SEG8 && HOIST && !MIXED, WarpSmemCarry, WarpSmem>::type;
  __shared__ WS s_w[kWarps];
  __shared__ double2 s_tab_cs16[16];
  __shared__ double s_tab_e2c[16];
  __shared__ __align__(16) double s_tab_z[UWB_Z_SMEM ? 128 : 1];
  const StepTabs s_tabs{s_tab_cs16, s_tab_e2c, s_tab_z};
  init_step_tabs(s_tabs, threadIdx.x);
  if (threadIdx.x < 16) {
    s_exp2_tab[threadIdx.x] = c_exp2_tab16[threadIdx.x];
    s_cs16[threadIdx.x] = make_double2(c_tab_cos16[threadIdx.x], c_tab_sin16[threadIdx.x]);
    if (MIXED) {
      s_exp2_tabf[threadIdx.x] = __double2float_rn(c_exp2_tab16[threadIdx.x]);
      s_cos16f[threadIdx.x] = __double2float_rn(c_tab_cos16[threadIdx.x]);
      s_sin16f[threadIdx.x] = __double2float_rn(c_tab_sin16[threadIdx.x]);
    }
  }
#if UWB_Z_SMEM
  if (HOIST && threadIdx.x < 16 * K) s_tabs.z[threadIdx.x] = __ldg(P.zedge + threadIdx.x);
#endif
  __syncthreads();

  const int NS = 16 * (K > 0 ? K : P.col_stride / 16);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sl = lane & 15;
  const int seg = lane >> 4;
  WS& S = s_w[warp];
  const int per_probe = P.n_q * P.n_r;
  double Zr[K > 0 ? K : 1], Hr[K > 0 ? K : 1];
  int cur_probe = -1;
  if (HOIST && (!UWB_Z_SMEM || MIXED)) {  // the mixed kernel keeps its z edges in registers
#pragma unroll
    for (int b = 0; b < K; ++b) Zr[b] = __ldg(P.zedge + 16 * b + sl);
  }
  // single span (HOIST): its start z, zero for every grid build_distance_grid makes
  const bool z0zero = !HOIST || __ldg(P.zstart) == 0.0;

  for (;;) {
    int row = 0;
    if (lane == 0) row = static_cast<int>(atomicAdd(P.counter, 1u));
    row = __shfl_sync(kFull, row, 0);
    if (row >= P.total_rows) break;
    const int probe = row / per_probe;
    // prepared path: the probe's channel is dark in this evaluation -> the
    // reference skips it (gn_integral.hpp:349-352); its rows add nothing
    if (P.probe_chan && !(__ldg(P.psd + __ldg(P.probe_chan + probe)) > 0.0)) {
      if (lane == 0) {
        P.rowsum[row] = __longlong_as_double(0x7ff8000000000000ll);
        P.rowcnt[row] = make_uint2(0u, 0u);
      }
      continue;
    }
    if (HOIST && probe != cur_probe) {
      cur_probe = probe;
      if constexpr (UWB_SEG8 && !MIXED) {
        __syncwarp();  // the previous probe's column is no longer read
        for (int m = lane; m < NS; m += 32) S_h(S)[m] = __ldg(P.hl2 + static_cast<size_t>(probe) * NS + m);
        __syncwarp();
      } else {
#pragma unroll
        for (int b = 0; b < K; ++b) Hr[b] = __ldg(P.hl2 + static_cast<size_t>(probe) * NS + 16 * b + sl);
      }
    }
    const int n_r = P.n_r;
    double du1;
    {
      // the row's u1 bin and u2 range, precomputed by row_params_kernel (the
      // same arithmetic, one thread per row instead of every lane of a warp)
      const double2 rp0 = __ldg(reinterpret_cast<const double2*>(P.rowpar) + 2 * row);
      const double2 rp1 = __ldg(reinterpret_cast<const double2*>(P.rowpar) + 2 * row + 1);
      const double su = rp0.x;
      if (!(su >= 0.0)) {  // quadrant collapsed or empty u2 range: the reference `continue`s
        if (lane == 0) {
          P.rowsum[row] = __longlong_as_double(0x7ff8000000000000ll);
          P.rowcnt[row] = make_uint2(0u, 0u);
        }
        continue;
      }
      du1 = __ldg(P.rowsum + row);  // parked there by row_params_kernel
      const int rem = row - probe * per_probe;
      const int q = rem / n_r + 1;
      const double nu = __ldg(P.probe_nu + probe);
      const double f = nu - P.centre;
      const double s1 = (q == 1 || q == 4) ? 1.0 : -1.0;
      const double s2 = (q == 1 || q == 2) ? 1.0 : -1.0;
      __syncwarp();
      if (lane == 0) {
        S.nu = nu;
        S.f = f;
        S.s1 = s1;
        S.s2 = s2;
        S.su = su;
        S.u1 = rp0.y;
        S.lo = rp1.x;
        S.du2 = rp1.y;
        // quadrants 1 and 3 (s1 == s2, b1 == b2); quadrant 2 at f = 0 has
        // b1 == b2 too but maps (f1, f2) -> (-f2, -f1): not a symmetry
        const double bm = P.half_band - f, bp = P.half_band + f;
        const double b1 = (q == 1 || q == 4) ? bm : bp, b2 = (q == 1 || q == 2) ? bm : bp;
        S.sym = (P.mirror_u2 && s1 == s2 && b1 == b2) ? 1 : 0;
      }
      __syncwarp();
    }
    unsigned n_eval = 0, n_act_row = 0;
    // point_kernel8 path: points listed but not yet evaluated (they wait for a
    // full group of four: a warp iteration costs the same with idle segments)
    constexpr bool kCarry = UWB_SEG8 && HOIST && !MIXED;
    int n_pend = 0;
    double row_acc = 0.0;
    // Symmetric rows (quadrants 1 and 3: s1 == s2, b1 == b2): u2 -> -u2 swaps f1 and f2,
    // and the integrand is symmetric in them (phase_mismatch is bit-exactly
    // symmetric, gn_integral.hpp:43-50; the power factor is a product over
    // the three stencils), so column n_r-1-j carries the |K|^2 of column j up
    // to the few-ulp difference of the recomputed coordinates.  Each column
    // still gets its own setup (PSD window tests, p1 p2 p3), so the active set
    // is exactly the reference's; only |K|^2 is shared.  Lanes 0..15 take
    // columns j, lanes 16..31 their mirrors.
    const bool sym = S.sym != 0;
    const int half = sym ? (n_r + 1) / 2 : n_r;
    const int span = sym ? 16 : 32;
    for (int jb = 0; jb < half; jb += span) {
      // ---- per-point setup, one u2 column per lane (gn_integral.hpp:288-303)
      const int m = sym ? jb + (lane & 15) : jb + lane;
      const bool primary = !sym || lane < 16;
      const int j = primary ? m : n_r - 1 - m;
      const bool valid = m < half && (primary || j != m);
      bool active = false;
      bool fast = false;
      Stencil st1, st2, st3;
      double phi = 0.0, pw = 0.0;
      if (valid) {
        const double nu = S.nu, su = S.su, u1 = S.u1;
        const double u2 = S.lo + (static_cast<double>(j) + 0.5) * S.du2;
        // exp and the division as a 2^x table kernel and a correctly rounded
        // reciprocal (a few ulp from the reference's libm/IEEE ops; no slow paths)
        const double g1 = su * dev_exp2_16(u2 * (16.0 * kLog2e));
        const double g2 = u1 * __drcp_rn(g1);
        const double f1 = S.s1 * g1;
        const double f2 = S.s2 * g2;
        double p1, p2, p3;
        st1 = psd_and_stencil(P, nu + f1, &p1);
        st2 = psd_and_stencil(P, nu + f2, &p2);
        st3 = psd_and_stencil(P, nu + f1 + f2, &p3);
        active = p1 != 0.0 && p2 != 0.0 && p3 != 0.0;
        if (active) {
          phi = phase_mismatch(f1, f2, S.f, P.beta2, P.beta3, P.beta4);
          pw = p1 * p2 * p3;
          fast = fabs(phi) * __ldg(P.wlast) > 1e-4;
        }
      }
      const unsigned am = __ballot_sync(kFull, active);
      // a mirror column evaluates its own |K|^2 only if its partner is inactive
      const bool partner_active = sym && ((am >> (lane ^ 16)) & 1u);
      const double pw_partner = __shfl_xor_sync(kFull, pw, 16);
      const bool need = active && (primary || !partner_active);
      const unsigned nm = __ballot_sync(kFull, need);
      const unsigned fm = __ballot_sync(kFull, need && fast);
      const unsigned sm = nm & ~fm;
      const unsigned lt = (1u << lane) - 1u;
      if (need) {
        // fast points first, then slow ones, so half-warp pairs rarely diverge.
        // Column i0 + 1 is always read: clamped stencils have hw1 = 0 and the
        // table carries a zero pad column n.
        const int pos = (kCarry ? n_pend : 0) +
                        (fast ? __popc(fm & lt) : __popc(fm) + __popc(sm & lt));
        UWB_BOUND(pos >= 0 && pos < 36);
        UWB_BOUND(st1.i1 <= P.n_ch && st2.i1 <= P.n_ch && st3.i1 <= P.n_ch);
        PointRec& R = S.pt[pos];
        R.col[0] = st1.i0 * NS;
        R.col[1] = st2.i0 * NS;
        R.col[2] = st3.i0 * NS;
        if (kCarry) {
          R.src = fast ? 1 : 0;
          // this column's weight plus its mirror's when the mirror shares |K|^2
          R.pws = pw + ((sym && primary && partner_active) ? pw_partner : 0.0);
        } else {
          R.src = lane;
        }
        R.w[0] = st1.hw0 * 16.0; R.w[1] = st1.hw1 * 16.0;
        R.w[2] = st2.hw0 * 16.0; R.w[3] = st2.hw1 * 16.0;
        R.w[4] = st3.hw0 * 16.0; R.w[5] = st3.hw1 * 16.0;
        const double phi8 = phi * kUnitInv;
        R.phi8 = phi8;
        R.rphi8 = phi != 0.0 ? __drcp_rn(phi8) : 0.0;
        R.phi = phi;
      }
      __syncwarp();
      const int n_need = __popc(nm);
      const int n_fast = __popc(fm);
      n_eval += n_need;
      n_act_row += __popc(am);
      // warp-uniform trip count: with an odd count the idle half-warp repeats
      // its partner's point (same branch, result dropped) instead of diverging
      if constexpr (kCarry) {
        // four points per warp, one per 8-lane segment, in full groups only;
        // the rest (at most three) move to the front and wait for the next
        // chunk.  Row sum (gn_integral.hpp:288-305): each group's four
        // weighted |K|^2 by a fixed tree, groups added in order -- the order
        // depends on the row's activity pattern only, so rows are
        // reproducible and independent of scheduling and partitioning.
        const int sg = lane >> 3, s8 = lane & 7;
        const int avail = n_pend + n_need;
        const int full4 = avail & ~3;
        for (int base = 0; base < full4; base += 4) {
          const int idx = base + sg;
          const double kv = point_kernel8<K, FULL, TINY>(P, S, idx, s8, z0zero, s_tabs);
          double v = s8 == 0 ? S.pt[idx].pws * kv : 0.0;
          v += __shfl_xor_sync(kFull, v, 8);
          v += __shfl_xor_sync(kFull, v, 16);
          row_acc += v;
        }
        __syncwarp();
        n_pend = avail - full4;
        if (full4 > 0 && n_pend > 0) {  // source [full4, avail) and target [0, n_pend) are disjoint
          double* d = reinterpret_cast<double*>(S.pt);
          const double* src = reinterpret_cast<const double*>(S.pt + full4);
          constexpr int kWords = static_cast<int>(sizeof(PointRec) / sizeof(double));
          for (int t = lane; t < n_pend * kWords; t += 32) d[t] = src[t];
        }
        __syncwarp();
        continue;
      } else {
        for (int base = 0; base < n_need; base += 2) {
          const bool ok = base + seg < n_need;
          const int idx = ok ? base + seg : base;
          double kv;
          if constexpr (MIXED)
            kv = point_kernel_mixed<K, FULL, HOIST>(P, S, idx, probe, sl, Zr, Hr);
          else
            kv = point_kernel<K, FULL, HOIST, TINY>(P, S, idx, probe, sl, idx < n_fast, z0zero,
                                                    s_tabs, Zr, Hr);
          if (ok && sl == 0) S.kv[S.pt[idx].src] = kv;
        }
        __syncwarp();
        UWB_BOUND(!valid || (j >= 0 && j < n_r));
        // row sum (gn_integral.hpp:288-305): each chunk's 32 column values by a
        // fixed xor tree, chunks added in ascending order -- the order depends
        // on (n_r, row symmetry) only, so rows are reproducible and independent of
        // scheduling and partitioning, and no per-row array is kept
        double v = (valid && active) ? pw * (need ? S.kv[lane] : S.kv[lane ^ 16]) : 0.0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
        row_acc += v;
        __syncwarp();
      }
    }
    if constexpr (kCarry) {
      if (n_pend > 0) {  // the row's last (at most three) points; idle segments repeat point 0
        const int sg = lane >> 3, s8 = lane & 7;
        const bool ok = sg < n_pend;
        const int idx = ok ? sg : 0;
        const double kv = point_kernel8<K, FULL, TINY>(P, S, idx, s8, z0zero, s_tabs);
        double v = (ok && s8 == 0) ? S.pt[idx].pws * kv : 0.0;
        v += __shfl_xor_sync(kFull, v, 8);
        v += __shfl_xor_sync(kFull, v, 16);
        row_acc += v;
        __syncwarp();
      }
    }
    if (lane == 0) {
      UWB_BOUND(row < P.total_rows);
      P.rowsum[row] = row_acc * du1 * S.du2;
      P.rowcnt[row] = make_uint2(n_eval, n_act_row);  // summed per probe by the finalize
    }
    __syncwarp();

  }
}

// ---- split evaluation (launch_nli_setup / launch_nli_lists) ----------------
// Pass 1 (nli_setup_kernel, beside the Raman ODE): every row's column setup
// (coordinates, the three PSD windows and stencils, phi, the mirror sharing),
// compacted exactly like the fused kernel's chunks, written as point records
// to the row's slot list.  Pass 2 (nli_list_kernel): the fused kernel's group
// loop over the listed records.  Both keep the fused order, so the row sums
// are bit-identical to nli_rows_kernel's.
constexpr int kSetupWarps = 8;

__global__ void __launch_bounds__(kSetupWarps * 32) nli_setup_kernel(const NliParams P) {
  if (threadIdx.x < 16) s_exp2_tab[threadIdx.x] = c_exp2_tab16[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int NS = P.col_stride;
  const int n_r = P.n_r;
  const int per_probe = P.n_q * n_r;
  for (;;) {
    int row = 0;
    if (lane == 0) row = static_cast<int>(atomicAdd(P.counter, 1u));
    row = __shfl_sync(kFull, row, 0);
    if (row >= P.total_rows) break;
    const int probe = row / per_probe;
    const double2 rp0 = __ldg(reinterpret_cast<const double2*>(P.rowpar) + 2 * row);
    const double2 rp1 = __ldg(reinterpret_cast<const double2*>(P.rowpar) + 2 * row + 1);
    const bool dark = P.probe_chan && !(__ldg(P.psd + __ldg(P.probe_chan + probe)) > 0.0);
    if (dark || !(rp0.x >= 0.0)) {  // the reference `continue`s (gn_integral.hpp:349-352, :283)
      if (lane == 0) {
        P.rowsum[row] = __longlong_as_double(0x7ff8000000000000ll);
        P.rowcnt[row] = make_uint2(0u, 0u);
        P.plist_n[row] = -1;
      }
      continue;
    }
    const int rem = row - probe * per_probe;
    const int q = rem / n_r + 1;
    const double nu = __ldg(P.probe_nu + probe);
    const double f = nu - P.centre;
    const double s1 = (q == 1 || q == 4) ? 1.0 : -1.0;
    const double s2 = (q == 1 || q == 2) ? 1.0 : -1.0;
    const double bm = P.half_band - f, bp = P.half_band + f;
    const double b1 = (q == 1 || q == 4) ? bm : bp, b2 = (q == 1 || q == 2) ? bm : bp;
    const bool sym = P.mirror_u2 && s1 == s2 && b1 == b2;
    const double su = rp0.x, u1 = rp0.y, lo = rp1.x, du2 = rp1.y;
    PointRec* out = static_cast<PointRec*>(P.plist) + static_cast<size_t>(row) * n_r;
    int count = 0;
    unsigned n_eval = 0, n_act_row = 0;
    const int half = sym ? (n_r + 1) / 2 : n_r;
    const int span = sym ? 16 : 32;
    for (int jb = 0; jb < half; jb += span) {
      // the fused kernel's column setup (nli_rows_kernel, gn_integral.hpp:288-303)
      const int m = sym ? jb + (lane & 15) : jb + lane;
      const bool primary = !sym || lane < 16;
      const int j = primary ? m : n_r - 1 - m;
      const bool valid = m < half && (primary || j != m);
      bool active = false;
      bool fast = false;
      Stencil st1, st2, st3;
      double phi = 0.0, pw = 0.0;
      if (valid) {
        const double u2 = lo + (static_cast<double>(j) + 0.5) * du2;
        const double g1 = su * dev_exp2_16(u2 * (16.0 * kLog2e));
        const double g2 = u1 * __drcp_rn(g1);
        const double f1 = s1 * g1;
        const double f2 = s2 * g2;
        double p1, p2, p3;
        st1 = psd_and_stencil(P, nu + f1, &p1);
        st2 = psd_and_stencil(P, nu + f2, &p2);
        st3 = psd_and_stencil(P, nu + f1 + f2, &p3);
        active = p1 != 0.0 && p2 != 0.0 && p3 != 0.0;
        if (active) {
          phi = phase_mismatch(f1, f2, f, P.beta2, P.beta3, P.beta4);
          pw = p1 * p2 * p3;
          fast = fabs(phi) * __ldg(P.wlast) > 1e-4;
        }
      }
      const unsigned am = __ballot_sync(kFull, active);
      const bool partner_active = sym && ((am >> (lane ^ 16)) & 1u);
      const double pw_partner = __shfl_xor_sync(kFull, pw, 16);
      const bool need = active && (primary || !partner_active);
      const unsigned nm = __ballot_sync(kFull, need);
      const unsigned fm = __ballot_sync(kFull, need && fast);
      const unsigned sm = nm & ~fm;
      const unsigned lt = (1u << lane) - 1u;
      if (need) {
        const int pos = count + (fast ? __popc(fm & lt) : __popc(fm) + __popc(sm & lt));
        UWB_BOUND(pos >= 0 && pos < n_r);
        const double phi8 = phi * kUnitInv;
        double2* r2 = reinterpret_cast<double2*>(out + pos);
        __stcs(r2 + 0, make_double2(st1.hw0 * 16.0, st1.hw1 * 16.0));
        __stcs(r2 + 1, make_double2(st2.hw0 * 16.0, st2.hw1 * 16.0));
        __stcs(r2 + 2, make_double2(st3.hw0 * 16.0, st3.hw1 * 16.0));
        __stcs(r2 + 3, make_double2(phi8, phi != 0.0 ? __drcp_rn(phi8) : 0.0));
        __stcs(reinterpret_cast<int4*>(r2 + 4),
               make_int4(st1.i0 * NS, st2.i0 * NS, st3.i0 * NS, fast ? 1 : 0));
        __stcs(r2 + 5, make_double2(phi, pw + ((sym && primary && partner_active) ? pw_partner : 0.0)));
      }
      count += __popc(nm);
      n_eval += __popc(nm);
      n_act_row += __popc(am);
    }
    if (lane == 0) {
      P.plist_n[row] = count;
      P.rowcnt[row] = make_uint2(n_eval, n_act_row);
    }
  }
}

#ifndef UWB_LIST_WARPS
// 10 warps x 2 CTAs (96 registers): the list kernel keeps no row setup, so it
// fits in fewer registers than the fused kernel's 128; 8 / 9 / 11 / 12 warps
// measured 7.09 / 7.17 / 8.10 / 7.74 ms against 7.00 (profiles/r02_integrand_experiments.md)
#define UWB_LIST_WARPS 10
#endif
#ifndef UWB_LIST_MIN_BLOCKS
#define UWB_LIST_MIN_BLOCKS UWB_NLI_MIN_BLOCKS
#endif
template <int K, bool FULL, bool TINY>
__global__ void __launch_bounds__(UWB_LIST_WARPS * 32, UWB_LIST_MIN_BLOCKS)
    nli_list_kernel(const NliParams P) {
  constexpr int kWarps = UWB_LIST_WARPS;
  constexpr int NS = 16 * K;
  __shared__ ListWarpSmem s_w[kWarps];
  __shared__ double2 s_tab_cs16[16];
  __shared__ double s_tab_e2c[16];
  __shared__ __align__(16) double s_tab_z[128];
  const StepTabs s_tabs{s_tab_cs16, s_tab_e2c, s_tab_z};
  init_step_tabs(s_tabs, threadIdx.x);
  if (threadIdx.x < 16)
    s_cs16[threadIdx.x] = make_double2(c_tab_cos16[threadIdx.x], c_tab_sin16[threadIdx.x]);
  if (threadIdx.x < NS) s_tab_z[threadIdx.x] = __ldg(P.zedge + threadIdx.x);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  ListWarpSmem& S = s_w[threadIdx.x >> 5];
  const int n_r = P.n_r;
  const int per_probe = P.n_q * n_r;
  const bool z0zero = __ldg(P.zstart) == 0.0;
  int cur_probe = -1;
  for (;;) {
    int row = 0;
    if (lane == 0) row = static_cast<int>(atomicAdd(P.counter, 1u));
    row = __shfl_sync(kFull, row, 0);
    if (row >= P.total_rows) break;
    const int n = __ldg(P.plist_n + row);
    if (n < 0) continue;  // skipped: the setup pass wrote its NaN and counts
    const int probe = row / per_probe;
    if (probe != cur_probe) {
      cur_probe = probe;
      __syncwarp();
      for (int m = lane; m < NS; m += 32) S_h(S)[m] = __ldg(P.hl2 + static_cast<size_t>(probe) * NS + m);
      __syncwarp();
    }
    const double2* src = reinterpret_cast<const double2*>(static_cast<const PointRec*>(P.plist) +
                                                          static_cast<size_t>(row) * n_r);
    constexpr int kRec2 = static_cast<int>(sizeof(PointRec) / sizeof(double2));
    int n_pend = 0;
    double row_acc = 0.0;
    const int sg = lane >> 3, s8 = lane & 7;
    for (int c0 = 0; c0 < n; c0 += kListChunk) {
      const int cnt = min(kListChunk, n - c0);
      double2* dst = reinterpret_cast<double2*>(S.pt + n_pend);
      for (int t = lane; t < cnt * kRec2; t += 32) dst[t] = __ldcs(src + c0 * kRec2 + t);
      __syncwarp();
      // the fused kernel's groups of four with the remainder carried over
      const int avail = n_pend + cnt;
      const int full4 = avail & ~3;
      for (int base = 0; base < full4; base += 4) {
        const int idx = base + sg;
        const double kv = point_kernel8<K, FULL, TINY>(P, S, idx, s8, z0zero, s_tabs);
        double v = s8 == 0 ? S.pt[idx].pws * kv : 0.0;
        v += __shfl_xor_sync(kFull, v, 8);
        v += __shfl_xor_sync(kFull, v, 16);
        row_acc += v;
      }
      __syncwarp();
      n_pend = avail - full4;
      if (full4 > 0 && n_pend > 0) {
        double* d = reinterpret_cast<double*>(S.pt);
        const double* sp = reinterpret_cast<const double*>(S.pt + full4);
        constexpr int kWords = static_cast<int>(sizeof(PointRec) / sizeof(double));
        for (int t = lane; t < n_pend * kWords; t += 32) d[t] = sp[t];
      }
      __syncwarp();
    }
    if (n_pend > 0) {
      const bool ok = sg < n_pend;
      const int idx = ok ? sg : 0;
      const double kv = point_kernel8<K, FULL, TINY>(P, S, idx, s8, z0zero, s_tabs);
      double v = (ok && s8 == 0) ? S.pt[idx].pws * kv : 0.0;
      v += __shfl_xor_sync(kFull, v, 8);
      v += __shfl_xor_sync(kFull, v, 16);
      row_acc += v;
      __syncwarp();
    }
    if (lane == 0) {
      const double du1 = P.rowsum[row];  // parked by row_params_kernel
      const double du2 = __ldg(P.rowpar + 4 * static_cast<size_t>(row) + 3);
      P.rowsum[row] = row_acc * du1 * du2;
    }
    __syncwarp();
  }
}

// Per-row parameters of the hyperbolic grid (gn_integral.hpp:258-286): the u1
// bin (log or uniform edges), su = sqrt(u1) and the u2 range, one thread per
// row with exactly the arithmetic the row kernel used to repeat in every lane.
// rowpar[row] = (su, u1, lo, du2); du1 is parked in rowsum[row] (the row
// kernel overwrites it with the row's sum).  su = -1 marks a skipped row.
__global__ void row_params_kernel(const NliParams P) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= P.total_rows) return;
  const int n_r = P.n_r;
  const int per_probe = P.n_q * n_r;
  const int probe = row / per_probe;
  const int rem = row - probe * per_probe;
  const int q = rem / n_r + 1;
  const int i = rem - (q - 1) * n_r;
  const double nu = P.probe_nu[probe];
  const double f = nu - P.centre;
  // quadrant_limits (gn_integral.hpp:63-79)
  const double bm = P.half_band - f, bp = P.half_band + f;
  double b1, b2;
  switch (q) {
    case 1: b1 = bm; b2 = bm; break;
    case 2: b1 = bp; b2 = bm; break;
    case 3: b1 = bp; b2 = bp; break;
    default: b1 = bm; b2 = bp; break;
  }
  double2* rp = reinterpret_cast<double2*>(P.rowpar) + 2 * row;
  const double u1_max = b1 * b2;
  if (!(u1_max > 0.0)) {
    rp[0] = make_double2(-1.0, 0.0);
    return;
  }
  double e0, e1;
  if (P.u1_uniform) {
    e0 = u1_max * static_cast<double>(i) / n_r;
    e1 = u1_max * static_cast<double>(i + 1) / n_r;
  } else {
    e0 = i == 0 ? 0.0 : u1_max * exp(P.ln_min * static_cast<double>(n_r - i) / (n_r - 1));
    e1 = u1_max * exp(P.ln_min * static_cast<double>(n_r - i - 1) / (n_r - 1));
  }
  const double u1 = (e0 == 0.0 || P.u1_uniform) ? 0.5 * (e0 + e1) : sqrt(e0 * e1);
  const double su = sqrt(u1);
  const double hi = log(b1 / su);
  const double lo = -log(b2 / su);
  if (!(hi > lo)) {
    rp[0] = make_double2(-1.0, 0.0);
    return;
  }
  rp[0] = make_double2(su, u1);
  rp[1] = make_double2(lo, (hi - lo) / n_r);
  P.rowsum[row] = e1 - e0;
}

// Probe half-log columns (gn_integral.hpp:234-251), in log2 units, plus the
// per-probe quadrant_limits validity check done on the host.
__global__ void probe_halflog_kernel(const NliParams P) {
  const int probe = blockIdx.x;
  const double nu = P.probe_nu[probe];
  double unused;
  const Stencil sc = psd_and_stencil(P, nu, &unused);
  const int NS = P.col_stride;
  for (int k = 0; k < P.n_spans; ++k) {
    const double* T = P.log2rho + k * P.span_stride;
    double* out = P.hl2 + (static_cast<size_t>(probe) * P.n_spans + k) * NS;
    for (int m = threadIdx.x; m < NS; m += blockDim.x) {
      // 16 x (the reference's half-log, in log2): the integrand works in 2^-4 log2 units
      out[m] = 16.0 * (sc.hw0 * T[static_cast<size_t>(sc.i0) * NS + m] +
                       sc.hw1 * T[static_cast<size_t>(sc.i1) * NS + m]);
    }
  }
}

// Kahan sum over rows in ascending i per quadrant (gn_integral.hpp:258,306),
// Q4 mirror (:310) and G = 16/27 gamma^2 sum_q (:312).  One CTA per probe,
// one warp per quadrant: the warp stages its n_r row sums in shared memory
// with coalesced loads, then lane 0 runs the (inherently sequential) Kahan
// sum from shared memory.
__global__ void finalize_probes_kernel(const NliParams P, const FinalizeParams F) {
  extern __shared__ double fin_smem[];
  const int probe = blockIdx.x;
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double quad[4];
  __shared__ unsigned long long cnt[4][2];
  if (q < P.n_q) {
    double* rs_s = fin_smem + q * P.n_r;
    const double* rs = P.rowsum + (static_cast<size_t>(probe) * P.n_q + q) * P.n_r;
    const uint2* rc = P.rowcnt + (static_cast<size_t>(probe) * P.n_q + q) * P.n_r;
    unsigned long long ce = 0, ca = 0;
    for (int i = lane; i < P.n_r; i += 32) {
      rs_s[i] = rs[i];
      const uint2 c2 = rc[i];
      ce += c2.x;
      ca += c2.y;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      ce += __shfl_xor_sync(0xffffffffu, ce, o);
      ca += __shfl_xor_sync(0xffffffffu, ca, o);
    }
    if (lane == 0) {
      cnt[q][0] = ce;
      cnt[q][1] = ca;
    }
    __syncwarp();
    if (lane == 0) {
      double sum = 0.0, comp = 0.0;
      for (int i = 0; i < P.n_r; ++i) {
        const double x = rs_s[i];
        if (isnan(x)) continue;
        const double y = x - comp;
        const double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
      }
      quad[q] = sum;
    }
  } else if (lane == 0 && q < 4) {
    quad[q] = 0.0;
    cnt[q][0] = cnt[q][1] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // work counters: one atomic per probe (not per row)
    const unsigned long long ce = cnt[0][0] + cnt[1][0] + cnt[2][0] + cnt[3][0];
    const unsigned long long ca = cnt[0][1] + cnt[1][1] + cnt[2][1] + cnt[3][1];
    atomicAdd(P.n_eval, ce);
    atomicAdd(P.n_active, ca);
    if (P.probe_work) P.probe_work[probe] = ce;
    double qd[4] = {quad[0], quad[1], quad[2], P.n_q > 3 ? quad[3] : 0.0};
    if (F.mirror_q4) qd[3] = qd[1];
    const double g = F.probe_gamma[probe];
    F.probe_g[probe] = (16.0 / 27.0) * g * g * (qd[0] + qd[1] + qd[2] + qd[3]);
    for (int k = 0; k < 4; ++k) F.probe_quad[4 * probe + k] = qd[k];
  }
}

// channel_nli + the all_channels_nli epilogue (gn_integral.hpp:316-359).
__global__ void finalize_channels_kernel(const FinalizeParams F) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= F.n_ch) return;
  const int p0 = F.chan_probe0[ch];
  // p0 < 0: not probed (guard, outside the subset, or dark at the call);
  // psd <= 0 with a probe: dark in this evaluation of a prepared link
  if (p0 < 0 || !(F.psd[ch] > 0.0)) {
    F.eta[ch] = F.nli_psd[ch] = F.nli_power[ch] = 0.0;
    for (int q = 0; q < 4; ++q) F.quad[4 * ch + q] = 0.0;
    F.skipped[ch] = 1;
    return;
  }
  double psd = F.probe_g[p0];
  if (F.simpson) psd = (F.probe_g[p0 + 1] + 4.0 * psd + F.probe_g[p0 + 2]) / 6.0;
  const double p = F.psd[ch] * F.bch;
  F.nli_psd[ch] = psd;
  F.nli_power[ch] = psd * F.bch;
  F.eta[ch] = F.nli_power[ch] / (p * p * p);
  for (int q = 0; q < 4; ++q) F.quad[4 * ch + q] = F.probe_quad[4 * p0 + q];
  F.skipped[ch] = 0;
}

using RowKernel = void (*)(const NliParams);

// threads per CTA of an instantiation: its launch bounds (WarpsFor)
int row_threads(RowKernel k) {
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return 0;
  return fa.maxThreadsPerBlock;
}

// full: every span has exactly 16 K steps (no masked lanes).
template <int K, bool MIXED>
RowKernel pick2(bool full, bool one_span, bool tiny) {
  constexpr bool kHoist = K <= 8;
  if (one_span && kHoist) {
    if (!MIXED && tiny)
      return full ? nli_rows_kernel<K, true, kHoist, MIXED, !MIXED>
                  : nli_rows_kernel<K, false, kHoist, MIXED, !MIXED>;
    return full ? nli_rows_kernel<K, true, kHoist, MIXED, false>
                : nli_rows_kernel<K, false, kHoist, MIXED, false>;
  }
  return full ? nli_rows_kernel<K, true, false, MIXED, false>
              : nli_rows_kernel<K, false, false, MIXED, false>;
}

template <int K>
RowKernel pick(bool full, bool one_span, bool mixed, bool tiny) {
  return mixed ? pick2<K, true>(full, one_span, tiny) : pick2<K, false>(full, one_span, tiny);
}

// Long spans (257..512 steps, e.g. 80 km at > 3.2 steps/km): FP64, per-step
// z / half-log loads (no hoisting at this K); the compensated-FP32 mode stops
// at 256 steps.
template <int K>
RowKernel pick_long(bool full, bool mixed) {
  if (mixed) return nullptr;
  return full ? nli_rows_kernel<K, true, false, false, false>
              : nli_rows_kernel<K, false, false, false, false>;
}

// steps: the longest span's step count; ragged: spans differ in step count.
RowKernel row_kernel_for(int steps, bool one_span, bool mixed, bool tiny, bool ragged = false) {
  const int K = (steps + 15) / 16;
  const bool full = steps == 16 * K && !ragged;
  if (K > 32) return mixed ? nullptr : nli_rows_kernel<0, false, false, false, false>;
  switch (K) {
    case 1: return pick<1>(full, one_span, mixed, tiny);
    case 2: return pick<2>(full, one_span, mixed, tiny);
    case 3: return pick<3>(full, one_span, mixed, tiny);
    case 4: return pick<4>(full, one_span, mixed, tiny);
    case 5: return pick<5>(full, one_span, mixed, tiny);
    case 6: return pick<6>(full, one_span, mixed, tiny);
    case 7: return pick<7>(full, one_span, mixed, tiny);
    case 8: return pick<8>(full, one_span, mixed, tiny);
    case 9: return pick<9>(full, one_span, mixed, tiny);
    case 10: return pick<10>(full, one_span, mixed, tiny);
    case 11: return pick<11>(full, one_span, mixed, tiny);
    case 12: return pick<12>(full, one_span, mixed, tiny);
    case 13: return pick<13>(full, one_span, mixed, tiny);
    case 14: return pick<14>(full, one_span, mixed, tiny);
    case 15: return pick<15>(full, one_span, mixed, tiny);
    case 16: return pick<16>(full, one_span, mixed, tiny);
    case 17: return pick_long<17>(full, mixed);
    case 18: return pick_long<18>(full, mixed);
    case 19: return pick_long<19>(full, mixed);
    case 20: return pick_long<20>(full, mixed);
    case 21: return pick_long<21>(full, mixed);
    case 22: return pick_long<22>(full, mixed);
    case 23: return pick_long<23>(full, mixed);
    case 24: return pick_long<24>(full, mixed);
    case 25: return pick_long<25>(full, mixed);
    case 26: return pick_long<26>(full, mixed);
    case 27: return pick_long<27>(full, mixed);
    case 28: return pick_long<28>(full, mixed);
    case 29: return pick_long<29>(full, mixed);
    case 30: return pick_long<30>(full, mixed);
    case 31: return pick_long<31>(full, mixed);
    case 32: return pick_long<32>(full, mixed);
    default: return nullptr;
  }
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

int nli_bounds_status() {
#if UWB_BOUNDS_CHECK
  int v = 0;
  cudaMemcpyFromSymbol(&v, g_nli_bounds_fail, sizeof v);
  return v;
#else
  return -1;  // not a bounds-checked build
#endif
}

double fp64_fma_peak_tflops(int sm_count, cudaStream_t st) {
  const int blocks = sm_count * 8, threads = 256, iters = 2048;
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * blocks * threads) != cudaSuccess) return 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    dfma_peak_kernel<<<blocks, threads, 0, st>>>(out, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
    if (rep > 0 && ms > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

int launch_finalize_channels_only(const FinalizeParams& f, cudaStream_t st) {
  finalize_channels_kernel<<<(f.n_ch + 127) / 128, 128, 0, st>>>(f);
  return 1;
}

namespace {
size_t row_smem(int) { return 0; }  // rows keep no per-column array (running chunk sums)
// Shared-memory carveout: the smallest configuration that holds the CTAs one
// SM runs (launch bounds), so the rest of the 256 KB stays L1 for the log2 rho
// table (the default picked a 132 KB carveout for 2 x 38 KB: 124 KB of L1).
void allow_row_smem(RowKernel k, int /*n_r*/, size_t coresident = 0) {
  // The attribute is per (device, kernel); contexts on several devices are
  // driven from concurrent host threads (optimise_launch_powers), hence the lock.
  struct Seen {
    int dev;
    RowKernel k;
    size_t co;
  };
  static std::mutex mu;
  static Seen seen[256];
  static int n_seen = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  Seen* slot = nullptr;
  for (int i = 0; i < n_seen; ++i)
    if (seen[i].dev == dev && seen[i].k == k) {
      if (seen[i].co == coresident) return;
      slot = &seen[i];
      break;
    }
  static const bool no_carveout = [] {  // UWB_NLI_NO_CARVEOUT=1: driver default (A/B)
    const char* e = std::getenv("UWB_NLI_NO_CARVEOUT");
    return e && e[0] == '1';
  }();
  cudaFuncAttributes fa{};
  int per_sm = 0;
  if (!no_carveout && cudaFuncGetAttributes(&fa, k) == cudaSuccess &&
      cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) ==
          cudaSuccess &&
      per_sm > 0) {
    // CTAs the register file holds (the launch bounds' target)
    const int ctas = std::max(1, 65536 / (std::max(fa.numRegs, 1) * fa.maxThreadsPerBlock));
    const size_t need = static_cast<size_t>(ctas) * (fa.sharedSizeBytes + 1024) +
                        (coresident ? coresident + 1024 : 0);
    const int pct = static_cast<int>(std::min<size_t>(100, (100 * need + per_sm - 1) / per_sm));
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  if (slot)
    slot->co = coresident;
  else if (n_seen < 256)
    seen[n_seen++] = Seen{dev, k, coresident};
}
}  // namespace

int nli_ctas_per_sm(int steps, bool one_span, int n_r, bool mixed, bool tiny, bool ragged) {
  RowKernel k = row_kernel_for(steps, one_span, mixed, tiny, ragged);
  if (!k) return 0;
  allow_row_smem(k, n_r);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, row_threads(k), row_smem(n_r)) !=
      cudaSuccess)
    return 0;
  return n;
}

using ListKernel = void (*)(const NliParams);

template <int K>
ListKernel pick_list(bool full, bool tiny) {
  if (tiny) return full ? nli_list_kernel<K, true, true> : nli_list_kernel<K, false, true>;
  return full ? nli_list_kernel<K, true, false> : nli_list_kernel<K, false, false>;
}

ListKernel list_kernel_for(const NliParams& p) {
  const int K = (p.steps + 15) / 16;
  const bool full = p.steps == 16 * K;
  const bool tiny = p.slow_tiny != 0;
  switch (K) {
    case 1: return pick_list<1>(full, tiny);
    case 2: return pick_list<2>(full, tiny);
    case 3: return pick_list<3>(full, tiny);
    case 4: return pick_list<4>(full, tiny);
    case 5: return pick_list<5>(full, tiny);
    case 6: return pick_list<6>(full, tiny);
    case 7: return pick_list<7>(full, tiny);
    case 8: return pick_list<8>(full, tiny);
    default: return nullptr;
  }
}

int launch_nli(const NliParams& p, const FinalizeParams& f, int grid_ctas, cudaStream_t stream,
               cudaEvent_t ev_k0, cudaEvent_t ev_k1, size_t coresident_smem) {
  // UWB_NLI_NO_HOIST=1 selects the per-point z/half-log loads (A/B experiments)
  static const bool no_hoist = [] {
    const char* e = std::getenv("UWB_NLI_NO_HOIST");
    return e && e[0] == '1';
  }();
  RowKernel k = row_kernel_for(p.steps, p.n_spans == 1 && !no_hoist, p.mixed != 0, p.slow_tiny != 0,
                               p.span_steps != nullptr);
  if (!k || p.n_probes <= 0 || p.col_stride != 16 * ((p.steps + 15) / 16)) return -1;
  int launches = 0;
  cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), stream);
  cudaMemsetAsync(p.n_eval, 0, 2 * sizeof(unsigned long long), stream);  // n_eval, n_active
  probe_halflog_kernel<<<p.n_probes, 128, 0, stream>>>(p);
  row_params_kernel<<<(p.total_rows + 255) / 256, 256, 0, stream>>>(p);
  launches += 2;
  if (ev_k0) cudaEventRecord(ev_k0, stream);
  static const bool no_co = [] {  // UWB_NLI_NO_CO=1: ignore coresident_smem (A/B)
    const char* e = std::getenv("UWB_NLI_NO_CO");
    return e && e[0] == '1';
  }();
  allow_row_smem(k, p.n_r, no_co ? 0 : coresident_smem);
  k<<<grid_ctas, row_threads(k), row_smem(p.n_r), stream>>>(p);
  ++launches;
  if (ev_k1) cudaEventRecord(ev_k1, stream);
  const size_t fin_smem = static_cast<size_t>(p.n_q) * p.n_r * sizeof(double);
  if (fin_smem > 48 * 1024)
    cudaFuncSetAttribute(finalize_probes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(fin_smem));
  finalize_probes_kernel<<<f.n_probes, 128, fin_smem, stream>>>(p, f);
  ++launches;
  if (f.n_ch > 0) {
    finalize_channels_kernel<<<(f.n_ch + 127) / 128, 128, 0, stream>>>(f);
    ++launches;
  }
  return launches;
}

bool nli_split_ok(const NliParams& p) {
  static const bool off = [] {  // UWB_NLI_NO_SPLIT=1: the fused kernel only (A/B)
    const char* e = std::getenv("UWB_NLI_NO_SPLIT");
    return e && e[0] == '1';
  }();
  return !off && UWB_SEG8 && UWB_Z_SMEM && p.n_spans == 1 && !p.span_steps && !p.mixed &&
         p.steps >= 1 && p.steps <= 128 && p.col_stride == 16 * ((p.steps + 15) / 16);
}

size_t nli_point_record_bytes() { return sizeof(PointRec); }

int nli_list_ctas_per_sm(const NliParams& p) {
  ListKernel k = list_kernel_for(p);
  if (!k) return 0;
  allow_row_smem(k, p.n_r);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, UWB_LIST_WARPS * 32, 0) != cudaSuccess)
    return 0;
  return n;
}

int nli_setup_ctas_per_sm() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, nli_setup_kernel, kSetupWarps * 32, 0) !=
      cudaSuccess)
    return 0;
  return n;
}

int launch_nli_setup(const NliParams& p, int grid_ctas, cudaStream_t side) {
  if (!nli_split_ok(p) || !p.plist || !p.plist_n || p.n_probes <= 0) return -1;
  cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), side);
  cudaMemsetAsync(p.n_eval, 0, 2 * sizeof(unsigned long long), side);  // n_eval, n_active
  row_params_kernel<<<(p.total_rows + 255) / 256, 256, 0, side>>>(p);
  nli_setup_kernel<<<grid_ctas, kSetupWarps * 32, 0, side>>>(p);
  cudaMemsetAsync(p.counter, 0, sizeof(unsigned int), side);  // the list pass's queue
  return 2;
}

int launch_nli_lists(const NliParams& p, const FinalizeParams& f, int grid_ctas,
                     cudaStream_t stream, cudaEvent_t ev_k0, cudaEvent_t ev_k1) {
  ListKernel k = list_kernel_for(p);
  if (!k) return -1;
  int launches = 0;
  probe_halflog_kernel<<<p.n_probes, 128, 0, stream>>>(p);
  ++launches;
  if (ev_k0) cudaEventRecord(ev_k0, stream);
  allow_row_smem(k, p.n_r);  // the same carveout rule as the fused kernel
  k<<<grid_ctas, UWB_LIST_WARPS * 32, 0, stream>>>(p);
  ++launches;
  if (ev_k1) cudaEventRecord(ev_k1, stream);
  const size_t fin_smem = static_cast<size_t>(p.n_q) * p.n_r * sizeof(double);
  if (fin_smem > 48 * 1024)
    cudaFuncSetAttribute(finalize_probes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(fin_smem));
  finalize_probes_kernel<<<f.n_probes, 128, fin_smem, stream>>>(p, f);
  ++launches;
  if (f.n_ch > 0) {
    finalize_channels_kernel<<<(f.n_ch + 127) / 128, 128, 0, stream>>>(f);
    ++launches;
  }
  return launches;
}

}  // namespace uwb
