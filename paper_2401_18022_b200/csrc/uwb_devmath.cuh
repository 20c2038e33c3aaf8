// FP64 transcendentals for the NLI integrand, written for the B200 FP64 pipe.
//
// The integrand's inner step (gn_integral.hpp:161-172) needs one exp and one
// (cos, sin) pair per distance step.  CUDA's libdevice exp/sincos cost ~25 and
// ~41 DFMA-equivalents on sm_100a (measured, profiles/r01_microbench.md): they
// carry Payne-Hanek slow paths and overflow handling this path never needs.
// These versions are branch-free, use only DFMA/DMUL/DADD plus integer ops on
// the exponent, and stay within ~2 ulp of glibc:
//   exp2_pos  : 2^x via k = rint(32x), 32-entry 2^(j/32) table, degree-6
//               Taylor polynomial on |r| <= 1/64 (trunc. error 3.4e-18)
//               -> 10 FP64 instructions.
//   sincos_rd : Cody-Waite reduction by pi/2 with an exact FMA first part
//               (valid |x| < 2^50), fdlibm minimax kernels on [-pi/4, pi/4]
//               -> 18 FP64 instructions, quadrant fix-up on the ALU pipe.
// Both are __host__ __device__ so tests/ can compare them with libm on CPU.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define UWB_HD __host__ __device__ __forceinline__
#else
#define UWB_HD inline
#endif

namespace uwb {

constexpr double kPi = 3.14159265358979323846;
constexpr double kLog2e = 1.4426950408889634074;
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: rint via addition

UWB_HD int lo_word(double x) {
#if defined(__CUDA_ARCH__)
  return __double2loint(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return static_cast<int>(static_cast<uint32_t>(u));
#endif
}

UWB_HD int hi_word(double x) {
#if defined(__CUDA_ARCH__)
  return __double2hiint(x);
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return static_cast<int>(static_cast<uint32_t>(u >> 32));
#endif
}

UWB_HD double from_words(int hi, int lo) {
#if defined(__CUDA_ARCH__)
  return __hiloint2double(hi, lo);
#else
  const uint64_t u = (static_cast<uint64_t>(static_cast<uint32_t>(hi)) << 32) |
                     static_cast<uint32_t>(lo);
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}

UWB_HD double fmad(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// 2^(j/32), j = 0..31, correctly rounded (generated with 60-digit arithmetic).
#define UWB_EXP2_TABLE \
  {1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237,  \
   1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,  \
   1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332,  \
   1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,  \
   1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,  \
   1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,  \
   1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072,  \
   1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002}

// 2^(j/128), j = 0..127, correctly rounded (60-digit arithmetic).
#define UWB_EXP2_TABLE128 \
  { \
    1.0, 1.0054299011128027, 1.0108892860517005, 1.016378314910953, \
    1.0218971486541166, 1.0274459491187637, 1.0330248790212284, 1.0386341019613787, \
    1.0442737824274138, 1.0499440858006872, 1.0556451783605572, 1.061377227289262, \
    1.0671404006768237, 1.0729348675259756, 1.0787607977571199, 1.0846183622133092, \
    1.0905077326652577, 1.0964290818163769, 1.102382583307841, 1.1083684117236787, \
    1.1143867425958924, 1.1204377524096067, 1.1265216186082418, 1.1326385195987192, \
    1.1387886347566916, 1.1449721444318042, 1.1511892299529827, 1.1574400736337511, \
    1.1637248587775775, 1.1700437696832502, 1.1763969916502812, 1.182784710984341, \
    1.189207115002721, 1.1956643920398273, 1.202156731452703, 1.2086843236265816, \
    1.215247359980469, 1.2218460329727576, 1.22848053610687, 1.2351510639369334, \
    1.241857812073484, 1.2486009771892048, 1.255380757024691, 1.2621973503942507, \
    1.2690509571917332, 1.275941778396392, 1.2828700160787783, 1.2898358734066657, \
    1.2968395546510096, 1.3038812651919358, 1.3109612115247644, 1.318079601266064, \
    1.3252366431597413, 1.3324325470831615, 1.339667524053303, 1.3469417862329458, \
    1.3542555469368927, 1.3616090206382248, 1.3690024229745905, 1.3764359707545302, \
    1.383909881963832, 1.3914243757719262, 1.3989796725383112, 1.4065759938190154, \
    1.4142135623730951, 1.4218926021691656, 1.42961333839197, 1.4373759974489824, \
    1.4451808069770467, 1.4530279958490526, 1.460917794180647, 1.4688504333369818, \
    1.4768261459394993, 1.4848451658727524, 1.4929077282912648, 1.5010140696264256, \
    1.5091644275934228, 1.5173590411982147, 1.5255981507445384, 1.533881997840956, \
    1.5422108254079407, 1.550584877685, 1.559004400237837, 1.567469639965553, \
    1.5759808451078865, 1.5845382652524937, 1.593142151342267, 1.6017927556826934, \
    1.6104903319492543, 1.6192351351948637, 1.6280274218573478, 1.6368674497669644, \
    1.645755478153965, 1.6546917676561943, 1.6636765803267364, 1.6727101796415966, \
    1.681792830507429, 1.6909247992693053, 1.7001063537185235, 1.709337763100463, \
    1.718619298122478, 1.7279512309618377, 1.7373338352737062, 1.746767386199169, \
    1.7562521603732995, 1.7657884359332727, 1.7753764925265212, 1.785016611318935, \
    1.7947090750031072, 1.804454167806624, 1.8142521755003989, 1.8241033854070534, \
    1.8340080864093424, 1.843966568958626, 1.8539791250833855, 1.864046048397789, \
    1.8741676341103, 1.8843441790323345, 1.8945759815869656, 1.9048633418176741, \
    1.9152065613971474, 1.925605943636125, 1.9360617934922943, 1.9465744175792332, \
    1.9571441241754002, 1.9677712232331759, 1.978456026387951, 1.9891988469672663 \
  }

// Taylor coefficients of 2^r = exp(r ln2): (ln 2)^n / n!
constexpr double kE2c1 = 0.69314718055994530942;
constexpr double kE2c2 = 0.24022650695910071233;
constexpr double kE2c3 = 0.055504108664821579953;
constexpr double kE2c4 = 0.0096181291076284771620;
constexpr double kE2c5 = 0.0013333558146428443423;
constexpr double kE2c6 = 0.00015403530393381609954;

// 2^x for |x| < 1000 (the path's log2 power ratios are O(10)).  `tab` is the
// 32-entry table above (shared memory on the device).
UWB_HD double exp2_pos(double x, const double* tab) {
  const double t = fmad(x, 32.0, kMagic);
  const int k = lo_word(t);
  const double kd = t - kMagic;
  const double r = fmad(kd, -0.03125, x);  // exact: x - k/32, |r| <= 1/64
  double p = fmad(kE2c6, r, kE2c5);
  p = fmad(p, r, kE2c4);
  p = fmad(p, r, kE2c3);
  p = fmad(p, r, kE2c2);
  p = fmad(p, r, kE2c1);
  p = fmad(p, r, 1.0);
  const double s = tab[k & 31] * p;
  return from_words(hi_word(s) + ((k >> 5) << 20), lo_word(s));
}

// 2^(x/128) for the integrand's tables pre-scaled by 128 (x = 128 log2 p):
// k = rint(x) by DADD, r = x - k exact in [-1/2, 1/2], 2^(r/128) by a degree-5
// Taylor polynomial (|r ln2/128| <= 0.0027: truncation 5.4e-19), table 2^(j/128).
constexpr double kE7c1 = 0.0054152123481245725;
constexpr double kE7c2 = 1.4662262387640425e-05;
constexpr double kE7c3 = 2.646642144433097e-08;
constexpr double kE7c4 = 3.583032305400251e-11;
constexpr double kE7c5 = 3.880576156786539e-14;

UWB_HD double exp2_128(double x, const double* tab128) {
  const double t = x + kMagic;
  const int k = lo_word(t);
  const double r = x - (t - kMagic);
  double p = fmad(kE7c5, r, kE7c4);
  p = fmad(p, r, kE7c3);
  p = fmad(p, r, kE7c2);
  p = fmad(p, r, kE7c1);
  p = fmad(p, r, 1.0);
  const double s = tab128[k & 127] * p;
  return from_words(hi_word(s) + ((k >> 7) << 20), lo_word(s));
}

// 2^(x/16) for the integrand's tables pre-scaled by 16 (x = 16 log2 p): k =
// rint(x) by DADD, r = x - k exact in [-1/2, 1/2], 2^(r/16) by a degree-6
// minimax polynomial (Chebyshev fit in 40-digit arithmetic, |error| 7.0e-18
// relative), table 2^(j/16).  16 doubles fill the 32 shared-memory banks
// exactly: lookups never conflict.
#define UWB_EXP2_TABLE16                                                                    \
  {1.0, 1.0442737824274138, 1.0905077326652577, 1.1387886347566916, 1.189207115002721,      \
   1.241857812073484, 1.2968395546510096, 1.3542555469368927, 1.4142135623730951,           \
   1.4768261459394993, 1.5422108254079407, 1.6104903319492543, 1.681792830507429,           \
   1.7562521603732995, 1.8340080864093424, 1.9152065613971474}
constexpr double kE4c1 = 0.043321698784996678946;
constexpr double kE4c2 = 0.00093838479280898768341;
constexpr double kE4c3 = 0.000013550807776390032287;
constexpr double kE4c4 = 1.4676100321236696878e-7;
constexpr double kE4c5 = 1.2716120543851126972e-9;
constexpr double kE4c6 = 9.1813541921721152771e-12;

UWB_HD double exp2_16(double x, const double* tab16) {
  const double t = x + kMagic;
  const int k = lo_word(t);
  const double r = x - (t - kMagic);
  double p = fmad(kE4c6, r, kE4c5);
  p = fmad(p, r, kE4c4);
  p = fmad(p, r, kE4c3);
  p = fmad(p, r, kE4c2);
  p = fmad(p, r, kE4c1);
  p = fmad(p, r, 1.0);
  const double s = tab16[k & 15] * p;
  return from_words(hi_word(s) + ((k >> 4) << 20), lo_word(s));
}

// pi/2 split for the reduction: kPio2Hi = RN(pi/2), kPio2Lo = RN(pi/2 - kPio2Hi).
constexpr double kTwoOverPi = 0.63661977236758134308;
constexpr double kPio2Hi = 1.5707963267948966;
constexpr double kPio2Lo = 6.123233995736766e-17;

// fdlibm __kernel_sin / __kernel_cos minimax coefficients on [-pi/4, pi/4].
constexpr double kS1 = -1.66666666666666324348e-01;
constexpr double kS2 = 8.33333333332248946124e-03;
constexpr double kS3 = -1.98412698298579493134e-04;
constexpr double kS4 = 2.75573137070700676789e-06;
constexpr double kS5 = -2.50507602534068634195e-08;
constexpr double kS6 = 1.58969099521155010221e-10;
constexpr double kC1 = 4.16666666666666019037e-02;
constexpr double kC2 = -1.38888888888741095749e-03;
constexpr double kC3 = 2.48015872894767294178e-05;
constexpr double kC4 = -2.75573143513906633035e-07;
constexpr double kC5 = 2.08757232129817482790e-09;
constexpr double kC6 = -1.13596475577881948265e-11;

// (cos x, sin x) for |x| < 2^50.
UWB_HD void sincos_rd(double x, double* c_out, double* s_out) {
  const double t = fmad(x, kTwoOverPi, kMagic);
  const int q = lo_word(t);
  const double kd = t - kMagic;
  double r = fmad(kd, -kPio2Hi, x);  // exact (FMA, |result| < 2)
  r = fmad(kd, -kPio2Lo, r);
  const double z = r * r;
  double ps = fmad(kS6, z, kS5);
  ps = fmad(ps, z, kS4);
  ps = fmad(ps, z, kS3);
  ps = fmad(ps, z, kS2);
  ps = fmad(ps, z, kS1);
  const double rz = r * z;
  const double s = fmad(rz, ps, r);
  double pc = fmad(kC6, z, kC5);
  pc = fmad(pc, z, kC4);
  pc = fmad(pc, z, kC3);
  pc = fmad(pc, z, kC2);
  pc = fmad(pc, z, kC1);
  pc = fmad(pc, z, -0.5);
  const double c = fmad(pc, z, 1.0);  // 1 - z/2 + z^2 P(z), Horner
  // quadrant: sin(r + q pi/2), cos(r + q pi/2)
  const bool swap = (q & 1) != 0;
  double so = swap ? c : s;
  double co = swap ? s : c;
  const int sneg = (q & 2) << 30;        // bit 31 if q&2
  const int cneg = ((q + 1) & 2) << 30;  // bit 31 if (q+1)&2
  so = from_words(hi_word(so) ^ sneg, lo_word(so));
  co = from_words(hi_word(co) ^ cneg, lo_word(co));
  *c_out = co;
  *s_out = so;
}

// 16-entry full-circle sincos (nli_kernel.cu dev_sincos_table): x = k pi/8 + r.
constexpr double kEightOverPi = 2.5464790894703253723;
constexpr double kPio8Hi = 0.39269908169872414;      // RN(pi/8)
constexpr double kPio8Lo = 1.5308084989341915e-17;   // RN(pi/8 - kPio8Hi)
// sin r = r + r^3 S(r^2), minimax deg 3 on r^2 in [0, (pi/16)^2]
constexpr double kS16c1 = -0.1666666666666662344925285;
constexpr double kS16c2 = 0.008333333332974616029035064;
constexpr double kS16c3 = -0.0001984126518883108036053884;
constexpr double kS16c4 = 0.000002753800903667705587684024;
// cos r = 1 + r^2 C(r^2), minimax deg 4
constexpr double kC16c0 = -0.4999999999999999996528941;
constexpr double kC16c1 = 0.04166666666666621649926084;
constexpr double kC16c2 = -0.001388888888795474470406861;
constexpr double kC16c3 = 0.00002480158051684238140842294;
constexpr double kC16c4 = -0.0000002753720453432431172966888;
// cos(k pi/8), sin(k pi/8), k = 0..15, correctly rounded
#define UWB_COS_TABLE16                                                                     \
  {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,                 \
   -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,                  \
   -0.92387953251128674, -0.70710678118654757, -0.38268343236508978, 0.0,                   \
   0.38268343236508978, 0.70710678118654757, 0.92387953251128674}
#define UWB_SIN_TABLE16                                                                     \
  {0.0, 0.38268343236508978, 0.70710678118654757, 0.92387953251128674, 1.0,                 \
   0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,                      \
   -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,                  \
   -0.92387953251128674, -0.70710678118654757, -0.38268343236508978}

// Host/device restatement of the integrand's sincos (nli_kernel.cu
// dev_sincos_table): x = k pi/8 + r by Cody-Waite, minimax kernels on r, then
// the angle addition with cos/sin(k pi/8).  Tested against long double libm.
UWB_HD void sincos_tab16(double x, const double* cos16, const double* sin16, double* c_out,
                         double* s_out) {
  const double t = fmad(x, kEightOverPi, kMagic);
  const int q = lo_word(t) & 15;
  const double kd = t - kMagic;
  double r = fmad(kd, -kPio8Hi, x);
  r = fmad(kd, -kPio8Lo, r);
  const double z = r * r;
  double ps = fmad(z, kS16c4, kS16c3);
  ps = fmad(ps, z, kS16c2);
  ps = fmad(ps, z, kS16c1);
  const double sr = fmad(r * z, ps, r);
  double pc = fmad(z, kC16c4, kC16c3);
  pc = fmad(pc, z, kC16c2);
  pc = fmad(pc, z, kC16c1);
  pc = fmad(pc, z, kC16c0);
  const double cr = fmad(pc, z, 1.0);
  *c_out = fmad(cos16[q], cr, -(sin16[q] * sr));
  *s_out = fmad(sin16[q], cr, cos16[q] * sr);
}

// ---- step kernels of the integrand's hot loop (nli_kernel.cu, UWB_FAST_POLY=2)
// Shorter than the ulp-accurate kernels above: they only enter the per-step
// phasor sums, never a discrete decision (the row setup keeps exp2_16).
// Chebyshev fits in 50-digit arithmetic on the reduced ranges:
//   2^(r/16), |r| <= 1/2: 1 + r P(r), P degree 3 (quartic)  max rel. error 5e-12
//   sin r, |r| <= pi/16:  r + r^3 S(r^2), S degree 2        max abs. error 3.7e-14
//   cos r, |r| <= pi/16:  1 + r^2 C(r^2), C degree 2        max abs. error 1.7e-12
// nli_kernel.cu copies these into __constant__ banks (c_e4f, c_s3f, c_c3f);
// tests/test_devmath.py checks the restatements below against long double.
constexpr double kStepE0 = 0.043321698775062166;
constexpr double kStepE1 = 0.0009383847926296648;
constexpr double kStepE2 = 1.3551125679628034e-05;
constexpr double kStepE3 = 1.4676387236979493e-07;
constexpr double kStepS0 = -0.166666666661735;
constexpr double kStepS1 = 0.008333331030608612;
constexpr double kStepS2 = -0.0001982534004245333;
constexpr double kStepC0 = -0.4999999999556206;
constexpr double kStepC1 = 0.04166664594464585;
constexpr double kStepC2 = -0.0013874553368951438;

// The fast branch's sincos works in units of pi/8: with phi8 = phi 8/pi per
// point, x = phi z = (pi/8)(k + r) where k = rint(phi8 z) and r = phi8 z - k
// by one FMA (|r| <= 1/2), so the Cody-Waite reduction and the phi z product
// drop out.  The kernels return cos / sin (a r) divided by a = pi/8, i.e. the
// phasor scaled by 8/pi; the integrand folds the scale back in through
// 1/phi8 = (pi/8)/phi.  Coefficients: the kStepS* / kStepC* fits above with
// the powers of a folded in (50-digit arithmetic, tools/README.md):
//   sin(a r)/a = r + r^3 (a^2 S0 + r^2 (a^4 S1 + r^2 a^6 S2))
//   cos(a r)/a = 1/a + r^2 (a C0 + r^2 (a^3 C1 + r^2 a^5 C2))
// Equivalent to evaluating at phi' = phi8 pi/8 = phi (1 + d), |d| <= 2^-52:
// a phase error |d phi z| of the same size as the reference's own rounding of
// phi * (z_base + edge) (gn_integral.hpp:165).
constexpr double kStep8S0 = -0.02570209479374301;
constexpr double kStep8S1 = 0.00019817924828540812;
constexpr double kStep8S2 = -7.270762510593567e-07;
constexpr double kStep8C0 = -0.19634954083193434;
constexpr double kStep8C1 = 0.0025232960009761362;
constexpr double kStep8C2 = -1.2957417140207165e-05;
constexpr double kInvPio8 = 2.5464790894703255;  // RN(8/pi) = 1/a

// Quarter-turn variant without the (cos, sin)(q pi/8) table (the shipping
// nli_kernel.cu step_sincos8, UWB_SINCOS_NOTAB=1): k = rint(phi8 z / 4) by a
// 1.5 * 2^54 shifter (its ulp is 4), r = phi8 z - 4k in [-2, 2] by one FMA
// (|a r| <= pi/4), then
//   sin(a r)/a = r + r^3 (QS0 + r^2 (QS1 + r^2 (QS2 + r^2 QS3)))     (2.5e-12 abs)
//   cos(a r)/a = 1/a + r^2 (QC0 + r^2 (QC1 + ... + r^2 QC4))           (1.4e-13 abs)
// and the rotation by k pi/2 as a swap (k odd) and two sign flips.  Fits:
// weighted least squares on 6000 Chebyshev nodes of r^2 in [0, 4], refined in
// long double (errors measured against long-double libm; tests/test_devmath.py).
// The rotation has no arithmetic, so the phasor costs 14 FP64 instructions (the
// table version 15) and no shared-memory lookup.
constexpr double kStepQS0 = -0.025702094732684134;
constexpr double kStepQS1 = 0.00019817917932534872;
constexpr double kStepQS2 = -7.275778874298369e-07;
constexpr double kStepQS3 = 1.53596213791826e-09;
constexpr double kStepQC0 = -0.19634954084614456;
constexpr double kStepQC1 = 0.0025232972466868123;
constexpr double kStepQC2 = -1.2970795849995253e-05;
constexpr double kStepQC3 = 3.571476152561739e-08;
constexpr double kStepQC4 = -6.0315590453199e-11;

UWB_HD void step_sincos8q(double phi8, double z, double* c_out, double* s_out) {
  constexpr double kMagic4 = 4.0 * kMagic;
  const double t = fmad(phi8, z, kMagic4);
  const int q = lo_word(t);
  const double kd = t - kMagic4;
  const double r = fmad(phi8, z, -kd);
  const double zz = r * r;
  double ps = fmad(zz, kStepQS3, kStepQS2);
  ps = fmad(ps, zz, kStepQS1);
  ps = fmad(ps, zz, kStepQS0);
  const double sr = fmad(r * zz, ps, r);
  double pc = fmad(zz, kStepQC4, kStepQC3);
  pc = fmad(pc, zz, kStepQC2);
  pc = fmad(pc, zz, kStepQC1);
  pc = fmad(pc, zz, kStepQC0);
  const double cr = fmad(pc, zz, kInvPio8);
  const bool sw = (q & 1) != 0;
  const double c = sw ? sr : cr, s = sw ? cr : sr;
  *c_out = ((q + 1) & 2) ? -c : c;
  *s_out = (q & 2) ? -s : s;
}

// nli_kernel.cu step_sincos8 with UWB_SINCOS_NOTAB=0 (same operation
// sequence): (cos, sin)(phi z) / a.
UWB_HD void step_sincos8(double phi8, double z, const double* cos16, const double* sin16,
                         double* c_out, double* s_out) {
  const double t = fmad(phi8, z, kMagic);
  const int q = lo_word(t) & 15;
  const double kd = t - kMagic;
  const double r = fmad(phi8, z, -kd);
  const double zz = r * r;
  double ps = fmad(zz, kStep8S2, kStep8S1);
  ps = fmad(ps, zz, kStep8S0);
  const double sr = fmad(r * zz, ps, r);
  double pc = fmad(zz, kStep8C2, kStep8C1);
  pc = fmad(pc, zz, kStep8C0);
  const double cr = fmad(pc, zz, kInvPio8);
  *c_out = fmad(cos16[q], cr, -(sin16[q] * sr));
  *s_out = fmad(sin16[q], cr, cos16[q] * sr);
}

// nli_kernel.cu step_exp2_16 (same operation sequence).
UWB_HD double step_exp2_16(double x, const double* tab16) {
  const double t = x + kMagic;
  const int k = lo_word(t);
  const double r = x - (t - kMagic);
  double p = fmad(r, kStepE3, kStepE2);
  p = fmad(p, r, kStepE1);
  p = fmad(p, r, kStepE0);
  p = fmad(p, r, 1.0);
  const double s = tab16[k & 15] * p;
  return from_words(hi_word(s) + ((k >> 4) << 20), lo_word(s));
}

// nli_kernel.cu dev_sincos_table at UWB_FAST_POLY=2 (same operation sequence).
UWB_HD void step_sincos_tab16(double x, const double* cos16, const double* sin16, double* c_out,
                              double* s_out) {
  const double t = fmad(x, kEightOverPi, kMagic);
  const int q = lo_word(t) & 15;
  const double kd = t - kMagic;
  double r = fmad(kd, -kPio8Hi, x);
  r = fmad(kd, -kPio8Lo, r);
  const double z = r * r;
  double ps = fmad(z, kStepS2, kStepS1);
  ps = fmad(ps, z, kStepS0);
  const double sr = fmad(r * z, ps, r);
  double pc = fmad(z, kStepC2, kStepC1);
  pc = fmad(pc, z, kStepC0);
  const double cr = fmad(pc, z, 1.0);
  *c_out = fmad(cos16[q], cr, -(sin16[q] * sr));
  *s_out = fmad(sin16[q], cr, cos16[q] * sr);
}

}  // namespace uwb
