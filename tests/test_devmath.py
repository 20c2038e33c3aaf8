"""CPU: the integrand's FP64 transcendentals against long-double libm.

csrc/uwb_devmath.cuh holds __host__ __device__ restatements of the device
code: the ulp-accurate kernels of the row setup (exp2_16, sincos_tab16) and
the SHORTER step kernels the hot loop actually runs at UWB_FAST_POLY=2
(step_exp2_16: 2^x quartic; step_sincos8, the fast branch's phasor in units
of pi/8; step_sincos_tab16, the sinc branch's: sin degree 7, cos degree 6),
whose coefficients nli_kernel.cu's __constant__ banks are initialised from
(checked below).  Their documented error bounds are asserted here; the GPU
parity tests cover the kernels end to end."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include "uwb_devmath.cuh"
#include <cmath>
extern "C" {
static const double T32[32] = UWB_EXP2_TABLE;
static const double T16[16] = UWB_EXP2_TABLE16;
static const double T128[128] = UWB_EXP2_TABLE128;
static const double C16[16] = UWB_COS_TABLE16;
static const double S16[16] = UWB_SIN_TABLE16;
void exp2_16_v(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = uwb::exp2_16(x[i], T16); }
void exp2_128_v(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = uwb::exp2_128(x[i], T128); }
void exp2_pos_v(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = uwb::exp2_pos(x[i], T32); }
void sincos_v(const double* x, double* c, double* s, long n) { for (long i = 0; i < n; ++i) uwb::sincos_rd(x[i], c + i, s + i); }
double err_exp2_16(const double* x, long n) { long double m = 0; for (long i = 0; i < n; ++i) {
  long double r = exp2l((long double)x[i] / 16); long double e = fabsl((uwb::exp2_16(x[i], T16) - r) / r); if (e > m) m = e; } return (double)m; }
void sincos16_v(const double* x, double* c, double* s, long n) { for (long i = 0; i < n; ++i) uwb::sincos_tab16(x[i], C16, S16, c + i, s + i); }
double err_sincos16(const double* x, long n) { long double m = 0; for (long i = 0; i < n; ++i) {
  double c, s; uwb::sincos_tab16(x[i], C16, S16, &c, &s); long double ec = fabsl(c - cosl((long double)x[i])), es = fabsl(s - sinl((long double)x[i]));
  if (ec > m) m = ec; if (es > m) m = es; } return (double)m; }
double err_step_exp2_16(const double* x, long n) { long double m = 0; for (long i = 0; i < n; ++i) {
  long double r = exp2l((long double)x[i] / 16); long double e = fabsl((uwb::step_exp2_16(x[i], T16) - r) / r); if (e > m) m = e; } return (double)m; }
double err_step_sincos16(const double* x, long n, int which) { long double m = 0; for (long i = 0; i < n; ++i) {
  double c, s; uwb::step_sincos_tab16(x[i], C16, S16, &c, &s); long double ec = fabsl(c - cosl((long double)x[i])), es = fabsl(s - sinl((long double)x[i]));
  long double e = which == 0 ? ec : es; if (e > m) m = e; } return (double)m; }
double err_step_sincos8(const double* phi8, const double* z, long n, int which) { long double m = 0;
  const long double a = 3.14159265358979323846264338327950288L / 8; for (long i = 0; i < n; ++i) {
  double c, s; uwb::step_sincos8(phi8[i], z[i], C16, S16, &c, &s);
  // the kernel evaluates at phi' = phi8 pi/8 exactly and returns the phasor / a; the
  // reference phase is reduced exactly: phi8 z = k + r (r by a long double FMA),
  // x = a ((k mod 16) + r) differs from a phi8 z by a multiple of 2 pi
  const double k = rint(phi8[i] * z[i]);
  const long double r = fmal((long double)phi8[i], (long double)z[i], -(long double)k);
  long double x = a * ((long double)fmod(k, 16.0) + r);
  long double ec = fabsl(c * a - cosl(x)), es = fabsl(s * a - sinl(x));
  long double e = which == 0 ? ec : es; if (e > m) m = e; } return (double)m; }
double err_step_sincos8q(const double* phi8, const double* z, long n, int which) { long double m = 0;
  const long double a = 3.14159265358979323846264338327950288L / 8; for (long i = 0; i < n; ++i) {
  double c, s; uwb::step_sincos8q(phi8[i], z[i], &c, &s);
  const double k = rint(phi8[i] * z[i]);
  const long double r = fmal((long double)phi8[i], (long double)z[i], -(long double)k);
  long double x = a * ((long double)fmod(k, 16.0) + r);
  long double ec = fabsl(c * a - cosl(x)), es = fabsl(s * a - sinl(x));
  long double e = which == 0 ? ec : es; if (e > m) m = e; } return (double)m; }
double err_sincos(const double* x, long n) { long double m = 0; for (long i = 0; i < n; ++i) {
  double c, s; uwb::sincos_rd(x[i], &c, &s); long double ec = fabsl(c - cosl((long double)x[i])), es = fabsl(s - sinl((long double)x[i]));
  if (ec > m) m = ec; if (es > m) m = es; } return (double)m; }
}
'''


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    d = tmp_path_factory.mktemp("devmath")
    src = d / "dm.cpp"
    src.write_text(SRC)
    so = d / "dm.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2401_18022_b200", "csrc"), str(src), "-o",
                    str(so)], check=True)
    L = ctypes.CDLL(str(so))
    L.err_exp2_16.restype = ctypes.c_double
    L.err_sincos.restype = ctypes.c_double
    L.err_sincos16.restype = ctypes.c_double
    L.err_step_exp2_16.restype = ctypes.c_double
    L.err_step_sincos16.restype = ctypes.c_double
    L.err_step_sincos8.restype = ctypes.c_double
    L.err_step_sincos8q.restype = ctypes.c_double
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def test_exp2_16_accuracy(lib):
    # the integrand's argument: 16 log2(p), p in [2^-40, 2^4]
    x = np.random.default_rng(1).uniform(-40 * 16, 4 * 16, 400000)
    assert lib.err_exp2_16(_p(x), len(x)) < 4e-16
    y = np.zeros(3)
    lib.exp2_16_v(_p(np.array([0.0, 16.0, -16.0])), _p(y), 3)
    assert y.tolist() == [1.0, 2.0, 0.5]


@pytest.mark.parametrize("scale", [1.0, 1e3, 1e6, 3e7, 1e9])
def test_sincos_accuracy(lib, scale):
    # angles phi z reach ~3e7 rad on the 589-ch plan (SURVEY §7 hard part 1)
    x = np.random.default_rng(2).uniform(-scale, scale, 300000)
    assert lib.err_sincos(_p(x), len(x)) < 2.5e-16


def test_sincos_exact_zero(lib):
    c, s = np.zeros(1), np.zeros(1)
    lib.sincos_v(_p(np.zeros(1)), _p(c), _p(s), 1)
    assert c[0] == 1.0 and s[0] == 0.0  # E(z_0 = 0) of the first span


@pytest.mark.parametrize("scale", [1.0, 1e3, 1e6, 3e7, 1e9])
def test_sincos_table16_accuracy(lib, scale):
    """The integrand's 16-entry full-circle sincos (nli_kernel.cu dev_sincos_table)."""
    x = np.random.default_rng(3).uniform(-scale, scale, 300000)
    assert lib.err_sincos16(_p(x), len(x)) < 4e-16


def test_sincos_table16_exact_zero_and_quadrants(lib):
    x = np.array([0.0, np.pi / 2, np.pi, -np.pi / 2])
    c, s = np.zeros(4), np.zeros(4)
    lib.sincos16_v(_p(x), _p(c), _p(s), 4)
    assert c[0] == 1.0 and s[0] == 0.0
    assert np.allclose(c, np.cos(x), atol=3e-16) and np.allclose(s, np.sin(x), atol=3e-16)


# ---------------------------------------------------------------- step kernels (hot loop)
def test_step_exp2_16_error_bound(lib):
    """The hot loop's 2^(x/16) (quartic on |r| <= 1/2): relative error <= 5e-12
    (DESIGN.md §3.1), over the integrand's argument range."""
    x = np.random.default_rng(4).uniform(-40 * 16, 4 * 16, 400000)
    e = lib.err_step_exp2_16(_p(x), len(x))
    assert 1e-13 < e < 5.5e-12  # a real truncation error, within the documented bound


@pytest.mark.parametrize("scale", [1.0, 1e3, 1e6, 3e7])
def test_step_sincos_error_bounds(lib, scale):
    """The hot loop's sincos at UWB_FAST_POLY=2: the kernels are cos degree 6
    (1.7e-12) and sin degree 7 (3.7e-14) on |r| <= pi/16; the angle addition
    with the (cos, sin)(k pi/8) table mixes them, so cos x and sin x each stay
    within 1.75e-12 absolute -- and no better than ~1e-13 (a real truncation)."""
    x = np.random.default_rng(5).uniform(-scale, scale, 300000)
    ec = lib.err_step_sincos16(_p(x), len(x), 0)
    es = lib.err_step_sincos16(_p(x), len(x), 1)
    assert 1e-13 < ec < 1.75e-12 and 1e-13 < es < 1.75e-12, (ec, es)


@pytest.mark.parametrize("scale", [1.0, 1e3, 1e5, 3e7])
def test_step_sincos8_error_bounds(lib, scale):
    """The fast branch's phasor (step_sincos8): phase phi8 z in
    units of pi/8 reduced by one FMA, kernels with the powers of pi/8 folded in,
    result scaled by 8/pi.  Against long double at the exactly represented phase
    (pi/8) phi8 z: cos and sin each within 1.75e-12 absolute (the fits' own
    bounds, as for step_sincos_tab16), and a real truncation (> 1e-13)."""
    rng = np.random.default_rng(7)
    z = rng.uniform(0.0, 2e5, 300000)
    phi8 = rng.uniform(-1.0, 1.0, len(z)) * scale / 2e5 * 8 / np.pi
    ec = lib.err_step_sincos8(_p(phi8), _p(z), len(z), 0)
    es = lib.err_step_sincos8(_p(phi8), _p(z), len(z), 1)
    assert 1e-13 < ec < 1.75e-12 and 1e-13 < es < 1.75e-12, (ec, es)


@pytest.mark.parametrize("scale", [1.0, 1e3, 1e5, 3e7])
def test_step_sincos8q_error_bounds(lib, scale):
    """The shipping fast-branch phasor (step_sincos8q = nli_kernel.cu
    step_sincos8 at UWB_SINCOS_NOTAB=1): quarter-turn reduction, sin degree 9,
    cos degree 10, swap + sign flips.  cos and sin each within 2.75e-12
    absolute of long double (the sin fit's 2.5e-12 lands in either after the
    swap), and a real truncation (> 1e-13)."""
    rng = np.random.default_rng(7)
    z = rng.uniform(0.0, 2e5, 300000)
    phi8 = rng.uniform(-1.0, 1.0, len(z)) * scale / 2e5 * 8 / np.pi
    ec = lib.err_step_sincos8q(_p(phi8), _p(z), len(z), 0)
    es = lib.err_step_sincos8q(_p(phi8), _p(z), len(z), 1)
    assert 1e-13 < max(ec, es) and ec < 2.75e-12 and es < 2.75e-12, (ec, es)


def test_step_sincos8q_quadrants_and_device_coefficients(lib):
    """Every quarter turn (k mod 4 = 0..3, negative k included) lands on the
    right (cos, sin); the device constant banks are the header's kStepQ*."""
    phi8 = np.array([0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0, 8.0, 12.0, -4.0, -8.0, -12.0, 9.9])
    z = np.ones_like(phi8)
    ec = lib.err_step_sincos8q(_p(phi8), _p(z), len(z), 0)
    es = lib.err_step_sincos8q(_p(phi8), _p(z), len(z), 1)
    assert ec < 2.75e-12 and es < 2.75e-12, (ec, es)
    dev = open(os.path.join(ROOT, "paper_2401_18022_b200", "csrc", "nli_kernel.cu")).read()
    assert "c_s8q[4] = {kStepQS0, kStepQS1, kStepQS2, kStepQS3}" in dev
    assert "c_c8q[5] = {kStepQC0, kStepQC1, kStepQC2, kStepQC3, kStepQC4}" in dev
    assert "#define UWB_SINCOS_NOTAB 1" in dev


def test_step_sincos8_coefficients_are_the_scaled_fits():
    """kStep8* = kStep* with the powers of a = pi/8 folded in (to 1 ulp)."""
    import re
    src = open(os.path.join(ROOT, "paper_2401_18022_b200", "csrc", "uwb_devmath.cuh")).read()
    c = {m.group(1): float(m.group(2)) for m in
         re.finditer(r"constexpr double (k\w+) = ([-0-9.e+]+);", src)}
    a = np.pi / 8
    for k in range(3):
        assert c[f"kStep8S{k}"] == pytest.approx(c[f"kStepS{k}"] * a ** (2 * k + 2), rel=4e-16)
        assert c[f"kStep8C{k}"] == pytest.approx(c[f"kStepC{k}"] * a ** (2 * k + 1), rel=4e-16)
    assert c["kInvPio8"] == 8 / np.pi
    dev = open(os.path.join(ROOT, "paper_2401_18022_b200", "csrc", "nli_kernel.cu")).read()
    assert "c_s8[3] = {kStep8S0, kStep8S1, kStep8S2}" in dev
    assert "c_c8[4] = {kStep8C0, kStep8C1, kStep8C2, kInvPio8}" in dev


def test_step_kernel_coefficients_are_the_device_ones():
    """nli_kernel.cu's __constant__ banks are initialised from the header's
    kStep* constants (the ones the host restatements above use)."""
    src = open(os.path.join(ROOT, "paper_2401_18022_b200", "csrc", "nli_kernel.cu")).read()
    assert "c_e4f[4] = {kStepE0, kStepE1, kStepE2, kStepE3}" in src
    assert "c_s3f[3] = {kStepS0, kStepS1, kStepS2}" in src
    assert "c_c3f[3] = {kStepC0, kStepC1, kStepC2}" in src
    assert "#define UWB_FAST_POLY 2" in src
