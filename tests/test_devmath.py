"""CPU: the integrand's FP64 transcendentals (csrc/uwb_devmath.cuh are
__host__ __device__) against long-double libm.  The device versions in
nli_kernel.cu use the same coefficients; the GPU parity tests cover them end
to end."""
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
