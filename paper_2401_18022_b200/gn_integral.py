"""Python mirror of the reference's hot-path API (uwblink, gn_integral.hpp and
its inputs), running on the B200 engine through the C-ABI.

Same names, argument meaning and error behaviour as the reference:

=============================  ==============================================
this module                    reference (/root/reference/proj/include/uwblink)
=============================  ==============================================
GnSolverConfig, NliResult      gn_integral.hpp:19-37
ChannelGrid, make_uniform_grid channel_grid.hpp:15-81
make_default_uwb_grid          channel_grid.hpp:133-143 (+ default_band_plan :118)
DistanceGrid, build_distance_  distance_grid.hpp:13-73
grid
FibreSpec, default_fibre,      fibre_model.hpp:76-351 (sampled by the engine's
flat_fibre, gamma_at,          host model; flat_fibre = tests/support/
beta_from_dispersion           test_helpers.hpp:22)
PowerEvolution,                raman_power.hpp:19-122 (device ODE)
solve_power_evolution
nli_psd_at / channel_nli /     gn_integral.hpp:218-363 (device NLI)
all_channels_nli
evaluate_link, LinkReport      link_optimizer.hpp:139-245 (device ODE+NLI+SNR)
=============================  ==============================================

Errors: ConfigError / SolverError as in units.hpp:16-24; CudaError when no
B200 is usable (there is no CPU fallback).
"""
from __future__ import annotations

import enum
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import ConfigError, CudaError, SolverError  # noqa: F401

KC0 = 299792458.0


# ----------------------------------------------------------------- configs
class U1Sampling(enum.Enum):
    kLog = 0
    kUniform = 1


@dataclass
class GnSolverConfig:
    """gn_integral.hpp:19-28."""
    n_r: int = 150
    mean_step_density: float = 1.4
    workers: int = 0  # accepted for API parity; GPU count is chosen by the launcher
    u1_sampling: U1Sampling = U1Sampling.kLog
    u1_min_ratio: float = 1e-10
    simpson_channel_average: bool = False
    mirror_q4: bool = True

    def _c(self):
        return N.NliCfg(int(self.n_r), 1 if self.u1_sampling == U1Sampling.kUniform else 0,
                        float(self.u1_min_ratio), int(bool(self.simpson_channel_average)),
                        int(bool(self.mirror_q4)))


@dataclass
class NliResult:
    """gn_integral.hpp:30-37."""
    eta: np.ndarray
    nli_psd: np.ndarray
    nli_power: np.ndarray
    quadrant: np.ndarray
    skipped: np.ndarray
    elapsed_seconds: float = 0.0


@dataclass
class BetaCoefficients:
    beta2: float = 0.0
    beta3: float = 0.0
    beta4: float = 0.0

    def as_array(self):
        return np.array([self.beta2, self.beta3, self.beta4], dtype=np.float64)


@dataclass
class RamanSolveOptions:
    """raman_power.hpp:39-43."""
    include_raman: bool = True
    rtol: float = 1e-9
    atol: float = 1e-16


# ----------------------------------------------------------------- grids
@dataclass
class ChannelGrid:
    """channel_grid.hpp:15-62."""
    freq: np.ndarray
    psd: np.ndarray
    guard: np.ndarray
    spacing: float
    bch: float
    centre: float
    half_band: float
    band: np.ndarray | None = None    # BandPlan::band_of_lambda per channel
    nf_db: np.ndarray | None = None   # amplifier NF of that band

    def size(self):
        return len(self.freq)

    def channel_power(self, i):
        return self.psd[i] * self.bch

    def set_channel_power(self, i, watts):
        self.psd[i] = 0.0 if self.guard[i] else watts / self.bch

    def copy(self):
        return ChannelGrid(self.freq.copy(), self.psd.copy(), self.guard.copy(), self.spacing,
                           self.bch, self.centre, self.half_band,
                           None if self.band is None else self.band.copy(),
                           None if self.nf_db is None else self.nf_db.copy())

    def _c(self):
        self._keep = (N.f64(self.freq), N.f64(self.psd),
                      np.ascontiguousarray(self.guard, dtype=np.uint8))
        f, p, g = self._keep
        return N.Grid(len(f), N.dptr(f), N.dptr(p), N.u8ptr(g), self.spacing, self.bch,
                      self.centre, self.half_band)


def _model_grid(uwb_default, n, spacing, bch, centre):
    lib = N.load()
    if uwb_default:
        n = 589
    freq = np.zeros(n)
    guard = np.zeros(n, np.uint8)
    band = np.zeros(n, np.int32)
    nf = np.zeros(n)
    hb = np.zeros(1)
    N.check(lib.uwb_model_grid(int(uwb_default), int(n), float(spacing), float(bch),
                               float(centre), N.dptr(freq), N.u8ptr(guard), N.iptr(band),
                               N.dptr(nf), N.dptr(hb)))
    return freq, guard, band, nf, float(hb[0])


def make_uniform_grid(n_channels, spacing_hz, bch_hz, centre_hz) -> ChannelGrid:
    """channel_grid.hpp:64-81 (validation as ChannelGrid::validate :44-61)."""
    if n_channels <= 0:
        raise ConfigError("need at least one channel")
    if not (spacing_hz > 0 and bch_hz > 0):
        raise ConfigError("grid spacing and width must be > 0")
    if bch_hz > spacing_hz + 1e-9:
        raise ConfigError("channel width exceeds spacing")
    freq, guard, band, nf, hb = _model_grid(0, n_channels, spacing_hz, bch_hz, centre_hz)
    return ChannelGrid(freq, np.zeros(n_channels), guard, float(spacing_hz), float(bch_hz),
                       float(centre_hz), hb, band, nf)


def make_default_uwb_grid(symbol_rate_hz=96e9, spacing_hz=100e9, n_channels=589) -> ChannelGrid:
    """channel_grid.hpp:133-143 on default_band_plan() (the BASELINE 589-ch plan)."""
    if (symbol_rate_hz, spacing_hz, n_channels) != (96e9, 100e9, 589):
        raise ConfigError("only the default 589 x 96 GBd / 100 GHz plan is built in")
    freq, guard, band, nf, hb = _model_grid(1, 589, 100e9, 96e9, KC0 / 1438e-9)
    return ChannelGrid(freq, np.zeros(589), guard, 100e9, 96e9, KC0 / 1438e-9, hb, band, nf)


def set_uniform_launch(g: ChannelGrid, power_per_channel_w: float):
    """channel_grid.hpp:83-85."""
    g.psd = np.where(g.guard != 0, 0.0, power_per_channel_w / g.bch)


def set_launch(g: ChannelGrid, power_w: np.ndarray):
    g.psd = np.where(g.guard != 0, 0.0, np.asarray(power_w, dtype=np.float64) / g.bch)


@dataclass
class DistanceGrid:
    """distance_grid.hpp:13-20."""
    edge: np.ndarray
    mid: np.ndarray
    width: np.ndarray
    length: float
    density: float

    def steps(self):
        return len(self.mid)


def build_distance_grid(length_m, density_per_km) -> DistanceGrid:
    """distance_grid.hpp:23-73."""
    lib = N.load()
    cap = 8192
    e, m, w = np.zeros(cap + 1), np.zeros(cap), np.zeros(cap)
    steps = N.C.c_int()
    N.check(lib.uwb_model_distance_grid(float(length_m), float(density_per_km), cap, N.dptr(e),
                                        N.dptr(m), N.dptr(w), N.C.byref(steps)))
    s = steps.value
    if s > cap:
        raise ConfigError("distance grid too large")
    return DistanceGrid(e[: s + 1].copy(), m[:s].copy(), w[:s].copy(), float(length_m),
                        s / length_m * 1e3)


# ----------------------------------------------------------------- fibre
@dataclass
class FibreSpec:
    """The built-in fibre (fibre_model.hpp:287-351) or the test suite's flat
    variant; sampled per channel by the engine's host model."""
    length_m: float = 80e3
    span_count: int = 1
    flat_alpha_db_km: float | None = None  # None = default wavelength-dependent loss
    # RamanGainCurve override (fibre_model.hpp:213-219): gain table x [Hz],
    # y [1/(W m)]; None = the built-in triangle (:344-347)
    raman_x: object = None
    raman_y: object = None

    def sample(self, freq, lambda_beta):
        """Per-channel alpha / A_eff / gamma, the Raman table and beta at
        lambda_beta, from the engine's host fibre model.  A pure function of
        the spec and the frequencies: memoised (the optimisation loop and
        repeated evaluate_link calls sample the same grid)."""
        freq = N.f64(freq)
        key = (self.length_m, self.span_count, self.flat_alpha_db_km,
               None if self.raman_x is None else N.f64(self.raman_x).tobytes(),
               None if self.raman_y is None else N.f64(self.raman_y).tobytes(),
               float(lambda_beta), freq.tobytes())
        hit = _SAMPLE_CACHE.get(key)
        if hit is None:
            hit = self._sample(freq, lambda_beta)
            if len(_SAMPLE_CACHE) >= 16:
                _SAMPLE_CACHE.pop(next(iter(_SAMPLE_CACHE)))
            _SAMPLE_CACHE[key] = hit
        # copies: a caller may modify what it gets back
        return {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in hit.items()}

    def _sample(self, freq, lambda_beta):
        lib = N.load()
        n = len(freq)
        alpha, aeff, gamma = np.zeros(n), np.zeros(n), np.zeros(n)
        s = N.FibreSample()
        s.alpha, s.aeff, s.gamma = N.dptr(alpha), N.dptr(aeff), N.dptr(gamma)
        kind = 0 if self.flat_alpha_db_km is None else 1
        N.check(lib.uwb_model_fibre(kind, float(self.flat_alpha_db_km or 0.0), n, N.dptr(freq),
                                    float(lambda_beta), N.C.byref(s)))
        rn = s.raman_n
        rx, ry = np.array(s.raman_x[:rn]), np.array(s.raman_y[:rn])
        if self.raman_x is not None:
            rx, ry = N.f64(self.raman_x), N.f64(self.raman_y)
            if rx.size < 2 or rx.size != ry.size or np.any(np.diff(rx) <= 0):
                raise ConfigError("raman gain: table must ascend and have >= 2 rows")
        return dict(alpha=alpha, aeff=aeff, gamma=gamma, beta=np.array(s.beta[:]),
                    raman_x=rx, raman_y=ry,
                    raman_aeff_ref=s.raman_aeff_ref, dispersion=np.array(s.dispersion[:]))


_SAMPLE_CACHE: dict = {}


def default_fibre() -> FibreSpec:
    return FibreSpec()


def flat_fibre(alpha_db_km, length_m, spans=1) -> FibreSpec:
    """uwtest::flat_fibre (tests/support/test_helpers.hpp:22-29)."""
    return FibreSpec(length_m=length_m, span_count=spans, flat_alpha_db_km=alpha_db_km)


def beta_from_dispersion(fibre: FibreSpec, lambda_m: float) -> BetaCoefficients:
    """fibre_model.hpp:76-89 on the fibre's quadratic D fit."""
    b = fibre.sample(np.zeros(0), lambda_m)["beta"]
    return BetaCoefficients(*b)


def gamma_at(fibre: FibreSpec, lambda_m) -> np.ndarray:
    """fibre_model.hpp:264-267 (vectorised over wavelengths)."""
    lam = np.atleast_1d(np.asarray(lambda_m, dtype=np.float64))
    return fibre.sample(KC0 / lam, 1.5e-6)["gamma"]


# ----------------------------------------------------------------- engine
class Engine:
    """One CUDA context (device buffers resident in HBM across calls).

    ``devices=[d0, d1, ...]`` makes a multi-GPU context (uwb_ctx_create_multi):
    the reference's worker pool (GnSolverConfig.workers) with GPUs as the
    workers -- channels split over the devices for single evaluations,
    whole evaluations dealt for batches, results bit-identical to one GPU.
    """

    def __init__(self, device: int | None = None, devices=None):
        self.lib = N.load()
        h = N.C.c_void_p()
        if devices is not None:
            dv = np.ascontiguousarray(devices, dtype=np.int32)
            if dv.size < 1:
                raise ConfigError("need at least one device")
            self.device = int(dv[0])
            self.devices = [int(x) for x in dv]
            N.check(self.lib.uwb_ctx_create_multi(N.iptr(dv), int(dv.size), N.C.byref(h)))
        else:
            if device is None:
                device = int(os.environ.get("LOCAL_RANK", "0")) if "UWB_DEVICE" not in os.environ \
                    else int(os.environ["UWB_DEVICE"])
            self.device = device
            self.devices = [int(device)]
            N.check(self.lib.uwb_ctx_create(int(device), N.C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.lib.uwb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_channel_subset(self, channels):
        ch = np.ascontiguousarray(channels if channels is not None else [], dtype=np.int32)
        N.check(self.lib.uwb_set_channel_subset(self.h, len(ch), N.iptr(ch)))

    def width(self):
        """Devices behind this context."""
        n = N.C.c_int()
        N.check(self.lib.uwb_ctx_width(self.h, N.C.byref(n)))
        return n.value

    def last_channel_work(self, n_ch):
        """|K|^2 evaluations per channel of the last NLI (the split's cost model)."""
        w = np.zeros(n_ch)
        N.check(self.lib.uwb_last_channel_work(self.h, int(n_ch), N.dptr(w)))
        return w

    def last_partition_stats(self):
        """Per device of the last split evaluation: integrand / ODE ms and the
        first channel of its range."""
        n = self.width()
        a, b = np.zeros(n), np.zeros(n)
        f = np.zeros(n, np.int32)
        N.check(self.lib.uwb_last_partition_stats(self.h, n, N.dptr(a), N.dptr(b), N.iptr(f)))
        return dict(nli_ms=a.tolist(), ode_ms=b.tolist(), first_channel=f.tolist())

    def device_info(self):
        a, b, c = N.C.c_int(), N.C.c_int(), N.C.c_int()
        N.check(self.lib.uwb_device_info(self.h, N.C.byref(a), N.C.byref(b), N.C.byref(c)))
        return dict(sm_count=a.value, cc=(b.value, c.value))

    def last_launches(self):
        return self.lib.uwb_last_launch_count(self.h)

    def last_transfer_bytes(self):
        a, b = N.C.c_ulonglong(), N.C.c_ulonglong()
        N.check(self.lib.uwb_last_transfer_bytes(self.h, N.C.byref(a), N.C.byref(b)))
        return a.value, b.value

    def set_precision(self, mode: str):
        """Integrand step arithmetic for subsequent calls: "fp64" (default,
        the reference's arithmetic) or "mixed" (compensated FP32; see
        include/uwb_nli.h uwb_set_precision).  An extension: the reference
        has no such knob."""
        modes = {"fp64": 0, "mixed": 1}
        if mode not in modes:
            raise ConfigError(f"set_precision: unknown mode {mode!r}")
        N.check(self.lib.uwb_set_precision(self.h, modes[mode]))
        self.precision = mode

    def set_ode_stepping(self, mode: str):
        """Raman ODE step-size policy for subsequent calls: "restart" (default,
        the reference's restart at every midpoint) or "continuous" (the step
        size carries across midpoints; include/uwb_nli.h)."""
        modes = {"restart": 0, "continuous": 1}
        if mode not in modes:
            raise ConfigError(f"set_ode_stepping: unknown mode {mode!r}")
        N.check(self.lib.uwb_set_ode_stepping(self.h, modes[mode]))
        self.ode_stepping = mode

    def fp64_peak_tflops(self):
        t = N.C.c_double()
        N.check(self.lib.uwb_fp64_peak(self.h, N.C.byref(t)))
        return t.value

    def last_ode_stats(self):
        """Raman ODE stage of the last prepared/resident evaluation:
        {"ode_ms", "rhs_evals"} (synchronises)."""
        a, b = N.C.c_double(), N.C.c_longlong()
        N.check(self.lib.uwb_last_ode_stats(self.h, N.C.byref(a), N.C.byref(b)))
        return {"ode_ms": a.value, "rhs_evals": b.value}

    def last_nli_stats(self):
        a, b, c = N.C.c_double(), N.C.c_double(), N.C.c_double()
        N.check(self.lib.uwb_last_nli_stats(self.h, N.C.byref(a), N.C.byref(b), N.C.byref(c)))
        d = N.C.c_double()
        N.check(self.lib.uwb_last_nli_active(self.h, N.C.byref(d)))
        return dict(kernel_ms=a.value, inner_steps=b.value, evaluated_points=c.value,
                    active_points=d.value)


_engine: Engine | None = None


def get_engine() -> Engine:
    global _engine
    if _engine is None:
        _engine = Engine()
    return _engine


# ----------------------------------------------------------------- power evolution
@dataclass
class PowerEvolution:
    """raman_power.hpp:19-37 (log_rho layout ch*steps+m)."""
    grid: DistanceGrid
    freq: np.ndarray
    launch: np.ndarray
    log_rho: np.ndarray
    rho_end: np.ndarray
    spacing: float

    def channels(self):
        return len(self.freq)

    def steps(self):
        return self.grid.steps()

    def _c(self):
        self._keep = (N.f64(self.log_rho), N.f64(self.grid.edge), N.f64(self.grid.mid),
                      N.f64(self.grid.width))
        lr, e, m, w = self._keep
        return N.Span(self.grid.steps(), N.dptr(lr), N.dptr(e), N.dptr(m), N.dptr(w),
                      float(self.grid.length))


def _fibre_c(fibre: FibreSpec, grid: ChannelGrid):
    s = fibre.sample(grid.freq, KC0 / grid.centre)
    keep = [N.f64(s["alpha"]), N.f64(s["aeff"]), N.f64(s["gamma"]), N.f64(s["raman_x"]),
            N.f64(s["raman_y"])]
    fc = N.Fibre()
    fc.alpha, fc.aeff, fc.gamma = N.dptr(keep[0]), N.dptr(keep[1]), N.dptr(keep[2])
    fc.raman_n = len(keep[3])
    fc.raman_x, fc.raman_y = N.dptr(keep[3]), N.dptr(keep[4])
    fc.raman_aeff_ref = s["raman_aeff_ref"]
    for i in range(3):
        fc.beta[i] = s["beta"][i]
    fc.length_m = fibre.length_m
    fc.span_count = fibre.span_count
    return fc, keep, s


def solve_power_evolution(fibre: FibreSpec, grid: ChannelGrid, zgrid: DistanceGrid,
                          opt: RamanSolveOptions = RamanSolveOptions(), engine=None) -> PowerEvolution:
    """raman_power.hpp:52-122, on the device (raman_ode.cu)."""
    eng = engine or get_engine()
    n, s = grid.size(), zgrid.steps()
    fc, keep, _ = _fibre_c(fibre, grid)
    lk = N.LinkCfg(int(bool(opt.include_raman)), float(opt.rtol), float(opt.atol), 1.0)
    g = grid._c()
    mid = N.f64(zgrid.mid)
    lr, re = np.zeros(n * s), np.zeros(n)
    N.check(eng.lib.uwb_power_evolution(eng.h, N.C.byref(g), N.C.byref(fc), N.C.byref(lk), s,
                                        N.dptr(mid), N.dptr(lr), N.dptr(re)))
    return PowerEvolution(zgrid, grid.freq.copy(), grid.psd * grid.bch, lr, re, grid.spacing)


# ----------------------------------------------------------------- the path
def _spans_c(spans):
    arr = (N.Span * max(len(spans), 1))()
    for k, s in enumerate(spans):
        arr[k] = s._c()
    return arr


def nli_psd_at(grid: ChannelGrid, spans, betas: BetaCoefficients, gamma_probe, cfg: GnSolverConfig,
               nu_probe, quadrant_diag=None, engine=None):
    """gn_integral.hpp:218-313.  `nu_probe`/`gamma_probe` may be arrays (one
    launch evaluates all probes); returns a float for scalar input."""
    eng = engine or get_engine()
    nu = np.atleast_1d(N.f64(nu_probe))
    gam = np.broadcast_to(N.f64(gamma_probe), nu.shape).copy()
    if not spans:
        raise ConfigError("nli_psd_at: need at least one span")
    for s in spans:
        if s.channels() != grid.size():
            raise ConfigError("nli_psd_at: span evolution does not match the channel grid")
    out, quad = np.zeros(len(nu)), np.zeros(4 * len(nu))
    g, sp, c = grid._c(), _spans_c(spans), cfg._c()
    b = betas.as_array()
    N.check(eng.lib.uwb_nli_psd_at(eng.h, N.C.byref(g), len(spans), sp, N.dptr(b), N.C.byref(c),
                                   len(nu), N.dptr(nu), N.dptr(gam), N.dptr(out), N.dptr(quad)))
    if quadrant_diag is not None:
        quadrant_diag[:] = quad[:4] if np.ndim(nu_probe) == 0 else quad.reshape(-1, 4)
    return float(out[0]) if np.ndim(nu_probe) == 0 else out


def channel_nli(grid: ChannelGrid, spans, betas: BetaCoefficients, gamma_ch, cfg: GnSolverConfig,
                ch, quadrant_diag=None, engine=None):
    """gn_integral.hpp:316-329."""
    eng = engine or get_engine()
    for s in spans:
        if s.channels() != grid.size():
            raise ConfigError("nli_psd_at: span evolution does not match the channel grid")
    g, sp, c = grid._c(), _spans_c(spans), cfg._c()
    b = betas.as_array()
    out, quad = N.C.c_double(), np.zeros(4)
    N.check(eng.lib.uwb_channel_nli(eng.h, N.C.byref(g), len(spans), sp, N.dptr(b),
                                    float(gamma_ch), N.C.byref(c), int(ch), N.C.byref(out),
                                    N.dptr(quad)))
    if quadrant_diag is not None:
        quadrant_diag[:] = quad
    return out.value


def all_channels_nli(grid: ChannelGrid, spans, betas: BetaCoefficients, fibre, cfg: GnSolverConfig,
                     engine=None, gamma=None) -> NliResult:
    """gn_integral.hpp:334-363.  `fibre` supplies gamma_at per channel (:353);
    pass `gamma` to override with explicit per-channel values."""
    eng = engine or get_engine()
    n = grid.size()
    if spans:
        for s in spans:
            if s.channels() != n:
                raise ConfigError("nli_psd_at: span evolution does not match the channel grid")
    gam = N.f64(gamma) if gamma is not None else fibre.sample(grid.freq, 1.5e-6)["gamma"]
    eta, psd, pw, quad = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(4 * n)
    sk = np.zeros(n, np.uint8)
    res = N.NliResultC(N.dptr(eta), N.dptr(psd), N.dptr(pw), N.dptr(quad), N.u8ptr(sk), 0.0)
    g, sp, c = grid._c(), _spans_c(spans or []), cfg._c()
    b = betas.as_array()
    N.check(eng.lib.uwb_all_channels_nli(eng.h, N.C.byref(g), len(spans or []), sp, N.dptr(b),
                                         N.dptr(gam), N.C.byref(c), N.C.byref(res)))
    return NliResult(eta, psd, pw, quad.reshape(n, 4), sk, res.elapsed_seconds)


def cfm_all_channels_nli(grid: ChannelGrid, spans, betas: BetaCoefficients, fibre,
                         engine=None, gamma=None) -> NliResult:
    """Closed-form SPM + XPM model, gn_closed_form.hpp:70-144 (on the device).
    `fibre` supplies gamma_at per channel (:84-87); `gamma` overrides it.
    The quadrant array is zeros, like the reference's."""
    eng = engine or get_engine()
    n = grid.size()
    if not spans:
        raise ConfigError("cfm: need at least one span")
    for s in spans:
        if s.channels() != n:
            raise ConfigError("cfm: span evolution does not match the grid")
    gam = N.f64(gamma) if gamma is not None else fibre.sample(grid.freq, 1.5e-6)["gamma"]
    eta, psd, pw, quad = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(4 * n)
    sk = np.zeros(n, np.uint8)
    res = N.NliResultC(N.dptr(eta), N.dptr(psd), N.dptr(pw), N.dptr(quad), N.u8ptr(sk), 0.0)
    g, sp = grid._c(), _spans_c(spans)
    b = betas.as_array()
    N.check(eng.lib.uwb_cfm_all_channels_nli(eng.h, N.C.byref(g), len(spans), sp, N.dptr(b),
                                             N.dptr(gam), N.C.byref(res)))
    return NliResult(eta, psd, pw, quad.reshape(n, 4), sk, res.elapsed_seconds)


# ----------------------------------------------------------------- full SNR evaluation
@dataclass
class LinkConfig:
    """link_optimizer.hpp:159-171 (the fields evaluate_link reads)."""
    gn: GnSolverConfig = field(default_factory=GnSolverConfig)
    raman: RamanSolveOptions = field(default_factory=RamanSolveOptions)
    snr_trx_db: float = 0.0
    use_snr_trx: bool = False


@dataclass
class LinkReport:
    """link_optimizer.hpp:139-157 (per-channel arrays)."""
    eta: np.ndarray
    p_ase: np.ndarray
    snr_db: np.ndarray
    capacity: np.ndarray
    rho_end: np.ndarray
    band_power_dbm: np.ndarray
    band_capacity: np.ndarray
    total_power_dbm: float
    total_capacity: float
    loss_value: float
    elapsed_seconds: float
    ode_seconds: float


N_BANDS = 6


def _link_c(grid: ChannelGrid, cfg: LinkConfig, gn: GnSolverConfig):
    nf = N.f64(grid.nf_db if grid.nf_db is not None else np.full(grid.size(), 5.0))
    band = np.ascontiguousarray(grid.band if grid.band is not None else np.full(grid.size(), -1),
                                dtype=np.int32)
    lk = N.LinkCfg(int(bool(cfg.raman.include_raman)), float(cfg.raman.rtol),
                   float(cfg.raman.atol), float(gn.mean_step_density), N.dptr(nf), N.iptr(band),
                   N_BANDS, int(bool(cfg.use_snr_trx)), float(cfg.snr_trx_db))
    return lk, (nf, band)


def evaluate_link(fibre: FibreSpec, grid: ChannelGrid, cfg: LinkConfig, gn: GnSolverConfig | None = None,
                  engine=None) -> LinkReport:
    """link_optimizer.hpp:241-245: distance grid + device ODE + device NLI +
    device assemble_link_report, host buffers in and out."""
    eng = engine or get_engine()
    gn = gn or cfg.gn
    n = grid.size()
    fc, keep, _ = _fibre_c(fibre, grid)
    lk, keep2 = _link_c(grid, cfg, gn)
    g, c = grid._c(), gn._c()
    out = {k: np.zeros(n) for k in ("eta", "p_ase", "snr_db", "capacity", "rho_end")}
    bp, bc = np.zeros(N_BANDS), np.zeros(N_BANDS)
    rep = N.LinkReportC(*(N.dptr(out[k]) for k in ("eta", "p_ase", "snr_db", "capacity", "rho_end")),
                        N.dptr(bp), N.dptr(bc))
    N.check(eng.lib.uwb_evaluate_link(eng.h, N.C.byref(g), N.C.byref(fc), N.C.byref(lk),
                                      N.C.byref(c), N.C.byref(rep)))
    return LinkReport(out["eta"], out["p_ase"], out["snr_db"], out["capacity"], out["rho_end"], bp,
                      bc, rep.total_power_dbm, rep.total_capacity, rep.loss_value,
                      rep.elapsed_seconds, rep.ode_seconds)


class ResidentLink:
    """Device-resident full SNR evaluation for repeated calls (the optimiser
    loop and the bench `value` leg): static state uploaded once; each call
    takes launch PSDs already in device memory and leaves the report there."""

    def __init__(self, fibre: FibreSpec, grid: ChannelGrid, cfg: LinkConfig,
                 gn: GnSolverConfig | None = None, engine=None):
        self.eng = engine or get_engine()
        gn = gn or cfg.gn
        self.n = grid.size()
        fc, self._keep, _ = _fibre_c(fibre, grid)
        lk, self._keep2 = _link_c(grid, cfg, gn)
        g, c = grid._c(), gn._c()
        self._g = g
        N.check(self.eng.lib.uwb_evaluate_link_prepare(self.eng.h, N.C.byref(g), N.C.byref(fc),
                                                       N.C.byref(lk), N.C.byref(c)))
        rl = N.C.c_int()
        N.check(self.eng.lib.uwb_report_len(self.eng.h, N.C.byref(rl)))
        self.report_len = rl.value  # 4 n + 3 + 2 n_bands (include/uwb_nli.h)

    def run(self, psd_dev_ptr: int, report_dev_ptr: int, stream_ptr: int = 0):
        """ODE + NLI + SNR assembly for the launch PSD at psd_dev_ptr."""
        N.check(self.eng.lib.uwb_evaluate_link_resident(self.eng.h, N.C.c_void_p(psd_dev_ptr),
                                                        N.C.c_void_p(report_dev_ptr),
                                                        N.C.c_void_p(stream_ptr)))

    def run_many(self, psd: np.ndarray, reports: bool = False):
        """uwb_evaluate_link_many: n_eval evaluations back to back on the device
        (the optimiser's value + finite-difference gradient calls) with one
        upload and one download.  psd [n_eval, n_ch] host launch PSDs (W/Hz) ->
        loss [n_eval] (and reports [n_eval, report_len] when asked)."""
        psd = np.ascontiguousarray(psd, dtype=np.float64).reshape(-1, self.n)
        ne = psd.shape[0]
        loss = np.zeros(ne)
        rep = np.zeros((ne, self.report_len)) if reports else None
        N.check(self.eng.lib.uwb_evaluate_link_many(self.eng.h, ne, N.dptr(psd), N.dptr(loss),
                                                    N.dptr(rep) if rep is not None else None))
        return (loss, rep) if reports else loss

    # split form for multi-GPU: noise on this rank's channels, all-reduce eta, report
    def run_noise(self, psd_dev_ptr: int, stream_ptr: int = 0):
        N.check(self.eng.lib.uwb_evaluate_link_resident_noise(
            self.eng.h, N.C.c_void_p(psd_dev_ptr), N.C.c_void_p(stream_ptr)))

    def run_report(self, report_dev_ptr: int, stream_ptr: int = 0):
        N.check(self.eng.lib.uwb_evaluate_link_resident_report(
            self.eng.h, N.C.c_void_p(report_dev_ptr), N.C.c_void_p(stream_ptr)))

    def eta_buffer(self):
        p, n = N.C.c_void_p(), N.C.c_int()
        N.check(self.eng.lib.uwb_link_eta_buffer(self.eng.h, N.C.byref(p), N.C.byref(n)))
        return p.value, n.value

    def check_status(self):
        N.check(self.eng.lib.uwb_resident_status(self.eng.h))
