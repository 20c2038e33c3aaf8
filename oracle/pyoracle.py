"""TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.

ctypes bindings for the two CPU checkers:

* ``Oracle``  — oracle/liboracle.so, the plain-C restatement (uwb_oracle.c);
* ``RefLib``  — oracle/_ref/libuwbref.so, the UNMODIFIED reference headers
  compiled by oracle/Makefile (present only where it was built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package
(paper_2401_18022_b200) never does.

The case builders here restate the reference's test fixtures
(tests/support/test_helpers.hpp:22-37) and the BASELINE.json configs.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libuwbref.so")

KC0 = 299792458.0
DP = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)


def _dp(a):
    return a.ctypes.data_as(DP) if a is not None else None


def _u8(a):
    return a.ctypes.data_as(U8P) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


# --------------------------------------------------------------------------
# Case description shared by both checkers (mirrors ref_harness.cpp RefCase).
# --------------------------------------------------------------------------
@dataclass
class Case:
    fibre_kind: int = 0            # 0 default_fibre, 1 flat_fibre(flat_alpha_db_km)
    flat_alpha_db_km: float = 0.2
    length_m: float = 80e3
    span_count: int = 1
    raman: int = 1
    uwb_default: int = 0
    n_ch: int = 11
    spacing: float = 100e9
    bch: float = 96e9
    centre: float = KC0 / 1550e-9
    launch_w: np.ndarray | None = None
    uniform_w: float = 1e-3
    guard: np.ndarray | None = None
    n_r: int = 150
    density: float = 1.4
    workers: int = 0
    u1_uniform: int = 0
    u1_min_ratio: float = 1e-10
    simpson: int = 0
    mirror_q4: int = 1
    betas: tuple | None = None     # None => beta_from_dispersion at lambda(centre)
    gamma: float | None = None     # explicit gamma for single-probe cases
    name: str = ""

    def to_json(self):
        d = {k: v for k, v in self.__dict__.items()}
        for k in ("launch_w", "guard"):
            if d[k] is not None:
                d[k] = np.asarray(d[k]).tolist()
        if d["betas"] is not None:
            d["betas"] = list(d["betas"])
        return d

    @classmethod
    def from_json(cls, d):
        d = dict(d)
        if d.get("launch_w") is not None:
            d["launch_w"] = np.asarray(d["launch_w"], dtype=np.float64)
        if d.get("guard") is not None:
            d["guard"] = np.asarray(d["guard"], dtype=np.uint8)
        if d.get("betas") is not None:
            d["betas"] = tuple(d["betas"])
        return cls(**d)


class _RefCase(C.Structure):
    _fields_ = [
        ("fibre_kind", C.c_int), ("flat_alpha_db_km", C.c_double), ("length_m", C.c_double),
        ("span_count", C.c_int), ("raman", C.c_int), ("uwb_default", C.c_int),
        ("n_ch", C.c_int), ("spacing", C.c_double), ("bch", C.c_double), ("centre", C.c_double),
        ("launch_w", DP), ("uniform_w", C.c_double), ("guard", U8P),
        ("n_r", C.c_int), ("density", C.c_double), ("workers", C.c_int),
        ("u1_uniform", C.c_int), ("u1_min_ratio", C.c_double), ("simpson", C.c_int),
        ("mirror_q4", C.c_int), ("betas_explicit", C.c_int),
        ("beta2", C.c_double), ("beta3", C.c_double), ("beta4", C.c_double),
    ]


def dbm_to_w(dbm):
    return 1e-3 * 10.0 ** (np.asarray(dbm, dtype=np.float64) / 10.0)


# ---------------- the reference's fixtures and the BASELINE configs ---------
def toy_case(n=3, **kw):
    """ToyCase of test_gn_integral.cpp:17-30 (flat 0.2 dB/km, toy_grid, Raman off)."""
    base = dict(fibre_kind=1, flat_alpha_db_km=0.2, raman=0, n_ch=n, spacing=12e9, bch=10e9,
                centre=193.5e12, uniform_w=1e-3, betas=(-21e-27, 0.0, 0.0), gamma=1.3e-3,
                density=0.95, name=f"toy{n}")
    base.update(kw)
    return Case(**base)


def cband11(**kw):
    """BASELINE config 1: C-band 11x96 GBd @1550 nm, 0 dBm, 80 km, Raman on."""
    base = dict(n_ch=11, spacing=100e9, bch=96e9, centre=KC0 / 1550e-9,
                uniform_w=float(dbm_to_w(0.0)), name="cband11")
    base.update(kw)
    return Case(**base)


def oband11(**kw):
    """BASELINE config 2: 11 ch straddling lambda_0 = 1302.3 nm, 2 dBm."""
    base = dict(n_ch=11, spacing=100e9, bch=96e9, centre=KC0 / 1302.3e-9,
                uniform_w=float(dbm_to_w(2.0)), name="oband11")
    base.update(kw)
    return Case(**base)


def uwb589(**kw):
    """BASELINE config 3: 589x96 GBd O->U band, 0 dBm, 80 km, Raman on."""
    base = dict(uwb_default=1, n_ch=589, uniform_w=float(dbm_to_w(0.0)), name="uwb589")
    base.update(kw)
    return Case(**base)


# --------------------------------------------------------------------------
class RefLib:
    """Reference headers compiled by oracle/Makefile (oracle/_ref/libuwbref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_phase_mismatch.restype = C.c_double
        L.ref_phase_mismatch.argtypes = [C.c_double] * 6

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _rc(self, case: Case):
        r = _RefCase()
        for name, _ in _RefCase._fields_:
            if name in ("launch_w", "guard", "betas_explicit", "beta2", "beta3", "beta4"):
                continue
            setattr(r, name, getattr(case, name))
        self._keep = []
        if case.launch_w is not None:
            a = np.ascontiguousarray(case.launch_w, dtype=np.float64)
            self._keep.append(a)
            r.launch_w = _dp(a)
        if case.guard is not None:
            gg = np.ascontiguousarray(case.guard, dtype=np.uint8)
            self._keep.append(gg)
            r.guard = _u8(gg)
        if case.betas is not None:
            r.betas_explicit = 1
            r.beta2, r.beta3, r.beta4 = case.betas
        return r

    def grid(self, case):
        n = 589 if case.uwb_default else case.n_ch
        freq, psd = np.zeros(n), np.zeros(n)
        guard = np.zeros(n, np.uint8)
        sc = np.zeros(4)
        nout = C.c_int()
        self._chk(self.lib.ref_grid(C.byref(self._rc(case)), _dp(freq), _dp(psd), _u8(guard),
                                    _dp(sc), C.byref(nout)))
        return dict(freq=freq, psd=psd, guard=guard, spacing=sc[0], bch=sc[1], centre=sc[2],
                    half_band=sc[3])

    def distance_grid(self, length_m, density):
        steps = C.c_int()
        cap = 4096
        e, m, w = np.zeros(cap + 1), np.zeros(cap), np.zeros(cap)
        self._chk(self.lib.ref_distance_grid(C.c_double(length_m), C.c_double(density), cap,
                                             _dp(e), _dp(m), _dp(w), C.byref(steps)))
        s = steps.value
        return dict(edge=e[: s + 1].copy(), mid=m[:s].copy(), width=w[:s].copy(), steps=s,
                    length=length_m)

    def power_evolution(self, case):
        n = 589 if case.uwb_default else case.n_ch
        cap = n * 4096
        lr, re = np.zeros(cap), np.zeros(n)
        steps = C.c_int()
        secs = C.c_double()
        self._chk(self.lib.ref_power_evolution(C.byref(self._rc(case)), cap, _dp(lr), _dp(re),
                                               C.byref(steps), C.byref(secs)))
        s = steps.value
        return dict(log_rho=lr[: n * s].copy(), rho_end=re, steps=s, seconds=secs.value)

    def fibre_at(self, case, freq):
        freq = np.ascontiguousarray(freq, dtype=np.float64)
        n = len(freq)
        a, ae, g = np.zeros(n), np.zeros(n), np.zeros(n)
        b = np.zeros(3)
        self._chk(self.lib.ref_fibre_at(C.byref(self._rc(case)), n, _dp(freq), _dp(a), _dp(ae),
                                        _dp(g), _dp(b)))
        return dict(alpha=a, aeff=ae, gamma=g, betas=b)

    def all_channels_nli(self, case):
        n = 589 if case.uwb_default else case.n_ch
        eta, psd, pw = np.zeros(n), np.zeros(n), np.zeros(n)
        q = np.zeros(4 * n)
        sk = np.zeros(n, np.uint8)
        tn, to = C.c_double(), C.c_double()
        self._chk(self.lib.ref_all_channels_nli(C.byref(self._rc(case)), _dp(eta), _dp(psd),
                                                _dp(pw), _dp(q), _u8(sk), C.byref(tn),
                                                C.byref(to)))
        return dict(eta=eta, nli_psd=psd, nli_power=pw, quadrant=q.reshape(n, 4), skipped=sk,
                    nli_seconds=tn.value, ode_seconds=to.value)

    def cfm_all_channels_nli(self, case):
        """cfm_all_channels_nli (gn_closed_form.hpp:70) after the reference ODE."""
        n = 589 if case.uwb_default else case.n_ch
        eta, psd, pw = np.zeros(n), np.zeros(n), np.zeros(n)
        sk = np.zeros(n, np.uint8)
        t = C.c_double()
        self._chk(self.lib.ref_cfm_all_channels_nli(C.byref(self._rc(case)), _dp(eta), _dp(psd),
                                                    _dp(pw), _u8(sk), C.byref(t)))
        return dict(eta=eta, nli_psd=psd, nli_power=pw, skipped=sk, seconds=t.value)

    def nli_psd_at(self, case, gamma, nu):
        q = np.zeros(4)
        out = C.c_double()
        self._chk(self.lib.ref_nli_psd_at(C.byref(self._rc(case)), C.c_double(gamma),
                                          C.c_double(nu), _dp(q), C.byref(out)))
        return out.value, q

    def cartesian_nli_psd(self, case, gamma, nu, n_cells):
        out = C.c_double()
        self._chk(self.lib.ref_cartesian_nli_psd(C.byref(self._rc(case)), C.c_double(gamma),
                                                 C.c_double(nu), n_cells, C.byref(out)))
        return out.value

    def phase_mismatch(self, f1, f2, fi, b):
        return self.lib.ref_phase_mismatch(f1, f2, fi, *b)

    def quadrant_limits(self, q, half_band, f):
        o = np.zeros(5)
        self._chk(self.lib.ref_quadrant_limits(q, C.c_double(half_band), C.c_double(f), _dp(o)))
        return o

    def evaluate_link(self, case):
        n = 589 if case.uwb_default else case.n_ch
        eta, pase, snr, cap = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(n)
        tot, tm = np.zeros(3), np.zeros(3)
        self._chk(self.lib.ref_evaluate_link(C.byref(self._rc(case)), _dp(eta), _dp(pase),
                                             _dp(snr), _dp(cap), _dp(tot), _dp(tm)))
        return dict(eta=eta, p_ase=pase, snr_db=snr, capacity=cap, loss=tot[0],
                    total_capacity=tot[1], total_power_dbm=tot[2], t_ode=tm[0], t_nli=tm[1],
                    t_asm=tm[2])


# --------------------------------------------------------------------------
class _OrTable(C.Structure):
    _fields_ = [("n", C.c_int), ("x", C.c_double * 96), ("y", C.c_double * 96)]


class _OrFibre(C.Structure):
    _fields_ = [
        ("lambda_c", C.c_double), ("d", C.c_double), ("s", C.c_double), ("sdot", C.c_double),
        ("order", C.c_int), ("d_table", _OrTable), ("alpha_db_km", _OrTable), ("aeff", _OrTable),
        ("n2_intercept", C.c_double), ("n2_slope", C.c_double), ("lambda_ref", C.c_double),
        ("n2_scale", C.c_double), ("raman_gain", _OrTable), ("aeff_ref", C.c_double),
        ("length_m", C.c_double), ("span_count", C.c_int),
    ]


class _OrGrid(C.Structure):
    _fields_ = [("n", C.c_int), ("freq", DP), ("psd", DP), ("guard", U8P),
                ("spacing", C.c_double), ("bch", C.c_double), ("centre", C.c_double),
                ("half_band", C.c_double)]


class _OrNliCfg(C.Structure):
    _fields_ = [("n_r", C.c_int), ("u1_uniform", C.c_int), ("u1_min_ratio", C.c_double),
                ("simpson", C.c_int), ("mirror_q4", C.c_int), ("workers", C.c_int)]


class _OrSpan(C.Structure):
    _fields_ = [("log_rho", DP), ("edge", DP), ("mid", DP), ("width", DP), ("steps", C.c_int),
                ("length", C.c_double)]


def build_oracle(quiet=True):
    """Compile oracle/liboracle.so with the committed Makefile (checker only)."""
    cmd = ["make", "-C", HERE, "oracle"]
    subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL if quiet else None)


class Oracle:
    """Plain-C restatement (oracle/uwb_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_last_error.restype = C.c_char_p
        for fn in ("or_table_at", "or_attenuation_at", "or_aeff_at", "or_gamma_at", "or_psd_at",
                   "or_phase_mismatch", "or_kernel_abs2_reference", "or_ase_power",
                   "or_raman_gain_between"):
            getattr(L, fn).restype = C.c_double
        L.or_phase_mismatch.argtypes = [C.c_double, C.c_double, C.c_double, DP]
        L.or_gamma_at.argtypes = [C.c_void_p, C.c_double]
        L.or_attenuation_at.argtypes = [C.c_void_p, C.c_double]
        L.or_aeff_at.argtypes = [C.c_void_p, C.c_double]
        L.or_psd_at.argtypes = [C.c_void_p, C.c_double]
        L.or_ase_power.argtypes = [C.c_double] * 4
        L.or_kernel_abs2_reference.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                               C.c_double, C.c_double, C.c_double]

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.or_last_error().decode())

    # ---------------- building blocks ----------------
    def fibre(self, case: Case):
        f = _OrFibre()
        if case.fibre_kind == 1:
            self.lib.or_flat_fibre(C.byref(f), C.c_double(case.flat_alpha_db_km),
                                   C.c_double(case.length_m), case.span_count)
        else:
            self.lib.or_default_fibre(C.byref(f))
        f.length_m = case.length_m
        f.span_count = case.span_count
        return f

    def grid(self, case: Case):
        g = _OrGrid()
        if case.uwb_default:
            self._chk(self.lib.or_make_default_uwb_grid(C.byref(g)))
        else:
            self._chk(self.lib.or_make_uniform_grid(C.byref(g), case.n_ch, C.c_double(case.spacing),
                                                    C.c_double(case.bch),
                                                    C.c_double(case.centre)))
        if case.guard is not None:
            for i in range(g.n):
                g.guard[i] = int(case.guard[i])
        for i in range(g.n):
            w = float(case.launch_w[i]) if case.launch_w is not None else case.uniform_w
            self.lib.or_set_channel_power(C.byref(g), i, C.c_double(w))
        return g

    @staticmethod
    def grid_arrays(g):
        n = g.n
        return dict(freq=np.ctypeslib.as_array(g.freq, (n,)).copy(),
                    psd=np.ctypeslib.as_array(g.psd, (n,)).copy(),
                    guard=np.ctypeslib.as_array(g.guard, (n,)).copy(),
                    spacing=g.spacing, bch=g.bch, centre=g.centre, half_band=g.half_band)

    def distance_grid(self, length_m, density):
        cap = 4096
        e, m, w = np.zeros(cap + 1), np.zeros(cap), np.zeros(cap)
        steps = C.c_int()
        self._chk(self.lib.or_distance_grid(C.c_double(length_m), C.c_double(density), cap,
                                            _dp(e), _dp(m), _dp(w), C.byref(steps)))
        s = steps.value
        return dict(edge=e[: s + 1].copy(), mid=m[:s].copy(), width=w[:s].copy(), steps=s,
                    length=length_m)

    def power_evolution(self, case: Case, zg=None):
        f, g = self.fibre(case), self.grid(case)
        zg = zg or self.distance_grid(case.length_m, case.density)
        n, s = g.n, zg["steps"]
        lr, re = np.zeros(n * s), np.zeros(n)
        ev = C.c_long()
        self._chk(self.lib.or_power_evolution(C.byref(f), C.byref(g), _dp(zg["mid"]), s,
                                              C.c_double(case.length_m), case.raman, _dp(lr),
                                              _dp(re), C.byref(ev)))
        return dict(log_rho=lr, rho_end=re, steps=s, rhs_evals=ev.value, zgrid=zg)

    def fibre_at(self, case: Case, freq):
        f = self.fibre(case)
        lam = KC0 / np.asarray(freq, dtype=np.float64)
        alpha = np.array([self.lib.or_attenuation_at(C.byref(f), C.c_double(x)) for x in lam])
        aeff = np.array([self.lib.or_aeff_at(C.byref(f), C.c_double(x)) for x in lam])
        gamma = np.array([self.lib.or_gamma_at(C.byref(f), C.c_double(x)) for x in lam])
        return dict(alpha=alpha, aeff=aeff, gamma=gamma, fibre=f)

    def betas(self, case: Case, centre):
        if case.betas is not None:
            return np.array(case.betas, dtype=np.float64)
        f = self.fibre(case)
        b = np.zeros(3)
        self._chk(self.lib.or_beta_from_dispersion(C.byref(f), C.c_double(KC0 / centre), _dp(b)))
        return b

    def phase_mismatch(self, f1, f2, fi, b):
        bb = np.ascontiguousarray(b, dtype=np.float64)
        return self.lib.or_phase_mismatch(f1, f2, fi, _dp(bb))

    def quadrant_limits(self, q, half_band, f):
        o = np.zeros(5)
        self._chk(self.lib.or_quadrant_limits(q, C.c_double(half_band), C.c_double(f), _dp(o)))
        return o

    # ---------------- path ----------------
    def _spans(self, tables):
        """tables: list of dict(log_rho, edge, mid, width, steps, length)."""
        arr = (_OrSpan * len(tables))()
        keep = []
        for k, t in enumerate(tables):
            parts = [np.ascontiguousarray(t[x], dtype=np.float64) for x in ("log_rho", "edge", "mid", "width")]
            keep += parts
            arr[k] = _OrSpan(_dp(parts[0]), _dp(parts[1]), _dp(parts[2]), _dp(parts[3]),
                             int(t["steps"]), float(t["length"]))
        return arr, keep

    def _cfg(self, case: Case):
        return _OrNliCfg(case.n_r, case.u1_uniform, case.u1_min_ratio, case.simpson,
                         case.mirror_q4, case.workers)

    def prepare(self, case: Case):
        """Everything the path consumes for `case`: grid, spans, betas, gamma."""
        g = self.grid(case)
        evo = self.power_evolution(case)
        zg = evo["zgrid"]
        span = dict(log_rho=evo["log_rho"], edge=zg["edge"], mid=zg["mid"], width=zg["width"],
                    steps=zg["steps"], length=case.length_m)
        ga = self.grid_arrays(g)
        gamma = self.fibre_at(case, ga["freq"])["gamma"]
        return dict(grid=g, grid_arrays=ga, spans=[span] * case.span_count,
                    betas=self.betas(case, ga["centre"]), gamma=gamma, rho_end=evo["rho_end"])

    def all_channels_nli(self, case: Case, prep=None, gamma=None):
        prep = prep or self.prepare(case)
        g = prep["grid"]
        n = g.n
        spans, keep = self._spans(prep["spans"])
        gam = np.ascontiguousarray(prep["gamma"] if gamma is None else gamma, dtype=np.float64)
        b = np.ascontiguousarray(prep["betas"], dtype=np.float64)
        eta, psd, pw, q = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(4 * n)
        sk = np.zeros(n, np.uint8)
        cfg = self._cfg(case)
        self._chk(self.lib.or_all_channels_nli(C.byref(g), spans, len(prep["spans"]), _dp(b),
                                               _dp(gam), C.byref(cfg), _dp(eta), _dp(psd),
                                               _dp(pw), _dp(q), _u8(sk)))
        return dict(eta=eta, nli_psd=psd, nli_power=pw, quadrant=q.reshape(n, 4), skipped=sk)

    def cfm_all_channels_nli(self, case: Case, prep=None):
        """or_cfm_all_channels_nli: the closed-form model (gn_closed_form.hpp:70-144)."""
        prep = prep or self.prepare(case)
        g = prep["grid"]
        n = g.n
        spans, keep = self._spans(prep["spans"])
        gam = np.ascontiguousarray(prep["gamma"], dtype=np.float64)
        b = np.ascontiguousarray(prep["betas"], dtype=np.float64)
        eta, psd, pw = np.zeros(n), np.zeros(n), np.zeros(n)
        sk = np.zeros(n, np.uint8)
        self._chk(self.lib.or_cfm_all_channels_nli(C.byref(g), spans, len(prep["spans"]), _dp(b),
                                                   _dp(gam), _dp(eta), _dp(psd), _dp(pw), _u8(sk)))
        return dict(eta=eta, nli_psd=psd, nli_power=pw, skipped=sk)

    def nli_psd_at(self, case: Case, gamma, nu, prep=None):
        prep = prep or self.prepare(case)
        spans, keep = self._spans(prep["spans"])
        b = np.ascontiguousarray(prep["betas"], dtype=np.float64)
        q = np.zeros(4)
        out = C.c_double()
        cfg = self._cfg(case)
        self._chk(self.lib.or_nli_psd_at(C.byref(prep["grid"]), spans, len(prep["spans"]), _dp(b),
                                         C.c_double(gamma), C.byref(cfg), C.c_double(nu), _dp(q),
                                         C.byref(out)))
        return out.value, q

    def cartesian_nli_psd(self, case: Case, gamma, nu, n_cells, prep=None):
        prep = prep or self.prepare(case)
        spans, keep = self._spans(prep["spans"])
        b = np.ascontiguousarray(prep["betas"], dtype=np.float64)
        out = C.c_double()
        self._chk(self.lib.or_cartesian_nli_psd(C.byref(prep["grid"]), spans, len(prep["spans"]),
                                                _dp(b), C.c_double(gamma), C.c_double(nu),
                                                n_cells, C.byref(out)))
        return out.value

    def kernel_abs2_reference(self, prep, nu1, nu2, nu_ch, phi):
        spans, keep = self._spans(prep["spans"])
        return self.lib.or_kernel_abs2_reference(C.byref(prep["grid"]), spans,
                                                 len(prep["spans"]), nu1, nu2, nu_ch, phi)

    def assemble_link_report(self, g, span_count, eta, rho_end, use_snr_trx=0, snr_trx_db=0.0):
        n = g.n
        pase, snr, cap, tot = np.zeros(n), np.zeros(n), np.zeros(n), np.zeros(3)
        self._chk(self.lib.or_assemble_link_report(
            C.byref(g), span_count, _dp(np.ascontiguousarray(eta)),
            _dp(np.ascontiguousarray(rho_end)), use_snr_trx, C.c_double(snr_trx_db), _dp(pase),
            _dp(snr), _dp(cap), _dp(tot)))
        return dict(p_ase=pase, snr_db=snr, capacity=cap, loss=tot[0], total_capacity=tot[1],
                    total_power_dbm=tot[2])

    def evaluate_link(self, case: Case):
        prep = self.prepare(case)
        nli = self.all_channels_nli(case, prep)
        rep = self.assemble_link_report(prep["grid"], case.span_count, nli["eta"],
                                        prep["rho_end"])
        rep["eta"] = nli["eta"]
        return rep
