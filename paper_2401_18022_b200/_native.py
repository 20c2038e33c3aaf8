"""ctypes binding of libuwbnli.so (include/uwb_nli.h, include/uwb_model.h).

The shared library is built in-tree by ``paper_2401_18022_b200.build`` (nvcc,
sm_100a).  There is no CPU fallback: if the library is missing, or no sm_100
device is visible, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UWB_LIB_PATH", os.path.join(PKG, "libuwbnli.so"))

DP = C.POINTER(C.c_double)
IP = C.POINTER(C.c_int)
U8P = C.POINTER(C.c_uint8)

UWB_OK, UWB_ERROR, UWB_CONFIG_ERROR, UWB_SOLVER_ERROR, UWB_CUDA_ERROR = 0, 1, 2, 3, 4


class UwbError(RuntimeError):
    code = UWB_ERROR


class ConfigError(UwbError):
    """uwblink::ConfigError (units.hpp:16-19): bad inputs."""
    code = UWB_CONFIG_ERROR


class SolverError(UwbError):
    """uwblink::SolverError (units.hpp:21-24): numerical breakdown."""
    code = UWB_SOLVER_ERROR


class CudaError(UwbError):
    """No usable B200 / CUDA failure.  The engine never falls back to the CPU."""
    code = UWB_CUDA_ERROR


_ERRORS = {UWB_CONFIG_ERROR: ConfigError, UWB_SOLVER_ERROR: SolverError, UWB_CUDA_ERROR: CudaError}


class Grid(C.Structure):
    _fields_ = [("n_ch", C.c_int), ("freq", DP), ("psd", DP), ("guard", U8P),
                ("spacing", C.c_double), ("bch", C.c_double), ("centre", C.c_double),
                ("half_band", C.c_double)]


class Span(C.Structure):
    _fields_ = [("steps", C.c_int), ("log_rho", DP), ("edge", DP), ("mid", DP), ("width", DP),
                ("length", C.c_double)]


class NliCfg(C.Structure):
    _fields_ = [("n_r", C.c_int), ("u1_uniform", C.c_int), ("u1_min_ratio", C.c_double),
                ("simpson", C.c_int), ("mirror_q4", C.c_int)]


class NliResultC(C.Structure):
    _fields_ = [("eta", DP), ("nli_psd", DP), ("nli_power", DP), ("quadrant", DP),
                ("skipped", U8P), ("elapsed_seconds", C.c_double)]


class Fibre(C.Structure):
    _fields_ = [("alpha", DP), ("aeff", DP), ("gamma", DP), ("raman_n", C.c_int),
                ("raman_x", DP), ("raman_y", DP), ("raman_aeff_ref", C.c_double),
                ("beta", C.c_double * 3), ("length_m", C.c_double), ("span_count", C.c_int)]


class LinkCfg(C.Structure):
    _fields_ = [("include_raman", C.c_int), ("rtol", C.c_double), ("atol", C.c_double),
                ("density", C.c_double), ("nf_db", DP), ("band", IP), ("n_bands", C.c_int),
                ("use_snr_trx", C.c_int), ("snr_trx_db", C.c_double)]


class LinkReportC(C.Structure):
    _fields_ = [("eta", DP), ("p_ase", DP), ("snr_db", DP), ("capacity", DP), ("rho_end", DP),
                ("band_power_dbm", DP), ("band_capacity", DP), ("loss_value", C.c_double),
                ("total_capacity", C.c_double), ("total_power_dbm", C.c_double),
                ("elapsed_seconds", C.c_double), ("ode_seconds", C.c_double)]


class FibreSample(C.Structure):
    _fields_ = [("alpha", DP), ("aeff", DP), ("gamma", DP), ("beta", C.c_double * 3),
                ("raman_n", C.c_int), ("raman_x", C.c_double * 16), ("raman_y", C.c_double * 16),
                ("raman_aeff_ref", C.c_double), ("dispersion", C.c_double * 4)]


# symbol -> (restype, argtypes); the test suite checks every one is exported
SIGNATURES = {
    "uwb_last_error": (C.c_char_p, []),
    "uwb_abi_version": (C.c_int, []),
    "uwb_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "uwb_ctx_destroy": (None, [C.c_void_p]),
    "uwb_ctx_create_multi": (C.c_int, [IP, C.c_int, C.POINTER(C.c_void_p)]),
    "uwb_ctx_width": (C.c_int, [C.c_void_p, IP]),
    "uwb_last_channel_work": (C.c_int, [C.c_void_p, C.c_int, DP]),
    "uwb_last_partition_stats": (C.c_int, [C.c_void_p, C.c_int, DP, DP, IP]),
    "uwb_device_info": (C.c_int, [C.c_void_p, IP, IP, IP]),
    "uwb_set_channel_subset": (C.c_int, [C.c_void_p, C.c_int, IP]),
    "uwb_all_channels_nli": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_int, C.POINTER(Span), DP,
                                       DP, C.POINTER(NliCfg), C.POINTER(NliResultC)]),
    "uwb_nli_psd_at": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_int, C.POINTER(Span), DP,
                                 C.POINTER(NliCfg), C.c_int, DP, DP, DP, DP]),
    "uwb_cfm_all_channels_nli": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_int, C.POINTER(Span),
                                           DP, DP, C.POINTER(NliResultC)]),
    "uwb_channel_nli": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.c_int, C.POINTER(Span), DP,
                                  C.c_double, C.POINTER(NliCfg), C.c_int, DP, DP]),
    "uwb_power_evolution": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.POINTER(Fibre),
                                      C.POINTER(LinkCfg), C.c_int, DP, DP, DP]),
    "uwb_evaluate_link": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.POINTER(Fibre),
                                    C.POINTER(LinkCfg), C.POINTER(NliCfg),
                                    C.POINTER(LinkReportC)]),
    "uwb_evaluate_link_prepare": (C.c_int, [C.c_void_p, C.POINTER(Grid), C.POINTER(Fibre),
                                            C.POINTER(LinkCfg), C.POINTER(NliCfg)]),
    "uwb_evaluate_link_resident": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "uwb_device_count": (C.c_int, [IP]),
    "uwb_evaluate_link_many": (C.c_int, [C.c_void_p, C.c_int, DP, DP, DP]),
    "uwb_evaluate_link_resident_noise": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "uwb_evaluate_link_resident_report": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "uwb_link_eta_buffer": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), IP]),
    "uwb_report_len": (C.c_int, [C.c_void_p, IP]),
    "uwb_resident_status": (C.c_int, [C.c_void_p]),
    "uwb_last_transfer_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_ulonglong),
                                          C.POINTER(C.c_ulonglong)]),
    "uwb_fp64_peak": (C.c_int, [C.c_void_p, DP]),
    "uwb_debug_bounds": (C.c_int, [IP, IP]),
    "uwb_set_precision": (C.c_int, [C.c_void_p, C.c_int]),
    "uwb_set_ode_stepping": (C.c_int, [C.c_void_p, C.c_int]),
    "uwb_last_launch_count": (C.c_int, [C.c_void_p]),
    "uwb_last_nli_stats": (C.c_int, [C.c_void_p, DP, DP, DP]),
    "uwb_last_nli_active": (C.c_int, [C.c_void_p, DP]),
    "uwb_last_ode_stats": (C.c_int, [C.c_void_p, DP, C.POINTER(C.c_longlong)]),
    "uwb_model_fibre": (C.c_int, [C.c_int, C.c_double, C.c_int, DP, C.c_double,
                                  C.POINTER(FibreSample)]),
    "uwb_model_grid": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, DP, U8P,
                                 IP, DP, DP]),
    "uwb_model_distance_grid": (C.c_int, [C.c_double, C.c_double, C.c_int, DP, DP, DP, IP]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libuwbnli.so once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CudaError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                        " (the engine has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int):
    if rc != UWB_OK:
        msg = _lib.uwb_last_error().decode() if _lib is not None else "uwb error"
        raise _ERRORS.get(rc, UwbError)(msg)


def dptr(a):
    return None if a is None else a.ctypes.data_as(DP)


def u8ptr(a):
    return None if a is None else a.ctypes.data_as(U8P)


def iptr(a):
    return None if a is None else a.ctypes.data_as(IP)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)
