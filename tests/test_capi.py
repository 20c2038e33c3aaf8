"""CPU: the C-ABI library (libuwbnli.so) loads, exports every entry point the
headers in include/ declare, fails loudly without a GPU, and its host-side
scenario builders (include/uwb_model.h) reproduce the reference's inputs
bit-exactly (tests/golden)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2401_18022_b200 as uwb
from paper_2401_18022_b200 import _native as N
from pyoracle import Case

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in ("uwb_nli.h", "uwb_model.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(uwb_[a-z0-9_]+)\s*\(", txt):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol():
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert syms <= set(N.SIGNATURES), syms - set(N.SIGNATURES)
    assert lib.uwb_abi_version() == 1


def test_library_is_sm100a_native():
    """The fatbin carries sm_100a SASS for the integrand (no PTX JIT path)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(uwb.CudaError):
        uwb.Engine(0)
    h = ctypes.c_void_p()
    assert N.load().uwb_ctx_create(0, ctypes.byref(h)) == N.UWB_CUDA_ERROR
    assert b"no CPU fallback" in N.load().uwb_last_error()


def test_model_builders_match_reference(golden):
    from helpers import product_scenario

    for name, g in golden["grids"].items():
        case = Case.from_json(g["case"])
        grid, fibre = product_scenario(case)
        assert np.array_equal(grid.freq, g["freq"]) and np.array_equal(grid.guard, g["guard"])
        assert grid.half_band == g["half_band"]
        s = fibre.sample(grid.freq, 299792458.0 / grid.centre)
        for k in ("alpha", "aeff", "gamma"):
            assert np.array_equal(s[k], np.array(g[k])), (name, k)
        if case.betas is None:
            assert np.array_equal(s["beta"], np.array(g["betas"]))
    for z in golden["distance_grids"]:
        zg = uwb.build_distance_grid(z["length"], z["density"])
        assert np.array_equal(zg.edge, z["edge"]) and np.array_equal(zg.width, z["width"])


def test_builder_errors():
    with pytest.raises(uwb.ConfigError):
        uwb.build_distance_grid(0.0, 1.0)
    with pytest.raises(uwb.ConfigError):
        uwb.build_distance_grid(80e3, -1.0)
    with pytest.raises(uwb.ConfigError):
        uwb.make_uniform_grid(0, 100e9, 96e9, 193e12)
    with pytest.raises(uwb.ConfigError):
        uwb.make_uniform_grid(4, 100e9, 120e9, 193e12)


def test_band_plan_of_default_grid():
    g = uwb.make_default_uwb_grid()
    assert g.size() == 589 and int(g.guard.sum()) == 32
    # segment counts of make_segment_profile depend on these bands (test_optimizer.cpp:119-141)
    assert set(np.unique(g.band)) == {0, 1, 2, 3, 4, 5}
    assert g.nf_db[g.band == 3][0] == 5.0 and g.nf_db[g.band == 0][0] == 7.0
