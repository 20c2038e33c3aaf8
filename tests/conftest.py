import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libuwbnli.so on cuda:0)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_cfm():
    with open(os.path.join(ROOT, "tests", "golden", "golden_cfm.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_stress():
    with open(os.path.join(ROOT, "tests", "golden", "golden_stress.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle, build_oracle

    build_oracle()
    return Oracle()


@pytest.fixture(scope="session")
def engine():
    import paper_2401_18022_b200 as uwb

    eng = uwb.Engine(0)
    yield eng
    eng.close()


@pytest.fixture(scope="session", autouse=True)
def _bounds_checked_build_stays_clean():
    """With a bounds-checked library (UWB_LIB_PATH=scratch/v/bounds.so, built
    with -DUWB_BOUNDS_CHECK=1 -- the stand-in for compute-sanitizer, which the
    GPU pool does not allow), every index check the kernels ran during the
    session must have passed."""
    yield
    import sys as _sys
    N = _sys.modules.get("paper_2401_18022_b200._native")
    if N is None or N._lib is None:
        return
    import ctypes as C
    a, b = C.c_int(), C.c_int()
    N._lib.uwb_debug_bounds(C.byref(a), C.byref(b))
    assert a.value in (0, -1) and b.value in (0, -1), \
        f"bounds check failed: integrand line {a.value}, ODE line {b.value}"
