"""The C++ drop-in (include/uwblink_b200/gn_integral.hpp) run as a reference
user would: tests/cxx/shim_parity.cpp is compiled against the UNMODIFIED
reference headers (oracle/Makefile `shim`, in the container that has
/root/reference) and restates the reference's own Catch2 assertions with
uwblink::b200::* in place of uwblink::*, comparing with the reference's CPU
result on the same inputs.  The binary travels to the GPU box prebuilt."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


def test_shim_header_is_self_contained():
    """The shim only needs uwb_nli.h + the reference headers (no torch, no
    Python): check the include list without compiling."""
    src = open(os.path.join(ROOT, "include", "uwblink_b200", "gn_integral.hpp")).read()
    incs = [l.split()[1] for l in src.splitlines() if l.startswith("#include")]
    assert '"uwb_nli.h"' in incs and '"uwblink/gn_integral.hpp"' in incs
    assert not any("torch" in i or "cuda" in i for i in incs)


@pytest.mark.gpu
def test_cxx_shim_parity():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


@pytest.mark.gpu
def test_cxx_shim_parity_multi_gpu_workers():
    """The same restated reference assertions with the drop-in's worker pool
    mapped to GPUs: UWB_DEVICES=0,0,0 gives three contexts on the one test
    GPU, so every all_channels_nli / evaluate_link with workers = 0 (all) or
    4 runs the multi-GPU split (uwb_ctx_create_multi) -- the reference's
    bit-identity across worker counts (test_gn_integral.cpp:291-300) must hold."""
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_parity not built (needs /root/reference at build time)")
    env = dict(os.environ, UWB_DEVICES="0,0,0")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


OPT = os.path.join(ROOT, "oracle", "_ref", "optimise_b200")


@pytest.mark.gpu
def test_cxx_optimise_matches_reference_optimiser():
    """Config 5 through the C++ drop-in: the reference's own L-BFGS-B driving
    device evaluations reaches the reference CPU optimiser's iterate and
    objective (uniform mode, 3 iterations, N_R=24 so the CPU side is quick)."""
    import json

    if not os.path.exists(OPT):
        pytest.skip("oracle/_ref/optimise_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([OPT, "--iters", "3", "--n-r", "24", "--density", "0.95", "--uniform", "1",
                        "--reference-iters", "3", "--devices", "1"],
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(d)
    ref = d["reference"]
    assert d["lbfgs_iterations"] == ref["lbfgs_iterations"]
    assert ref["rel_dobjective"] < 1e-9
    assert ref["max_abs_dx_db"] < 1e-6


@pytest.mark.gpu
def test_cxx_optimise_segmented_matches_reference_optimiser():
    """Config 5 exactly as BASELINE defines it: SEGMENTED mode (55 variables
    for the 589-ch plan, link_optimizer.hpp:68-102 / test_optimizer.cpp:127-133),
    bounds [-5, 5] dBm, fd step 1e-3 dB, 2 L-BFGS-B iterations at N_R = 24.
    Every cost call (value, 55-wide forward-difference batches, backtracks)
    runs on the device through the C++ drop-in; the reference CPU optimiser
    runs the same problem.  Same iteration count, objective within 1e-9,
    iterate within 1e-6 dB."""
    import json

    if not os.path.exists(OPT):
        pytest.skip("oracle/_ref/optimise_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([OPT, "--iters", "2", "--n-r", "24", "--density", "0.95", "--uniform", "0",
                        "--reference-iters", "2", "--devices", "1"],
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    print(d)
    assert "segmented" in d["config"]
    ref = d["reference"]
    assert d["lbfgs_iterations"] == ref["lbfgs_iterations"] == 2
    assert d["cost_evals"] >= 1 + 2 * 56  # value + two 55-wide gradients at least
    assert ref["rel_dobjective"] < 1e-9
    assert ref["max_abs_dx_db"] < 1e-6
