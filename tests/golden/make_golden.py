"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/libuwbref.so, compiled from /root/reference headers by
oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The JSON files it writes are committed; nothing on the GPU box reads
/root/reference.  Floats are stored with repr() (exact round trip).
"""
from __future__ import annotations

import json
import os
import platform
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import RefLib, cband11, oband11, toy_case, uwb589, dbm_to_w, KC0  # noqa: E402


def _tolist(x):
    if isinstance(x, np.ndarray):
        return x.tolist()
    if isinstance(x, (np.floating,)):
        return float(x)
    if isinstance(x, (np.integer,)):
        return int(x)
    if isinstance(x, dict):
        return {k: _tolist(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_tolist(v) for v in x]
    return x


def provenance():
    cxx = subprocess.run(["g++", "--version"], capture_output=True, text=True).stdout.splitlines()[0]
    libc = " ".join(platform.libc_ver())
    return dict(generator="tests/golden/make_golden.py", reference="/root/reference/proj/include/uwblink",
                harness="oracle/ref_harness.cpp", cxx=cxx, flags="-std=c++20 -O3 -fno-math-errno",
                libc=libc)


def random_launch_589(seed=20240131):
    """Parity input for config 5: per-channel launch powers U[-5, 5] dBm."""
    rng = np.random.default_rng(seed)
    return dbm_to_w(rng.uniform(-5.0, 5.0, 589))


def nli_cases():
    """(case, with_tables) pairs whose all_channels_nli outputs are pinned."""
    return [
        (cband11(), True),
        (oband11(), True),
        (oband11(simpson=1, name="oband11_simpson"), False),
        (cband11(n_r=40, name="cband11_nr40"), False),
        (cband11(n_r=30, u1_uniform=1, name="cband11_uniform"), False),
        (cband11(n_r=24, mirror_q4=0, name="cband11_direct_q4"), False),
        (toy_case(5, n_r=64, workers=1, name="toy5_nr64"), True),
        (toy_case(5, n_r=64, workers=1, guard=np.array([0, 0, 1, 0, 0], np.uint8),
                  name="toy5_guard"), False),
        (toy_case(5, n_r=64, workers=1, simpson=1, name="toy5_simpson"), False),
        (toy_case(5, n_r=64, workers=1, uniform_w=2e-3, name="toy5_2mw"), False),
        (toy_case(3, n_r=24, span_count=3, length_m=50e3, name="toy3_3span"), True),
        (cband11(n_r=40, density=0.05, name="cband11_uniform_z"), True),
        (uwb589(n_r=150, density=1.4, name="uwb589_150_1.4"), False),
        (uwb589(n_r=75, density=0.95, name="uwb589_75_0.95"), False),
        (uwb589(n_r=40, density=0.95, launch_w=random_launch_589(), name="uwb589_random_launch"),
         False),
    ]


def main():
    R = RefLib()
    out = dict(provenance=provenance())

    # ---- kernel-level pins from test_gn_integral.cpp:34-163 ----
    b = (-1.9474701795517992e-26, 9.84268860900867e-41, -3.036944725627878e-55)
    rng = np.random.default_rng(7)
    pm = []
    for _ in range(64):
        f1, f2, fi = rng.uniform(-3e12, 3e12, 3)
        pm.append([f1, f2, fi, R.phase_mismatch(f1, f2, fi, b), R.phase_mismatch(f2, f1, fi, b)])
    out["phase_mismatch"] = dict(betas=b, rows=pm,
                                 pinned=[1e11, 1e11, 0.0, -1.9474701795517992e-26,
                                         R.phase_mismatch(1e11, 1e11, 0.0,
                                                          (-1.9474701795517992e-26, 0, 0))])
    ql = []
    for q in (1, 2, 3, 4):
        for f in (0.0, 0.3e12, -0.15e12, 0.5e12, 1e12):
            ql.append([q, 1e12, f, R.quadrant_limits(q, 1e12, f).tolist()])
    out["quadrant_limits"] = ql

    # ---- inputs either side of the path ----
    out["distance_grids"] = [dict(density=d, **R.distance_grid(L, d))
                             for L, d in [(80e3, 0.5), (80e3, 0.95), (80e3, 1.4), (80e3, 2.0),
                                          (50e3, 0.95), (80e3, 0.05), (100e3, 1.0)]]
    grids = {}
    for c in (cband11(), oband11(), uwb589(), toy_case(3), toy_case(5)):
        g = R.grid(c)
        f = R.fibre_at(c, g["freq"])
        grids[c.name] = dict(case=c.to_json(), **g, alpha=f["alpha"], aeff=f["aeff"],
                             gamma=f["gamma"], betas=f["betas"])
    out["grids"] = grids

    evos = {}
    for c in (cband11(), oband11(), toy_case(3), toy_case(3, raman=0, fibre_kind=1,
                                                               flat_alpha_db_km=0.0,
                                                               name="toy3_lossless"),
              uwb589(), uwb589(uniform_w=float(dbm_to_w(2.0)), name="uwb589_2dbm"),
              uwb589(launch_w=random_launch_589(), name="uwb589_random_launch")):
        e = R.power_evolution(c)
        lr = e["log_rho"]
        rec = dict(case=c.to_json(), steps=e["steps"], rho_end=e["rho_end"],
                   log_rho_sum=float(np.sum(lr)), log_rho_min=float(lr.min()),
                   log_rho_samples=[[int(i), float(lr[i])] for i in
                                    np.linspace(0, lr.size - 1, 64).astype(int)])
        if lr.size <= 20000:
            rec["log_rho"] = lr
        evos[c.name] = rec
    out["power_evolution"] = evos

    # ---- the path ----
    nli = {}
    for c, tables in nli_cases():
        r = R.all_channels_nli(c)
        rec = dict(case=c.to_json(), eta=r["eta"], nli_psd=r["nli_psd"], nli_power=r["nli_power"],
                   quadrant=r["quadrant"], skipped=r["skipped"], ref_nli_seconds=r["nli_seconds"],
                   ref_ode_seconds=r["ode_seconds"])
        nli[c.name] = rec
        print(f"{c.name}: nli {r['nli_seconds']:.2f}s ode {r['ode_seconds']:.3f}s", flush=True)
    out["all_channels_nli"] = nli

    # single-probe + Cartesian pins (test_gn_integral.cpp:226-263, acceptance C1)
    probes = []
    toy = toy_case(3, n_r=150)
    for ch_nu in (193.5e12, 193.5e12 - 12e9, 193.5e12 + 12e9):
        v, q = R.nli_psd_at(toy, 1.3e-3, ch_nu)
        probes.append(dict(case=toy.to_json(), gamma=1.3e-3, nu=ch_nu, value=v, quad=q,
                           cartesian600=R.cartesian_nli_psd(toy, 1.3e-3, ch_nu, 600)))
    for nr in (75, 300):
        t2 = toy_case(3, n_r=nr)
        v, q = R.nli_psd_at(t2, 1.3e-3, 193.5e12)
        probes.append(dict(case=t2.to_json(), gamma=1.3e-3, nu=193.5e12, value=v, quad=q))
    t3 = toy_case(3, n_r=80, mirror_q4=0)
    v, q = R.nli_psd_at(t3, 1.3e-3, 193.5e12 - 12e9)
    probes.append(dict(case=t3.to_json(), gamma=1.3e-3, nu=193.5e12 - 12e9, value=v, quad=q))
    out["nli_psd_at"] = probes

    # ---- full SNR evaluation (evaluate_link) ----
    links = {}
    for c in (uwb589(n_r=75, density=0.95, name="uwb589_75_0.95"),
              uwb589(n_r=40, density=0.95, launch_w=random_launch_589(),
                     name="uwb589_random_launch")):
        r = R.evaluate_link(c)
        links[c.name] = dict(case=c.to_json(), **r)
        print(f"link {c.name}: ode {r['t_ode']:.3f} nli {r['t_nli']:.2f} asm {r['t_asm']:.2e}")
    out["evaluate_link"] = links

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as fh:
        json.dump(_tolist(out), fh)
    print("wrote", path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
