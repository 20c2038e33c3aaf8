"""Golden fixtures for BASELINE config 2's stress variant (paper §III-B: 101
channels at the zero-dispersion wavelength, MCI-dominated) and the Simpson
mode on it, from the UNMODIFIED reference (oracle/_ref/libuwbref.so).  Run
here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden_stress.py

Writes tests/golden/golden_stress.json (floats via repr(): exact round trip).
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _tolist, provenance  # noqa: E402
from pyoracle import RefLib, oband11  # noqa: E402


def stress_cases():
    return [oband11(n_ch=101, name="oband101"),
            oband11(n_ch=101, n_r=80, simpson=1, name="oband101_simpson_nr80")]


def main():
    R = RefLib()
    out = dict(provenance=provenance(), all_channels_nli={})
    for c in stress_cases():
        r = R.all_channels_nli(c)
        out["all_channels_nli"][c.name] = dict(
            case=c.to_json(), eta=r["eta"], nli_psd=r["nli_psd"], nli_power=r["nli_power"],
            quadrant=r["quadrant"], skipped=r["skipped"], ref_nli_seconds=r["nli_seconds"],
            ref_ode_seconds=r["ode_seconds"])
        print(f"{c.name}: nli {r['nli_seconds']:.2f}s", flush=True)
    with open(os.path.join(HERE, "golden_stress.json"), "w") as fh:
        json.dump(_tolist(out), fh, indent=0)


if __name__ == "__main__":
    main()
