"""Golden fixtures for the closed-form model (cfm_all_channels_nli,
gn_closed_form.hpp:70-144) from the UNMODIFIED reference
(oracle/_ref/libuwbref.so).  Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden_cfm.py

Writes tests/golden/golden_cfm.json (floats via repr(): exact round trip).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import _tolist, provenance, random_launch_589  # noqa: E402
from pyoracle import RefLib, cband11, oband11, toy_case, uwb589  # noqa: E402


def cfm_cases():
    return [
        cband11(),
        oband11(),
        toy_case(5, n_r=8, guard=np.array([0, 0, 1, 0, 0], np.uint8), name="toy5_guard"),
        toy_case(3, n_r=8, span_count=3, length_m=50e3, name="toy3_3span"),
        uwb589(n_r=8, density=0.95, name="uwb589_0.95"),
        uwb589(n_r=8, density=1.4, launch_w=random_launch_589(), name="uwb589_random_launch"),
    ]


def main():
    R = RefLib()
    out = dict(provenance=provenance(), cfm_all_channels_nli={})
    for case in cfm_cases():
        r = R.cfm_all_channels_nli(case)
        r.pop("seconds")
        out["cfm_all_channels_nli"][case.name] = dict(case=case.to_json(), **_tolist(r))
        print(case.name, float(np.max(r["eta"])), flush=True)
    with open(os.path.join(HERE, "golden_cfm.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
