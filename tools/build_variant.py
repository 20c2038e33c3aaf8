"""Build an A/B variant of libuwbnli.so with extra -D flags into abv/ (git-ignored, travels to the GPU box).

    python tools/build_variant.py NAME [-DFOO=1 ...]
Load it with UWB_LIB_PATH=abv/NAME.so (paper_2401_18022_b200/_native.py).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_18022_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "abv")  # git-ignored; not gpurun-ignored, so it travels
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, name + ".so")
try:
    b.compile_link(out, extra=defs)
except RuntimeError:
    sys.exit(1)
print(out)
