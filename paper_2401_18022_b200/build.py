"""Build libuwbnli.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2401_18022_b200.build [--verbose]

-fmad=false keeps the host-equivalent setup arithmetic (coordinates,
stencils, phase mismatch, ODE controller) rounded exactly like the reference;
the integrand's hot loop uses explicit fma().  -lineinfo maps ncu's source
page back to the .cu files.
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libuwbnli.so")
SOURCES = ["nli_kernel.cu", "raman_ode.cu", "uwb_capi.cu", "uwb_link.cu", "uwb_model.cu",
           "uwb_cfm.cu", "uwb_multi.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "-Xptxas", "-warn-spills"]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps += [os.path.join(PKG, "..", "include", f) for f in ("uwb_nli.h", "uwb_model.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


OBJ_DIR = os.path.join(os.path.dirname(PKG), "build", "obj")


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    inc = os.path.join(PKG, "..", "include")
    hs += [os.path.join(inc, f) for f in ("uwb_nli.h", "uwb_model.h")]
    return [h for h in hs if os.path.exists(h)]


def compile_link(out, extra=(), verbose=False, cache=True):
    """One nvcc -c per source in parallel (the template instantiations make
    each file slow on its own), then one shared-library link.  With `cache`,
    objects live in build/obj (git-ignored) and a source is recompiled only
    when it, a header or the flags changed."""
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJ_DIR, exist_ok=True)
    # objects are keyed by the CONTENT of the flags, the source and every
    # header (not by mtimes: an edit during a compile must not leave a stale
    # object that looks fresh)
    hh = hashlib.sha1(" ".join(ARCH + FLAGS + list(extra)).encode())
    for h in sorted(_headers()):
        hh.update(open(h, "rb").read())

    def key(src):
        k = hh.copy()
        k.update(open(os.path.join(CSRC, src), "rb").read())
        return k.hexdigest()[:12]

    objs = [os.path.join(OBJ_DIR, os.path.splitext(src)[0] + "." + key(src) + ".o") for src in SOURCES]

    def stale(src, obj):
        return not cache or not os.path.exists(obj)

    def cc(args):
        src, obj = args
        if not stale(src, obj):
            return subprocess.CompletedProcess([], 0, "", "")
        cmd = [nvcc()] + ARCH + FLAGS + list(extra) + ["-c", "-o", obj + ".tmp", os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode == 0:
            os.replace(obj + ".tmp", obj)
        return r

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(cc, zip(SOURCES, objs)))
    link = [nvcc()] + ARCH + ["-shared", "-o", out] + objs
    results.append(subprocess.run(link, capture_output=True, text=True)
                   if all(r.returncode == 0 for r in results) else None)
    for r in results:
        if r is None:
            continue
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed")
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)
    return out


def build(verbose=False, force=False):
    if not force and not needs_build():
        return OUT
    compile_link(OUT + ".tmp", verbose=verbose)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(OUT)
