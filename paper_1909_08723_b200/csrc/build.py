"""Build libfusedbeam_b200.so in-tree with nvcc for sm_100a (no JIT, no torch).

    python -m paper_1909_08723_b200.csrc.build [--force]

Each .cu compiles to an object with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -O3``; objects are relinked only when a source or header changed.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
ROOT = os.path.dirname(PKG)
INCLUDE = os.path.join(ROOT, "include")
# dev A/B builds: FB_BUILD_TAG=x (+ FB_NVCC_EXTRA=-D...) -> libfusedbeam_b200_x.so,
# loaded with FB_LIB_AB=libfusedbeam_b200_x.so
_TAG = os.environ.get("FB_BUILD_TAG", "")
OUT = os.path.join(PKG, f"libfusedbeam_b200{'_' + _TAG if _TAG else ''}.so")
OBJ = os.path.join(HERE, "_obj" + ("_" + _TAG if _TAG else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-I", HERE]

SOURCES = ["capi.cu", "lookahead.cu", "search.cu", "gemm_tc.cu", "asr.cu", "host_io.cu"]
# test-only device code (not in the product library): tests/libfb_testkit.so
TESTKIT_SRC = os.path.join(ROOT, "tests", "csrc", "simt_gemm.cu")
TESTKIT_OUT = os.path.join(ROOT, "tests", "libfb_testkit.so")


def _headers():
    hs = [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    hs += [os.path.join(HERE, f) for f in os.listdir(HERE) if f.endswith(".cuh")]
    return hs


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    objs = []
    for src in SOURCES:
        path = os.path.join(HERE, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(obj)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_mtime)):
            continue
        extra = os.environ.get("FB_NVCC_EXTRA", "").split()     # dev experiments only
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-lcuda"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if not _TAG:
        build_testkit(force, verbose, hdr_mtime)
    return OUT


def build_testkit(force: bool = False, verbose: bool = False, hdr_mtime: float = 0.0) -> str:
    """The test-only SIMT GEMM cross-check library (tests/csrc)."""
    if not os.path.exists(TESTKIT_SRC):
        return ""
    if (force or not os.path.exists(TESTKIT_OUT)
            or os.path.getmtime(TESTKIT_OUT) < max(os.path.getmtime(TESTKIT_SRC), hdr_mtime)):
        cmd = [NVCC, *ARCH, *FLAGS, "-shared", TESTKIT_SRC, "-o", TESTKIT_OUT]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return TESTKIT_OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=True))
    sys.exit(0)
