"""Builds libdash.so (and the test-only libdash_probe.so) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdash.so")
PROBE_LIB = os.path.join(HERE, "libdash_probe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
                     "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _sources():
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    return [s for s in srcs if not s.endswith("probe.cu")]


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "dash.h")])


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> str:
    deps = _deps()
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []
    if force or _stale(LIB, deps):
        objs = []
        for src in _sources():
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            _run([NVCC] + NVCC_FLAGS + extra + ["-c", src, "-o", obj], verbose)
            objs.append(obj)
        tmp = LIB + f".tmp{os.getpid()}"
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"], verbose)
        os.replace(tmp, LIB)
    if force or _stale(PROBE_LIB, deps):
        tmp = PROBE_LIB + f".tmp{os.getpid()}"
        _run([NVCC] + NVCC_FLAGS + extra + ["-shared", "-o", tmp, os.path.join(CSRC, "probe.cu")],
             verbose)
        os.replace(tmp, PROBE_LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="-v" in sys.argv)
