"""Experiment builds: libdash.so compiled with extra -D flags into
paper_2601_21824_b200/variants/libdash_<name>.so (git-ignored, travels to the
GPU box with gpurun); select one with DASH_LIB_PATH=<path> for A/B runs.

  python scripts/build_variant.py poly4 -DDASH_POLY_EXP_EVERY=4
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_21824_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "paper_2601_21824_b200", "variants")
obj_dir = os.path.join(out_dir, "obj_" + name)
os.makedirs(obj_dir, exist_ok=True)
objs = []
for src in B._sources():
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    subprocess.check_call([B.NVCC] + B.NVCC_FLAGS + defs + ["-c", src, "-o", obj])
    objs.append(obj)
lib = os.path.join(out_dir, f"libdash_{name}.so")
subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + ["-ldl"])
print(lib)
