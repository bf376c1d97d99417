"""Experiment builds of libdash.so into paper_2601_21824_b200/variants/libdash_<name>.so
(git-ignored, travels to the GPU box with gpurun); select one with
DASH_LIB_PATH=<path> for A/B runs (scripts/gpu_ab.sh compares the working tree
with variants/libdash_head.so).

  python scripts/build_variant.py poly4 -DDASH_POLY_EXP_EVERY=4   # working tree + -D flags
  python scripts/build_variant.py head --rev HEAD                 # the sources of a commit
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = sys.argv[1:]
name = args.pop(0)
rev = None
if "--rev" in args:
    i = args.index("--rev")
    rev = args[i + 1]
    del args[i:i + 2]
defs = args
src_root = ROOT
tmp = None
if rev is not None:
    tmp = tempfile.mkdtemp(prefix="dash_rev_")
    subprocess.check_call(f"git archive {rev} | tar -x -C {tmp}", shell=True, cwd=ROOT)
    src_root = tmp
sys.path.insert(0, src_root)
from paper_2601_21824_b200 import build as B  # noqa: E402

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
if tmp:
    shutil.rmtree(tmp, ignore_errors=True)
print(lib)
