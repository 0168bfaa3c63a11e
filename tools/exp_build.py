"""Experiment builds of libabft_stencil.so with -D switches (not the product):
    python tools/exp_build.py NAME -DABFT_EXP_...
writes paper_1909_00709_b200/exp/libabft_NAME.so"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_00709_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, "exp")
os.makedirs(out, exist_ok=True)
objs = []
for src in B._sources():
    o = os.path.join(out, f"{name}_{os.path.basename(src)}.o")
    subprocess.run([B.NVCC] + B.flags() + defs + ["-c", src, "-o", o], check=True, capture_output=True)
    objs.append(o)
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, f"libabft_{name}.so")] + objs + ["-ldl"], check=True)
for o in objs:
    os.remove(o)
print("built", name)
