"""Experiment variants of the K2 translation unit (not the product): rebuild
only k2_check.cu with -D switches and link it with the product's other
objects.   python tools/exp_k2.py NAME -DABFT_KU_FEW=4 ...
writes tools/explib/libabft_NAME.so (it travels to the GPU box)"""
import glob, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_00709_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "explib")
os.makedirs(out, exist_ok=True)
B.build()
src = os.path.join(B.CSRC, "k2_check.cu")
o = os.path.join(out, f"{name}_k2_check.o")
subprocess.run([B.NVCC] + B.flags() + defs + ["-c", src, "-o", o], check=True, capture_output=True)
objs = [p for p in glob.glob(os.path.join(B.BUILD, "*.o")) if not p.endswith("k2_check.cu.o")] + [o]
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, f"libabft_{name}.so")] + objs + ["-ldl"],
               check=True)
os.remove(o)
print("built", name)
