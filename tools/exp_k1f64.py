"""Experiment variants of the fp64 27-point K1 units (not the product): rebuild
only k1_f64_s3_ck*.cu with -D switches, link with the product's other
objects.   python tools/exp_k1f64.py NAME -DABFT_HALO_LDS=1 ...
writes tools/explib/libabft_NAME.so (it travels to the GPU box)"""
import glob, os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_00709_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "explib")
os.makedirs(out, exist_ok=True)
B.build()
units = sorted(glob.glob(os.path.join(B.CSRC, "k1_f64_s3_ck*.cu")))
def one(src):
    o = os.path.join(out, f"{name}_{os.path.basename(src)}.o")
    subprocess.run([B.NVCC] + B.flags() + defs + ["-c", src, "-o", o], check=True, capture_output=True)
    return o
with ThreadPoolExecutor(len(units)) as ex:
    new = list(ex.map(one, units))
skip = {os.path.basename(u) + ".o" for u in units}
objs = [p for p in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(p) not in skip] + new
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, f"libabft_{name}.so")] + objs + ["-ldl"],
               check=True)
for o in new:
    os.remove(o)
print("built", name)
