# experiment builds of the K1 translation units (HotSpot fp32 only) linked with
# the product's other objects: tools/explib/libabft_<name>.so
name=$1; shift
python - "$name" "$@" <<'PY'
import glob, os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_1909_00709_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(os.getcwd(), "tools", "explib"); os.makedirs(out, exist_ok=True)
B.build()
var = ["k1_f32_s4.cu", "k1_f32_s2.cu"]
objs = []
for s in var:
    o = os.path.join(out, f"{name}_{s}.o")
    subprocess.run([B.NVCC] + B.flags() + defs + ["-c", os.path.join(B.CSRC, s), "-o", o], check=True, capture_output=True)
    objs.append(o)
objs += [p for p in glob.glob(os.path.join(B.BUILD, "*.o")) if os.path.basename(p).replace(".o", "") not in var]
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(out, f"libabft_{name}.so")] + objs + ["-ldl"], check=True)
for o in objs[:len(var)]: os.remove(o)
print("built", name)
PY
