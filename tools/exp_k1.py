"""Times K1 (protected / unprotected) and K2 of the cfg4 workload for each
experiment library given on the command line (CUDA events via the C-ABI
profile hook).  Usage: python tools/exp_k1.py base noS2 ..."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft
name = sys.argv[1]
if name != "base":
    abft.LIB_PATH = os.path.join(os.path.dirname(abft.__file__), "exp", f"libabft_{name}.so")
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
p = make_problem(cfg)
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
res = {"lib": name}
for mode, tag in ((1, "prot"), (0, "unprot")):
    st = abft.from_problem(p, u0, P, device=dev, mode=mode)
    st.step(5)
    st.profile(True)
    st.step(40)
    r = st.profile_read()
    res[tag + "_k1_ms"] = round(r["k1_ms"] / r["k1_launches"], 4)
    if r["k2_launches"]:
        res[tag + "_k2_ms"] = round(r["k2_ms"] / r["k2_launches"], 4)
    st.destroy()
print(json.dumps(res))
