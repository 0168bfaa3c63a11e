"""A/B of K1 variants in one process (experiment libraries under tools/explib,
not the product): per-launch K1 device time (profile hook) of the unprotected,
LAZY and BOTH sweeps of cfg4, interleaved over repetitions, medians.
    python tools/exp_k1_ab.py base base0 [reps]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft

libs = [a for a in sys.argv[1:] if not a.isdigit()]
reps = int(([a for a in sys.argv[1:] if a.isdigit()] or ["5"])[0])
handles = {}
import ctypes as C
for name in libs:
    path = (os.path.join(os.path.dirname(abft.__file__), "libabft_stencil.so") if name == "base"
            else os.path.join(os.path.dirname(os.path.abspath(__file__)), "explib", f"libabft_{name}.so"))
    handles[name] = path
p = make_problem("cfg4")
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
res = {n: {"none": [], "lazy": [], "both": [], "k2_lazy": [], "k2_both": []} for n in libs}
for rep in range(reps):
    for name in libs:
        abft._lib = None
        abft.LIB_PATH = handles[name]
        for tag, mode, pol in (("none", 0, 0), ("lazy", 1, 1), ("both", 1, 0)):
            st = abft.from_problem(p, u0, P, device=dev, mode=mode, checksum_policy=pol, schedule=1)
            st.step(3)
            st.profile(True)
            st.step(10)
            r = st.profile_read()
            res[name][tag].append(r["k1_ms"] / r["k1_launches"])
            if tag != "none":
                res[name]["k2_" + tag].append(r["k2_ms"] / 10)
            st.destroy()
out = {n: {t: round(statistics.median(v), 5) for t, v in d.items()} for n, d in res.items()}
for n, d in out.items():
    d["lazy/none"] = round(d["lazy"] / d["none"], 4)
    d["both/none"] = round(d["both"] / d["none"], 4)
print(json.dumps(out))
