"""Live K1/K2 times per mode with nvidia-smi power/clock sampling per window.
Usage: python tools/exp_modes.py LIBNAME [cfg] [sweeps]"""
import os, sys, json, subprocess, tempfile, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft
name = sys.argv[1]
if name != "base":
    abft.LIB_PATH = os.path.join(os.path.dirname(abft.__file__), "exp", f"libabft_{name}.so")
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 200
p = make_problem(cfg)
if len(sys.argv) > 4:
    p = p.replace(nz=int(sys.argv[4]))
if p.mode == 2:
    p = p.replace(mode=1)   # per-sweep K1/K2 times: online
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
res = {"lib": name}
for mode, tag, pol in ((0, "unprot", 0), (1, "prot", 0), (1, "lazy", 1), (0, "unprot2", 0),
                       (1, "prot2", 0), (1, "lazy2", 1)):
    st = abft.from_problem(p, u0, P, device=dev, mode=mode, checksum_policy=pol)
    st.step(5)
    torch.cuda.synchronize()
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    sm = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "-i", "0",
                           "--format=csv,noheader,nounits", "-lms", "50"], stdout=f)
    time.sleep(0.3)
    st.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.step(K)
    e1.record()
    torch.cuda.synchronize()
    sm.terminate(); sm.wait(); f.seek(0)
    rows = [l.split(", ") for l in f.read().splitlines() if l.strip()]
    clk = [float(r[0]) for r in rows[6:]]; pw = [float(r[1]) for r in rows[6:]]
    r = st.profile_read()
    res[tag] = {"step_ms": round(e0.elapsed_time(e1) / K, 4),
                "k1_ms": round(r["k1_ms"] / r["k1_launches"], 4),
                "k2_ms": round(r["k2_ms"] / max(1, r["k2_launches"]), 4),
                "sm_mhz": statistics.median(clk) if clk else None,
                "power_w": statistics.median(pw) if pw else None}
    st.destroy()
print(json.dumps(res))
