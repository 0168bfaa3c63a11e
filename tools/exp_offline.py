"""Per-window cost of offline ABFT (not the product's measurement): step(K)
device time (CUDA events) of the cfg5 slab, error-free, NONE vs OFFLINE with
periods 1 / 5 / 20, both policies; medians of interleaved repetitions.
    python tools/exp_offline.py [cfg] [reps]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
K, W = 20, 5
p = make_problem(cfg, nz=128) if cfg == "cfg5" else make_problem(cfg)
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
stream = torch.cuda.Stream(dev)
arms = [("none", 0, 0, 1), ("off1_lazy", 2, 1, 1), ("off5_lazy", 2, 1, 5), ("off20_lazy", 2, 1, 20),
        ("off5_both", 2, 0, 5), ("off20_both", 2, 0, 20)]
res = {a[0]: [] for a in arms}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for name, mode, pol, delta in arms:
            q = p.replace(delta=delta)
            st = abft.from_problem(q, u0, P, device=dev, stream=stream, mode=mode, checksum_policy=pol)
            st.step(W)
            st.plan(K)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            st.step(K)
            e1.record(stream)
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / K * 1000.0)
            st.destroy()
base = statistics.median(res["none"])
for name, v in res.items():
    m = statistics.median(v)
    print(f"{cfg} {name:12s} {m:9.2f} us/sweep  overhead {100 * (m / base - 1):6.2f}%  [{min(v):.2f}, {max(v):.2f}]")
