"""Cost of recovering a dirty offline window (not the product's measurement):
step(K) device time (CUDA events) of the cfg5 slab, offline period 5, with
n flips per window at layers spread over the slab; recovery ROLLBACK vs
PARTIAL (the union of the flagged layers' cones, Q28), against the
error-free run; medians of interleaved repetitions.
    python tools/exp_partial.py [reps]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power, Fault
from paper_1909_00709_b200 import abft

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K, W = 20, 5
p = make_problem("cfg5", nz=128, checksums=1)   # policy LAZY: b-only windows (Q29), the bench headline
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
stream = torch.cuda.Stream(dev)


def flips(n):
    # n flips in every window of the timed region, at layers spread evenly
    # over the slab (the first one 12 layers from the lower face), bit 55
    out = []
    for w in range(K // p.delta):
        for i in range(n):
            z = 12 + i * (p.nz - 24) // max(1, n - 1) if n > 1 else p.nz // 2
            out.append(Fault(W + w * p.delta + 1 + (i % p.delta), z, 100 + 37 * i, 200 + 91 * i, 55))
    return out


arms = [("clean", 0, 0)] + [(f"{n}flips_{'partial' if r else 'rollback'}", n, r) for n in (1, 2, 3, 4) for r in (0, 1)]
res = {a[0]: [] for a in arms}
info = {}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for name, n, rec in arms:
            st = abft.from_problem(p.replace(recovery=rec), u0, P, device=dev, stream=stream)
            st.set_faults(flips(n) if n else [])
            st.step(W)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            st.step(K)
            e1.record(stream)
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) / K)
            s = st.stats()
            info[name] = (s["rollbacks"], s["persistent"], s["sweeps"])
            st.destroy()
base = statistics.median(res["clean"])
cells = p.nx * p.ny * p.nz
for name, v in res.items():
    m = statistics.median(v)
    print(f"cfg5 slab {name:16s} {m:8.3f} ms/sweep  {cells / m * 1e-6:7.1f} GCell/s  vs clean {100 * (m / base - 1):6.1f}%"
          f"  rollbacks {info[name][0]} persistent {info[name][1]}")
