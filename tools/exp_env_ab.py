"""A/B of environment switches read at launch time, in one process (not the
product's measurement): step(K) device time (CUDA events) after step(W) and
plan(K), error-free, NONE / LAZY / BOTH, arms interleaved, medians.
    python tools/exp_env_ab.py cfg3 VAR=a,b [reps]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft

cfg, spec = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
var, vals = spec.split("=")
vals = vals.split(",")
K, W = 20, 5
p = make_problem(cfg)
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
stream = torch.cuda.Stream(dev)
arms = [("none", 0, 0), ("lazy", 1, 1), ("both", 1, 0)]
res = {(v, a[0]): [] for v in vals for a in arms}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for v in vals:
            os.environ[var] = v
            for name, mode, pol in arms:
                st = abft.from_problem(p, u0, P, device=dev, stream=stream, mode=mode, checksum_policy=pol)
                st.step(W)
                st.plan(K)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                st.step(K)
                e1.record(stream)
                torch.cuda.synchronize()
                res[(v, name)].append(e0.elapsed_time(e1) / K * 1000.0)
                st.destroy()
for v in vals:
    base = statistics.median(res[(v, "none")])
    print(f"{cfg} {var}={v:4s} " + "  ".join(
        f"{n}: {statistics.median(res[(v, n)]):9.2f} us ({100 * (statistics.median(res[(v, n)]) / base - 1):+6.2f}%)"
        for n, _, _ in arms))
