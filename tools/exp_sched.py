"""A/B of the check schedules in one process (not the product's measurement):
step(K) device time (CUDA events on the handle's stream) after step(W) and
plan(K), error-free, for NONE / LAZY / BOTH under the serial and pipelined
schedules with and without step graphs; interleaved repetitions, medians.
    python tools/exp_sched.py cfg2 [reps] [K]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft

cfg = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
K = int(sys.argv[3]) if len(sys.argv) > 3 else 20
W = 5
p = make_problem(cfg)
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
stream = torch.cuda.Stream(dev)
arms = [("none", 0, 0, 0, 1, 0, 0), ("none_nog", 0, 0, 0, 0, 0, 0),
        ("lazy_serial", 1, 1, 1, 1, 0, 0),
        ("lazy_pipe", 1, 1, 0, 1, 0, 0), ("lazy_pipe_nog", 1, 1, 0, 0, 0, 0),
        ("lazy_pipe_lo", 1, 1, 0, 1, -1, 0), ("lazy_pipe_lo_nog", 1, 1, 0, 0, -1, 0),
        ("lazy_pipe_pdl", 1, 1, 0, 1, 0, 1), ("lazy_pipe_pdl_nog", 1, 1, 0, 0, 0, 1),
        ("both_serial", 1, 0, 1, 1, 0, 0), ("both_pipe", 1, 0, 0, 1, 0, 0), ("both_pipe_lo", 1, 0, 0, 1, -1, 0)]
res = {a[0]: [] for a in arms}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for name, mode, pol, sched, graphs, prio, pdl in arms:
            os.environ["ABFT_GRAPHS"] = str(graphs)
            os.environ["ABFT_S2_PRIO"] = str(prio)
            os.environ["ABFT_PIPE_PDL"] = str(pdl)
            st = abft.from_problem(p, u0, P, device=dev, stream=stream, mode=mode, checksum_policy=pol,
                                   schedule=sched)
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
    print(f"{cfg} {name:14s} {m:9.2f} us/sweep  overhead vs none(graph) {100 * (m / base - 1):7.2f}%  "
          f"[{min(v):.2f}, {max(v):.2f}]")
