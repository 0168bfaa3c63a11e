"""A/B of two builds in one process with the config's scheduled flips on (not
the product's measurement): step(K) device time after step(W), NONE error-free
and LAZY / BOTH with flips, libraries interleaved per repetition, medians.
    python tools/exp_flips_ab.py cfg3 base old [reps]   (old: tools/explib/libabft_old.so)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import Fault, make_problem, field_u0, field_power, fault_schedule
from paper_1909_00709_b200 import abft

cfg = sys.argv[1]
libs = [a for a in sys.argv[2:] if not a.isdigit()]
reps = int(([a for a in sys.argv[2:] if a.isdigit()] or ["5"])[0])
K, W = 20, 5
path = {n: (os.path.join(os.path.dirname(abft.__file__), "libabft_stencil.so") if n == "base" else
            os.path.join(os.path.dirname(os.path.abspath(__file__)), "explib", f"libabft_{n}.so")) for n in libs}
p = make_problem(cfg)
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
faults = [Fault(f.sweep + W, f.z, f.y, f.x, f.bit) for f in fault_schedule(p, K)]
stream = torch.cuda.Stream(dev)
arms = [("none", 0, 0, False), ("lazy+flips", 1, 1, True), ("both+flips", 1, 0, True)]
res = {(n, a[0]): [] for n in libs for a in arms}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for n in libs:
            abft._lib = None
            abft.LIB_PATH = path[n]
            for name, mode, pol, fl in arms:
                st = abft.from_problem(p, u0, P, device=dev, stream=stream, mode=mode, checksum_policy=pol)
                if fl:
                    st.set_faults(faults)
                st.step(W)
                st.plan(K)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(stream)
                st.step(K)
                e1.record(stream)
                torch.cuda.synchronize()
                res[(n, name)].append(e0.elapsed_time(e1) / K * 1000.0)
                st.destroy()
print(cfg, len(faults), "flips in", K, "sweeps")
for n in libs:
    base = statistics.median(res[(n, "none")])
    print(f"{cfg} {n:6s} " + "  ".join(f"{a}: {statistics.median(res[(n, a)]):9.2f} us "
                                         f"({100 * (statistics.median(res[(n, a)]) / base - 1):+6.2f}%)"
                                         for a, _, _, _ in arms))
