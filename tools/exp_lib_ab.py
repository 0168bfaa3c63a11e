"""A/B of two builds in one process (not the product's measurement): step(K)
device time (CUDA events on the handle's stream) after step(W) and plan(K),
error-free, NONE / LAZY / BOTH, libraries interleaved per repetition, medians.
    python tools/exp_lib_ab.py cfg4 base old [reps]   (old: tools/explib/libabft_old.so)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
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
stream = torch.cuda.Stream(dev)
arms = [("none", 0, 0), ("lazy", 1, 1), ("both", 1, 0)]
res = {(n, a[0]): [] for n in libs for a in arms}
with torch.cuda.stream(stream):
    for rep in range(reps):
        for n in libs:
            abft._lib = None
            abft.LIB_PATH = path[n]
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
                res[(n, name)].append(e0.elapsed_time(e1) / K * 1000.0)
                st.destroy()
for n in libs:
    base = statistics.median(res[(n, "none")])
    print(f"{cfg} {n:6s} " + "  ".join(f"{a}: {statistics.median(res[(n, a)]):9.2f} us "
                                         f"({100 * (statistics.median(res[(n, a)]) / base - 1):+6.2f}%)"
                                         for a, _, _ in arms))
