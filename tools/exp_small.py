"""Small-config launch timeline probe (run under ncu for per-kernel durations):
NONE, LAZY serial, BOTH serial and LAZY pipelined step(20) of one config.
    python tools/exp_small.py cfg2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft
p = make_problem(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
dev = torch.device("cuda:0")
u0, P = field_u0(p, dev), field_power(p, dev)
for name, mode, pol, sched in (("none", 0, 0, 0), ("lazy_serial", 1, 1, 1), ("both_serial", 1, 0, 1),
                               ("lazy_pipe", 1, 1, 0)):
    st = abft.from_problem(p, u0, P, device=dev, mode=mode, checksum_policy=pol, schedule=sched)
    st.step(5)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(name)
    st.step(20)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    st.destroy()
