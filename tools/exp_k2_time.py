"""Per-sweep K2 (+K3) and step times of experiment libraries (tools/explib/,
not the product) against the product library.
    python tools/exp_k2_time.py base ku44 ku42 ..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from abft_inputs import make_problem, field_u0, field_power
from paper_1909_00709_b200 import abft

def run(p, pol, K=20):
    dev = torch.device("cuda:0")
    u0, P = field_u0(p, dev), field_power(p, dev)
    out = {}
    for prof in (False, True):
        st = abft.from_problem(p, u0, P, device=dev, checksum_policy=pol)
        st.step(5)
        torch.cuda.synchronize()
        st.profile(prof)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); st.step(K); e1.record(); torch.cuda.synchronize()
        if prof:
            r = st.profile_read()
            out["k2_us"] = round(r["k2_ms"] / K * 1e3, 2)
        else:
            out["step_us"] = round(e0.elapsed_time(e1) / K * 1e3, 2)
        st.destroy()
    return out

for name in sys.argv[1:]:
    abft._lib = None
    abft.LIB_PATH = (os.path.join(os.path.dirname(abft.__file__), "libabft_stencil.so") if name == "base"
                     else os.path.join(os.path.dirname(os.path.abspath(__file__)), "explib", f"libabft_{name}.so"))
    res = {"lib": name}
    for cfg, pol in (("cfg4", 0), ("cfg4", 1), ("cfg3", 1), ("cfg2", 1), ("cfg5", 0)):
        p = make_problem(cfg)
        if cfg == "cfg5":
            p = p.replace(nz=128)
        res[f"{cfg}_{'lazy' if pol else 'both'}"] = run(p, pol)
    print(json.dumps(res), flush=True)
