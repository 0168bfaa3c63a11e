"""Shared helpers of the GPU-vs-oracle parity tests (test infrastructure).

Both sides consume the same seeded inputs from abft_inputs; the GPU side is
called only through the C-ABI binding, the oracle only through oracle/.
"""
from __future__ import annotations

import numpy as np
import torch

from abft_inputs import Fault, field_power, field_u0, fault_schedule
from oracle import oracle as O


def oracle_run(p, nsweeps=None, faults=None, u0=None, power=None):
    n = p.sweeps if nsweeps is None else nsweeps
    fl = fault_schedule(p, n) if faults is None else faults
    u0 = field_u0(p).numpy() if u0 is None else u0
    if power is None and p.power is not None:
        power = field_power(p).numpy()
    op = O.OProblem(p, [power] if p.power is not None else [])
    return O.run(op, u0, n, fl)


def gpu_run(p, nsweeps=None, faults=None, explicit=False, u0=None, power=None, **kw):
    from paper_1909_00709_b200 import abft
    n = p.sweeps if nsweeps is None else nsweeps
    fl = fault_schedule(p, n) if faults is None else faults
    dev = torch.device("cuda:0")
    u0 = field_u0(p, dev) if u0 is None else torch.as_tensor(u0).to(dev)
    if power is None and p.power is not None:
        power = field_power(p, dev)
    elif power is not None:
        power = torch.as_tensor(power).to(dev)
    st = abft.from_problem(p, u0, power, device=dev, **kw)
    st.set_faults(fl)
    status = 0
    if explicit:
        for _ in range(n):
            st.sweep()
            if p.mode == 1:
                na, nb = st.check()
                st.correct()
    else:
        status = st.step(n)
    out = dict(u=st.read_field().cpu().numpy(), stats=st.stats(), records=st.records(),
               status=max(status, st.status()), launches=st.launches)
    A, B = st.checksums()
    out["A"], out["B"] = A.numpy(), B.numpy()
    st.destroy()
    return out


def key(r):
    return (r["sweep"], r["z"], r["status"], r["y"], r["x"])


def assert_records_equal(g, o, exact_values=True, rtol=0.0):
    gr = sorted(g["records"], key=key)
    orr = sorted(o["records"], key=key)
    assert [key(r) for r in gr] == [key(r) for r in orr], (gr[:5], orr[:5])
    for a, b in zip(gr, orr):
        assert (a["nflag_a"], a["nflag_b"]) == (b["nflag_a"], b["nflag_b"])
        for f in ("observed", "corrected", "vx", "vy"):
            x, y = a[f], b[f]
            if exact_values:
                assert (x == y) or (np.isnan(x) and np.isnan(y)), (f, a, b)
            else:
                assert abs(x - y) <= rtol * max(abs(y), 1e-300) or (np.isnan(x) and np.isnan(y)), (f, a, b)


def assert_stats_equal(g, o):
    for k in ("sweeps", "detections", "located", "corrected", "unlocated", "uncorrectable",
              "rollbacks", "windows", "persistent"):
        assert g["stats"][k] == o["stats"][k], (k, g["stats"], o["stats"])


def assert_field_equal(g, o, dtype):
    a, b = g["u"], o["u"]
    if dtype == "f32":
        assert a.dtype == np.float32
        bad = np.flatnonzero(a.view(np.uint32) != b.view(np.uint32))
        assert bad.size == 0, (bad[:10], a.ravel()[bad[:5]], b.ravel()[bad[:5]])
    else:
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        assert np.nanmax(rel) <= 1e-12, np.nanmax(rel)


def assert_checksums_close(g, o, rtol):
    """a (sums over y) and b (sums over x) of the final field.  fp32 data in
    the configs' ranges sum exactly in fp64, so any summation order gives the
    same bits (rtol 0).  Where a sum is not exact -- an uncorrected exponent
    flip leaves a cell ~1e21 in the layer, or fp64 data -- the GPU's
    reduction order and the oracle's ascending order may round differently;
    both lie within the textbook bound (n - 1) 2^-53 sum|u| of the exact sum
    (DESIGN.md "Parity bars"), so they may differ by twice that."""
    u = np.abs(o["u"].astype(np.float64))
    bound = {"A": 2.0 * u.shape[1] * 2.0 ** -53 * u.sum(axis=1),
             "B": 2.0 * u.shape[2] * 2.0 ** -53 * u.sum(axis=2)}
    for k in ("A", "B"):
        a, b = g[k], o[k]
        same = (a == b) | (np.isnan(a) & np.isnan(b))
        if rtol == 0.0:
            bad = ~same & ~(np.abs(a - b) <= bound[k])
        else:
            rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
            bad = ~same & ~(rel <= rtol) & ~(np.abs(a - b) <= bound[k])
        assert not bad.any(), (k, np.flatnonzero(bad)[:10], a[bad][:3], b[bad][:3])


def parity(p, nsweeps=None, faults=None, explicit=False, dtype=None, **kw):
    """Run both sides; assert the paper's outputs agree (indices bit-exact,
    fp32 values bitwise, fp64 values within 1e-12)."""
    dtype = dtype or p.dtype
    o = oracle_run(p, nsweeps, faults)
    g = gpu_run(p, nsweeps, faults, explicit=explicit, **kw)
    assert_field_equal(g, o, dtype)
    assert_records_equal(g, o, exact_values=(dtype == "f32"), rtol=1e-12)
    assert_stats_equal(g, o)
    assert g["status"] == o["status"]
    assert_checksums_close(g, o, 0.0 if dtype == "f32" else 1e-13)
    return g, o
