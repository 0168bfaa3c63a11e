"""GPU parity at the sizes BASELINE.json states (Table 1 tiles,
BJ configs[2..4]): the sm_100a path through the C-ABI against the CPU oracle,
element by element, on the same seeded inputs and fault schedules.  The
oracle runs inside the test (nothing precomputed).

* cfg3: 512x512x64 fp32 HotSpot, 1000 sweeps, 20 flips, online and offline
  (period 10);
* cfg4: 1024^3 fp32 HotSpot, 10 sweeps with bench.py's fault schedule and
  checksum policy (LAZY), field, a, b and records bitwise;
* cfg5: the 2048x2048 fp64 27-point box z-reduced to 64 layers (SURVEY
  §8(d): the full 2048x2048x1024 needs ~100 GiB of host memory for the
  oracle), offline period 5, 20 sweeps with its flips;
* cfg5 at full size (2048x2048x1024 fp64, 100 sweeps): oracle-free
  invariants -- rollback restores the fault-free run bitwise when every
  flip is detected, and any z-slab decomposition is bitwise identical.

Bars: fp32 fields / checksums / record values bitwise; fp64 fields <= 1e-12
relative (bitwise in practice), checksums <= 1e-13; detected / located /
corrected indices and statuses exact (north_star).
"""
import numpy as np
import pytest
import torch

from abft_inputs import Fault, fault_schedule, field_power, field_u0, make_problem
from tests.parity_util import parity

pytestmark = pytest.mark.gpu


def setup_module(module):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_cfg3_full_online_1000_sweeps_20_flips():
    p = make_problem("cfg3")
    assert (p.nx, p.ny, p.nz, p.sweeps) == (512, 512, 64, 1000)
    g, o = parity(p)
    assert len(fault_schedule(p)) == 20
    assert o["stats"]["detections"] >= 4 and o["stats"]["sweeps"] == 1000


def test_cfg3_full_offline_period_10():
    p = make_problem("cfg3", mode=2, delta=10)
    g, o = parity(p)
    assert o["stats"]["windows"] >= 100 and o["stats"]["rollbacks"] >= 1


def test_cfg4_full_size_10_sweeps_bench_schedule():
    # bench.py's headline run: cfg4, checksum policy LAZY, the
    # schedule fault_schedule(p, K) -- one flip per 128-layer slab
    p = make_problem("cfg4", checksums=1)
    faults = fault_schedule(p, 10)
    assert len(faults) == 8
    g, o = parity(p, nsweeps=10, faults=faults)
    assert o["stats"]["detections"] >= 4


def test_cfg4_full_size_policy_both_5_sweeps():
    p = make_problem("cfg4")
    faults = [Fault(2, 5, 17, 900, 30), Fault(3, 1023, 1023, 0, 29), Fault(4, 512, 0, 1023, 27),
              Fault(5, 0, 511, 511, 25)]
    g, o = parity(p, nsweeps=5, faults=faults)
    assert o["stats"]["corrected"] == 4


def test_cfg5_2048_planes_z_reduced_offline():
    p = make_problem("cfg5", nz=64, sweeps=20)
    assert (p.nx, p.ny, p.delta, p.mode) == (2048, 2048, 5, 2)
    faults = fault_schedule(p)
    assert len(faults) == 50
    g, o = parity(p)
    assert o["stats"]["rollbacks"] >= 1 and o["stats"]["persistent"] == 0


# ---- cfg5 at full size: oracle-free invariants ----------------

def _cfg5_run(p, faults, G=1):
    """Run cfg5 on one GPU as G z-slabs (G > 1: a local group); the final
    field comes back to host memory (32 GiB) so the next run has the device."""
    from paper_1909_00709_b200 import abft
    dev = torch.device("cuda:0")
    sts = []
    zs = [(i * p.nz // G, (i + 1) * p.nz // G - i * p.nz // G) for i in range(G)]
    for i, (z0, zc) in enumerate(zs):
        u0 = field_u0(p, dev, z0, zc)
        kw = dict(z_begin=z0, z_count=zc, rank=i, nranks=G) if G > 1 else {}
        st = abft.from_problem(p, u0, None, device=dev,
                               stream=torch.cuda.Stream(dev) if G > 1 else None, **kw)
        torch.cuda.synchronize()
        st._u0 = None           # init copied it into the handle's buffer
        del u0
        st.set_faults(faults)
        sts.append(st)
    if G > 1:
        abft.group(sts)
        status = abft.step_group(sts, p.sweeps)
    else:
        status = sts[0].step(p.sweeps)
    out = dict(status=status, records=sum((s.records() for s in sts), []),
               stats=[s.stats() for s in sts])
    out["u"] = torch.empty((p.nz, p.ny, p.nx), dtype=torch.float64)
    for s, (z0, zc) in zip(sts, zs):
        s.read_field(out["u"][z0:z0 + zc])
        s.destroy()
    sts.clear()
    torch.cuda.empty_cache()
    return out


def _bits(t):
    return t.view(torch.int64)


def _need_memory(p):
    import gc
    import psutil
    gc.collect()
    torch.cuda.empty_cache()      # blocks the earlier tests left in torch's cache
    free, total = torch.cuda.mem_get_info()
    need_dev = 4 * p.cells * 8                 # 3 field buffers + the initial slab
    need_host = 2 * p.cells * 8 + (16 << 30)   # two final fields + headroom
    if free < need_dev:
        pytest.skip(f"needs {need_dev / 2**30:.0f} GiB of device memory")
    if psutil.virtual_memory().available < need_host:
        pytest.skip(f"needs {need_host / 2**30:.0f} GiB of host memory")


def test_cfg5_full_size_rollback_restores_fault_free_run():
    p = make_problem("cfg5")
    _need_memory(p)
    # the cfg5 cells and sweeps, bits moved to >= 40 so every flip is above
    # eps = 1e-10 relative to its row / column sum (delta >= 2^-14 against
    # sums ~1e3): every dirty window is rolled back and re-executed clean
    faults = [Fault(f.sweep, f.z, f.y, f.x, 40 + f.bit % 24) for f in fault_schedule(p)]
    ref = _cfg5_run(p, [])
    assert ref["stats"][0]["detections"] == 0           # no false positive over 100 sweeps
    got = _cfg5_run(p, faults)
    assert got["status"] == 0
    windows = {((f.sweep - 1) // p.delta + 1) * p.delta for f in faults}
    assert got["stats"][0]["rollbacks"] == len(windows)
    assert got["stats"][0]["persistent"] == 0
    assert torch.equal(_bits(got["u"]), _bits(ref["u"]))


def test_cfg5_full_size_slab_decomposition_is_bitwise_invariant():
    p = make_problem("cfg5")
    _need_memory(p)
    faults = fault_schedule(p)
    one = _cfg5_run(p, faults)
    eight = _cfg5_run(p, faults, G=8)
    assert torch.equal(_bits(eight["u"]), _bits(one["u"]))
    key = lambda r: (r["sweep"], r["z"], r["status"], r["y"], r["x"], r["nflag_a"], r["nflag_b"])
    assert sorted(map(key, one["records"])) == sorted(map(key, eight["records"]))
    assert one["stats"][0]["rollbacks"] == eight["stats"][0]["rollbacks"] >= 1
