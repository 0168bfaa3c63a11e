"""GPU parity of offline ABFT under checksum policy LAZY (Q29):
every window predicts, sums and compares b alone -- offline never corrects,
so the second vector, which the paper computes only "to enable correction"
(P:271-273), is never needed.  Field bitwise (fp32) / 1e-12
(fp64), records (nflag_a = 0, x = -1), stats and the final a, b against the
oracle of the same policy; single slab, partial re-execution, local groups.
"""
import numpy as np
import pytest
import torch

from abft_inputs import Fault, fault_schedule, make_problem
from tests.parity_util import assert_records_equal, gpu_run, oracle_run, parity

pytestmark = pytest.mark.gpu


def setup_module(module):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _bonly(g, o):
    assert all(r["nflag_a"] == 0 and r["x"] == -1 for r in o["records"])
    assert all(r["nflag_a"] == 0 and r["x"] == -1 for r in g["records"])


@pytest.mark.parametrize("name,kw", [
    ("cfg3", dict(nz=12, sweeps=60, nfaults=8, mode=2, delta=10)),
    ("cfg3", dict(nx=128, ny=96, nz=5, sweeps=23, nfaults=4, mode=2, delta=10)),   # short last window
    ("cfg3", dict(nx=203, ny=77, nz=9, sweeps=24, nfaults=6, mode=2, delta=4)),    # ragged tiles
    ("cfg3", dict(nx=96, ny=80, nz=12, sweeps=24, nfaults=6, mode=2, delta=6, bc=1)),
    ("cfg3", dict(nx=96, ny=80, nz=12, sweeps=24, nfaults=6, mode=2, delta=6, bc=3, bc_value=330.0)),
    ("cfg5", dict(nx=130, ny=67, nz=12, sweeps=20, nfaults=6)),
    ("cfg5", dict(nx=70, ny=33, nz=9, sweeps=15, nfaults=6, delta=1)),
])
def test_offline_b_only_equals_oracle(name, kw):
    p = make_problem(name, checksums=1, **kw)
    g, o = parity(p)
    _bonly(g, o)
    assert o["stats"]["rollbacks"] >= 1


@pytest.mark.parametrize("delta", [1, 3, 6])
def test_offline_b_only_partial_reexecution(delta):
    p = make_problem("cfg3", nx=96, ny=80, nz=40, sweeps=4 * delta, mode=2, delta=delta, recovery=1,
                     checksums=1)
    faults = [Fault(1, 11, 7, 9, 24), Fault(delta + 1, 0, 79, 95, 30), Fault(2 * delta + 1, 39, 0, 0, 28),
              Fault(3 * delta + 1, 5, 20, 20, 24), Fault(3 * delta + 1, 30, 3, 30, 29),
              Fault(4 * delta, 20, 40, 50, 3)]
    g, o = parity(p, faults=faults)
    _bonly(g, o)
    assert o["stats"]["rollbacks"] == 4


def test_offline_b_only_persistent_error():
    p = make_problem("cfg3", nx=32, ny=32, nz=10, sweeps=10, mode=2, delta=5, checksums=1)
    g, o = parity(p, faults=[Fault(3, 1, 5, 5, 30), Fault(3, 1, 5, 5, 30)])
    assert o["status"] == 3 and o["stats"]["persistent"] == 1


def test_offline_b_only_equals_both_when_b_flags():
    # flips that flag b: the b-only run rolls back the same windows as BOTH,
    # so the GPU field is bitwise the BOTH run's
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=20, mode=2, delta=5)
    faults = [Fault(2, 3, 10, 20, 29), Fault(7, 11, 79, 0, 27), Fault(14, 0, 0, 95, 30)]
    b = gpu_run(p, faults=faults)
    l = gpu_run(p.replace(checksums=1), faults=faults)
    assert b["stats"]["rollbacks"] == l["stats"]["rollbacks"] == 3
    assert np.array_equal(b["u"].view(np.uint32), l["u"].view(np.uint32))
    assert np.array_equal(b["A"], l["A"]) and np.array_equal(b["B"], l["B"])


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("recovery", [0, 1])
def test_offline_b_only_slab_group(G, recovery):
    from tests.test_gpu_parity import _group_run
    p = make_problem("cfg3", nx=96, ny=80, nz=24, sweeps=18, mode=2, delta=6, recovery=recovery,
                     checksums=1)
    faults = [Fault(1, 11, 7, 9, 24), Fault(7, 0, 79, 95, 30), Fault(13, 23, 0, 0, 28), Fault(13, 5, 5, 5, 29)]
    o = oracle_run(p, faults=faults)
    g = _group_run(p, G, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])
    for s in g["stats"]:
        for k in ("sweeps", "rollbacks", "windows", "persistent"):
            assert s[k] == o["stats"][k], (k, s, o["stats"])
