"""GPU parity of the pipelined online schedule (abft_schedule AUTO, DESIGN.md
§6): the checks of sweep s run beside the stencil update of sweep s + 1,
which may read a cell of u^s before or after the checks rewrite it; the
kernel finishing the checks then recomputes the cells of u^{s+1} that read a
rewritten cell (fix_next).  Every result must be the oracle's -- the paper's
serial order (fig.abft caption: detect and correct after each sweep)
-- bitwise for fp32, within 1e-12 for fp64.  ABFT_PIPELINE=1 forces the
schedule on every single-slab online handle (by default only short K1
z-chunks take it); ABFT_GRAPHS=0 enqueues every call directly instead of
replaying a captured graph.
"""
import numpy as np
import pytest
import torch

from abft_inputs import Fault, Problem, fault_schedule, field_power, field_u0, make_problem
from tests.parity_util import (assert_checksums_close, assert_field_equal, assert_records_equal,
                               assert_stats_equal, gpu_run, oracle_run, parity)

pytestmark = pytest.mark.gpu


def setup_module(module):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(params=["graphs", "direct", "serial"])
def pipelined(request, monkeypatch):
    # "serial": the same cases under the serial schedule (the reference order)
    monkeypatch.setenv("ABFT_PIPELINE", "0" if request.param == "serial" else "1")
    monkeypatch.setenv("ABFT_GRAPHS", "1" if request.param == "graphs" else "0")
    return request.param


def _uniq(faults):
    return list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())


CASES = [
    ("cfg2", dict()),
    ("cfg2", dict(checksums=1)),
    ("cfg3", dict(nz=12, sweeps=40, nfaults=8)),
    ("cfg3", dict(nz=12, sweeps=40, nfaults=8, checksums=1)),
    ("cfg2", dict(nx=203, ny=77, nz=9, sweeps=25, nfaults=6)),
    ("cfg2", dict(nx=5, ny=3, nz=4, sweeps=20, nfaults=3)),
    ("cfg2", dict(nx=260, ny=1, nz=1, sweeps=20, nfaults=3)),
    ("cfg2", dict(nx=128, ny=64, nz=5, sweeps=20, nfaults=5, bc=1)),
    ("cfg2", dict(nx=128, ny=64, nz=5, sweeps=20, nfaults=5, bc=2)),
    ("cfg2", dict(nx=128, ny=64, nz=5, sweeps=20, nfaults=5, bc=3, bc_value=330.0)),
    ("cfg2", dict(nx=96, ny=80, nz=6, sweeps=20, nfaults=5, correction_form=1)),
    ("cfg2", dict(nx=96, ny=80, nz=6, sweeps=20, nfaults=5, correction_form=2)),
    ("cfg1", dict(sweeps=30)),
    ("cfg5", dict(nx=66, ny=40, nz=7, sweeps=15, nfaults=5, mode=1)),
    ("cfg5", dict(nx=66, ny=40, nz=7, sweeps=15, nfaults=5, mode=1, checksums=1, bc=1)),
]


@pytest.mark.parametrize("name,kw", CASES)
def test_pipelined_equals_oracle(name, kw, pipelined):
    parity(make_problem(name, **kw))


@pytest.mark.parametrize("checksums", [0, 1])
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("form", [0, 2])
def test_pipelined_consecutive_flips_next_to_each_other(checksums, bc, form, pipelined):
    # a flip in every sweep, each next to the previous one (and across the x /
    # y / z faces, where periodic neighbourhoods wrap): the next sweep reads a
    # corrected cell while it may still hold the flipped value (bits 28-30:
    # values up to ~1e38 that poison the speculative row sums)
    p = make_problem("cfg2", nx=64, ny=48, nz=6, sweeps=19, checksums=checksums, bc=bc,
                     correction_form=form)
    cells = [(0, 0, 0), (0, 0, 1), (1, 0, 1), (1, 47, 63), (0, 47, 63), (5, 47, 0), (5, 0, 0),
             (2, 20, 31), (2, 21, 31), (3, 21, 32), (3, 21, 33), (4, 22, 33), (5, 22, 32), (0, 23, 32)]
    faults = [Fault(s + 2, z, y, x, 28 + (s % 3)) for s, (z, y, x) in enumerate(cells)]
    # two flips in one sweep, in neighbouring layers at the same (y, x) (a
    # sweep with no other flip: one per layer keeps every flip correctable)
    faults += [Fault(16, 2, 10, 10, 30), Fault(16, 3, 10, 10, 29), Fault(17, 3, 10, 11, 28)]
    g, o = parity(p, faults=_uniq(faults))
    assert o["stats"]["corrected"] == len(faults)


@pytest.mark.parametrize("checksums", [0, 1])
@pytest.mark.parametrize("bc", [0, 1])
def test_pipelined_many_rewrites_in_one_sweep(checksums, bc, pipelined):
    # more rewritten cells in one sweep than the fix lists (kChgCap = 32): the
    # fix recomputes whole layers around them
    p = make_problem("cfg2", nx=48, ny=40, nz=40, sweeps=6, checksums=checksums, bc=bc)
    faults = [Fault(3, z, (7 * z) % 40, (11 * z) % 48, 29 + (z % 2)) for z in range(40)]
    faults += [Fault(4, z, 5, 5, 30) for z in range(0, 40, 3)]
    g, o = parity(p, faults=faults)
    assert o["stats"]["corrected"] >= 40


@pytest.mark.parametrize("checksums", [0, 1])
def test_pipelined_layer_recompute(checksums, pipelined):
    # correction_form 2 with flags that do not intersect in one cell: the
    # layer recompute rewrites several cells of u^s at once (Q27)
    p = make_problem("cfg2", nx=40, ny=36, nz=4, sweeps=8, checksums=checksums, correction_form=2)
    faults = [Fault(4, z, y, x, 29) for z in (0, 3) for y, x in ((7, 9), (20, 31), (33, 2))]
    faults += [Fault(5, 0, 8, 9, 30), Fault(5, 1, 7, 9, 28)]
    g, o = parity(p, faults=faults)
    assert g["stats"]["corrected"] == len(faults)


def _steps(p, calls, n, **kw):
    """One handle, `calls` x step(n): a graph captured on the first call of a
    phase is replayed by the later ones (records offset on the device)."""
    from paper_1909_00709_b200 import abft
    dev = torch.device("cuda:0")
    st = abft.from_problem(p, field_u0(p, dev), field_power(p, dev) if p.power is not None else None,
                           device=dev, **kw)
    st.set_faults([])
    for _ in range(calls):
        st.step(n)
    out = dict(u=st.read_field().cpu().numpy(), stats=st.stats(), records=st.records(),
               status=st.status(), launches=st.launches)
    A, B = st.checksums()
    out["A"], out["B"] = A.numpy(), B.numpy()
    st.destroy()
    return out


@pytest.mark.parametrize("checksums", [0, 1])
def test_graph_replays_record_the_right_sweeps(checksums, monkeypatch):
    # eps below the fp32 rounding of the sweep: every layer flags every sweep
    # (deterministically: fp32 data sum exactly in fp64), form 2 verifies it;
    # 3 x step(6) replays the first call's graph at sweeps 13-18 (the
    # rotation phase repeats every 12 sweeps), whose records must carry their
    # own sweep numbers
    monkeypatch.setenv("ABFT_PIPELINE", "1")
    monkeypatch.setenv("ABFT_GRAPHS", "1")
    p = make_problem("cfg2", nx=64, ny=48, nz=6, sweeps=18, checksums=checksums, correction_form=2,
                     eps=1e-12)
    o = oracle_run(p, faults=[])
    g = _steps(p, 3, 6)
    assert o["stats"]["detections"] > 0
    assert_field_equal(g, o, "f32")
    assert_records_equal(g, o)
    assert_stats_equal(g, o)
    assert max(r["sweep"] for r in g["records"]) == 18


@pytest.mark.parametrize("mode", [0, 1])
def test_graph_replays_equal_oracle(mode, monkeypatch):
    # unprotected and protected error-free calls replayed from cached graphs
    monkeypatch.setenv("ABFT_PIPELINE", "1")
    p = make_problem("cfg2", nx=100, ny=70, nz=5, sweeps=36, mode=mode)
    o = oracle_run(p, faults=[])
    g = _steps(p, 6, 6)
    assert_field_equal(g, o, "f32")
    if mode == 1:
        assert_checksums_close(g, o, 0.0)
        assert g["records"] == []


def test_plan_then_step_with_faults_enqueues_directly(monkeypatch):
    # a call whose range holds a flip never uses a graph (the flips are launch
    # parameters); plan() of such a call is a no-op
    monkeypatch.setenv("ABFT_PIPELINE", "1")
    from paper_1909_00709_b200 import abft
    p = make_problem("cfg2", nx=64, ny=48, nz=6, sweeps=12)
    faults = [Fault(8, 2, 10, 10, 30)]
    o = oracle_run(p, faults=faults)
    dev = torch.device("cuda:0")
    st = abft.from_problem(p, field_u0(p, dev), field_power(p, dev), device=dev)
    st.set_faults(faults)
    st.plan(6)
    st.step(6)          # error-free range: graph
    st.plan(6)          # holds the flip: no-op
    st.step(6)
    u = st.read_field().cpu().numpy()
    recs = st.records()
    st.destroy()
    assert np.array_equal(u.view(np.uint32), o["u"].view(np.uint32))
    assert [(r["sweep"], r["z"], r["y"], r["x"]) for r in recs] == [(8, 2, 10, 10)]


def test_serial_schedule_still_selectable(monkeypatch):
    monkeypatch.setenv("ABFT_PIPELINE", "1")
    parity(make_problem("cfg2", nz=6, sweeps=20), schedule=1)
