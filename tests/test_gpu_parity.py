"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
the same seeded inputs and fault schedules.  Bar (BASELINE.json north_star,
DESIGN.md §Parity): detected / located / corrected indices bit-exact; fp32
field values and checksums bitwise (every decision input is computed in the
same order or exactly); fp64 fields within 1e-12, checksums within 1e-13.
"""
import random

import numpy as np
import pytest
import torch

from abft_inputs import Fault, Problem, fault_schedule, field_power, field_u0, make_problem
from tests.parity_util import (assert_field_equal, gpu_run, oracle_run, parity)

pytestmark = pytest.mark.gpu


def setup_module(module):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")




# ---- BASELINE.json configs at their own size (cfg1, cfg2) ------------------

def test_cfg1_online_with_its_flip():
    g, o = parity(make_problem("cfg1"))
    assert g["launches"] > 0


@pytest.mark.parametrize("seed", range(1, 13))
def test_cfg1_seeds(seed):
    # seeds exercise benign (bits 0-12) and detectable flips
    parity(make_problem("cfg1", seed=seed))


def test_cfg2_full_online_10_flips():
    g, o = parity(make_problem("cfg2"))
    assert o["stats"]["corrected"] >= 1


def test_cfg2_explicit_api_matches_fused_step():
    p = make_problem("cfg2", sweeps=30, nz=4)
    parity(p, explicit=True)


# ---- reduced cfg3 / cfg5, ragged tiles, degenerate shapes --------------------

def test_cfg3_reduced_online():
    parity(make_problem("cfg3", nz=12, sweeps=60, nfaults=8))


def test_cfg3_reduced_offline_rollback():
    p = make_problem("cfg3", nz=12, sweeps=60, nfaults=8, mode=2, delta=10)
    g, o = parity(p)
    assert o["stats"]["rollbacks"] >= 1


def test_offline_last_window_shorter_than_delta():
    p = make_problem("cfg3", nx=128, ny=96, nz=5, sweeps=23, nfaults=4, mode=2, delta=10)
    parity(p)


@pytest.mark.parametrize("nx,ny,nz", [(203, 77, 9), (129, 33, 3), (64, 100, 2), (5, 3, 4),
                                      (1, 1, 1), (1, 7, 3), (9, 1, 2), (260, 1, 1)])
def test_hotspot_ragged_and_degenerate_shapes(nx, ny, nz):
    p = make_problem("cfg2", nx=nx, ny=ny, nz=nz, sweeps=25, nfaults=2)
    faults = [Fault(7, nz - 1, ny - 1, nx - 1, 30), Fault(15, 0, 0, 0, 27)]
    parity(p, faults=faults)


@pytest.mark.parametrize("nx,ny", [(64, 64), (70, 45), (128, 33), (1, 1)])
def test_fig2_five_point_2d(nx, ny):
    p = make_problem("cfg1", nx=nx, ny=ny, sweeps=20)
    parity(p, faults=[Fault(10, 0, ny // 2, nx // 3, 29)])


def test_cfg5_reduced_fp64_box27_offline():
    p = make_problem("cfg5", nx=130, ny=67, nz=12, sweeps=20, nfaults=6)
    g, o = parity(p)


def test_cfg5_reduced_fp64_box27_online():
    p = make_problem("cfg5", nx=66, ny=40, nz=7, sweeps=15, nfaults=5, mode=1)
    parity(p)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("seed", [0, 1])
def test_generic_stencil_random_order(dtype, seed):
    # an arbitrary radius-1 point list in arbitrary order runs the generic kernel
    rng = random.Random(seed)
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    rng.shuffle(offs)
    k = rng.randint(4, 15)
    w = [rng.uniform(0.01, 1.0) for _ in range(k)]
    s = sum(w)
    pts = [(a, b, c, v / s) for (a, b, c), v in zip(offs[:k], w)]
    p = Problem("gen", 150, 61, 6, dtype, pts, [(0.002, True, 0.0), (0.5, False, 3.0)],
                eps=1e-5 if dtype == "f32" else 1e-10, mode=1, sweeps=12, init=(1.0, 2.0),
                power=(0.0, 1.0))
    faults = [Fault(3, 2, 30, 70, 30 if dtype == "f32" else 62), Fault(9, 5, 60, 149, 27)]
    parity(p, faults=faults)


def test_correction_literal_form_runs():
    p = make_problem("cfg1", sweeps=12, correction_form=1)
    g = gpu_run(p, faults=[Fault(5, 0, 10, 10, 25)])
    o = oracle_run(p, faults=[Fault(5, 0, 10, 10, 25)])
    assert [r["x"] for r in g["records"]] == [r["x"] for r in o["records"]]


# ---- non-interference: protection does not change the sweep (SPEC #3) -------

def test_protected_field_equals_unprotected_field():
    p = make_problem("cfg2", nz=6, sweeps=40)
    g1 = gpu_run(p, faults=[])
    g0 = gpu_run(p.replace(mode=0), faults=[])
    assert np.array_equal(g1["u"].view(np.uint32), g0["u"].view(np.uint32))
    assert g1["stats"]["detections"] == 0
    assert np.array_equal(g1["A"], g0["A"]) and np.array_equal(g1["B"], g0["B"])


# ---- full-size cfg4 in the launch configuration bench.py times ---------------

def test_cfg4_full_size_sampled_and_properties():
    p = make_problem("cfg4")
    dev = torch.device("cuda:0")
    from paper_1909_00709_b200 import abft
    from oracle import oracle as O
    u0 = field_u0(p, dev)
    P = field_power(p, dev)
    # (a) one sweep: sampled layers against the oracle, computed layer by layer
    st = abft.from_problem(p, u0, P, device=dev)
    st.step(1)
    u1 = st.read_field()
    A1, B1 = st.checksums()
    st.destroy()
    for z in (0, 1, 511, 1022, 1023):
        lo, hi = max(0, z - 1), min(p.nz - 1, z + 1)
        sub = p.replace(nz=hi - lo + 1)
        op = O.OProblem(sub, [P[lo:hi + 1].cpu().numpy()])
        ref = O.sweep(op, u0[lo:hi + 1].cpu().numpy())[z - lo]
        got = u1[z].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), z
        Ar, Br = O.checksums(O.OProblem(sub.replace(nz=1, sources=[], power=None)), ref[None])
        assert np.array_equal(A1[z].numpy(), Ar[0]) and np.array_equal(B1[z].numpy(), Br[0])
    del u1
    # (b) 200 sweeps with the cfg4 schedule: every record is a scheduled flip at
    # the injected cell; high-bit flips are all located; the corrected run stays
    # within the correction residual of the fault-free run.
    faults = fault_schedule(p)
    st = abft.from_problem(p, u0, P, device=dev)
    st.set_faults(faults)
    st.step(p.sweeps)
    recs = st.records()
    uf = st.read_field()
    st.destroy()
    sched = {(f.sweep, f.z): f for f in faults}
    for r in recs:
        f = sched[(r["sweep"], r["z"])]          # no false positive
        if r["status"] == 1:
            assert (r["y"], r["x"]) == (f.y, f.x), r
        else:                                     # borderline: only one vector flagged
            assert r["status"] == 2 and (r["y"] == f.y or r["x"] == f.x), r
    hi = [f for f in faults if f.bit >= 21]
    got = {(r["sweep"], r["z"]) for r in recs}
    assert all((f.sweep, f.z) in got for f in hi)
    st = abft.from_problem(p, u0, P, device=dev)
    st.step(p.sweeps)
    uc = st.read_field()
    st.destroy()
    rel = ((uf - uc).abs() / uc.abs()).max().item()
    assert rel < 1e-2, rel   # undetected low-bit flips diffuse; detected ones are repaired


# ---- z-slab decomposition on one GPU (local group: device-copy halos) --------

def _split(nz, G, uneven):
    if uneven and G == 2:
        return [(0, nz // 2 - 1), (nz // 2 - 1, nz - nz // 2 + 1)]
    base = [nz // G + (1 if i < nz % G else 0) for i in range(G)]
    out, z = [], 0
    for c in base:
        out.append((z, c))
        z += c
    return out


def _group_run(p, G, faults, uneven=False):
    from paper_1909_00709_b200 import abft
    dev = torch.device("cuda:0")
    u0 = field_u0(p, dev)
    P = field_power(p, dev)
    sts = []
    for i, (z0, zc) in enumerate(_split(p.nz, G, uneven)):
        st = abft.from_problem(p, u0[z0:z0 + zc].contiguous(),
                               None if P is None else P[z0:z0 + zc].contiguous(), device=dev,
                               stream=torch.cuda.Stream(dev), z_begin=z0, z_count=zc, rank=i,
                               nranks=G)
        st.set_faults(faults)
        sts.append(st)
    abft.group(sts)
    status = abft.step_group(sts, p.sweeps)
    u = np.concatenate([s.read_field().cpu().numpy() for s in sts])
    recs = sum((s.records() for s in sts), [])
    stats = [s.stats() for s in sts]
    AB = [s.checksums() for s in sts]
    A = np.concatenate([a.numpy() for a, b in AB])
    B = np.concatenate([b.numpy() for a, b in AB])
    for s in sts:
        s.destroy()
    return dict(u=u, records=recs, stats=stats, status=status, A=A, B=B)


@pytest.fixture(params=["fused", "copy"])
def halo(request, monkeypatch):
    """Local groups exchange halos either inside the kernels (fused: boundary
    layers, checksum rows and corrections stored into the neighbours' slots)
    or by device copies after each sweep (ABFT_GROUP_COPY=1)."""
    if request.param == "copy":
        monkeypatch.setenv("ABFT_GROUP_COPY", "1")
    else:
        monkeypatch.delenv("ABFT_GROUP_COPY", raising=False)
    return request.param


@pytest.mark.parametrize("G,uneven", [(2, False), (2, True), (3, False), (4, False)])
@pytest.mark.parametrize("mode", [1, 2])
def test_slab_group_equals_oracle(G, uneven, mode, halo):
    # per-layer arithmetic does not depend on the partition, so
    # any z-slab decomposition is bitwise identical to the single domain.
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=30, nfaults=8, mode=mode, delta=7)
    faults = fault_schedule(p)
    faults += [Fault(9, 5, 3, 4, 30), Fault(9, 6, 70, 90, 29)]   # next to a slab face
    o = oracle_run(p, faults=faults)
    g = _group_run(p, G, faults, uneven)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])
    for s in g["stats"]:
        for k in ("sweeps", "rollbacks", "windows", "persistent"):
            assert s[k] == o["stats"][k], (k, s, o["stats"])
    for k in ("detections", "corrected", "located"):
        assert sum(s[k] for s in g["stats"]) == o["stats"][k]


def test_slab_group_fp64_box27_offline(halo):
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg5", nx=70, ny=33, nz=9, sweeps=15, nfaults=6)
    faults = fault_schedule(p)
    o = oracle_run(p, faults=faults)
    g = _group_run(p, 3, faults)
    rel = np.abs(g["u"] - o["u"]) / np.abs(o["u"])
    assert rel.max() <= 1e-12
    assert_records_equal(g, o, exact_values=False, rtol=1e-12)


# ---- tiles: several z-chunks and x/y tiles, flips on chunk and tile edges -----

@pytest.mark.parametrize("nx,ny,nz", [(300, 200, 70), (129, 47, 33), (64, 16, 96)])
def test_tile_and_chunk_edges(nx, ny, nz):
    p = make_problem("cfg3", nx=nx, ny=ny, nz=nz, sweeps=16, nfaults=0)
    zs = sorted({0, 15, 16, 31, 32, min(63, nz - 1), nz - 1})
    faults = [Fault(2 + i, z, (7 * i) % ny, (37 * i + 127) % nx, 30 - i) for i, z in enumerate(zs)]
    faults += [Fault(9, nz // 2, ny - 1, nx - 1, 29), Fault(12, nz // 3, 0, 128 % nx, 28)]
    faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())
    parity(p, faults=faults)


# ---- checksum policy LAZY: b every sweep, a on detection

@pytest.mark.parametrize("seed", range(0, 8))
def test_lazy_cfg1_seeds(seed):
    parity(make_problem("cfg1", seed=seed, checksums=1))


def test_lazy_cfg2_full_online_10_flips():
    g, o = parity(make_problem("cfg2", checksums=1))
    assert o["stats"]["corrected"] >= 1


@pytest.mark.parametrize("nx,ny,nz", [(203, 77, 9), (129, 33, 3), (5, 3, 4), (1, 1, 1), (260, 1, 2)])
def test_lazy_hotspot_ragged_shapes(nx, ny, nz):
    p = make_problem("cfg2", nx=nx, ny=ny, nz=nz, sweeps=25, nfaults=2, checksums=1)
    faults = [Fault(7, nz - 1, ny - 1, nx - 1, 30), Fault(15, 0, 0, 0, 27), Fault(15, nz // 2, ny // 2, nx // 2, 28)]
    faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())   # one flip per cell and sweep
    parity(p, faults=faults)


def test_lazy_many_flagged_layers_in_one_sweep():
    # more flagged layers than K3's concurrent slots: every one is handled
    p = make_problem("cfg3", nx=96, ny=64, nz=20, sweeps=6, nfaults=0, checksums=1)
    faults = [Fault(3, z, (5 * z) % 64, (11 * z) % 96, 29) for z in range(20)]
    faults += [Fault(5, z, 0, 95, 30) for z in range(0, 20, 3)]
    g, o = parity(p, faults=faults)
    assert o["stats"]["corrected"] >= 20


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_lazy_generic_stencil(dtype):
    rng = random.Random(7)
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    rng.shuffle(offs)
    w = [rng.uniform(0.01, 1.0) for _ in range(9)]
    pts = [(a, b, c, v / sum(w)) for (a, b, c), v in zip(offs[:9], w)]
    p = Problem("gen", 150, 61, 6, dtype, pts, [(0.002, True, 0.0)],
                eps=1e-5 if dtype == "f32" else 1e-10, mode=1, sweeps=12, init=(1.0, 2.0),
                power=(0.0, 1.0), checksums=1)
    faults = [Fault(3, 2, 30, 70, 30 if dtype == "f32" else 62), Fault(9, 5, 60, 149, 27)]
    parity(p, faults=faults)


def test_lazy_cfg5_reduced_fp64_box27_online():
    parity(make_problem("cfg5", nx=66, ny=40, nz=7, sweeps=15, nfaults=5, mode=1, checksums=1))


@pytest.mark.parametrize("G", [2, 3])
def test_lazy_slab_group_equals_oracle(G, halo):
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=30, nfaults=8, mode=1, checksums=1)
    faults = fault_schedule(p) + [Fault(9, 5, 3, 4, 30), Fault(9, 6, 70, 90, 29), Fault(11, 4, 0, 0, 30)]
    o = oracle_run(p, faults=faults)
    g = _group_run(p, G, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])


def test_set_faults_rejects_overfull_sweeps():
    from paper_1909_00709_b200 import abft
    p = make_problem("cfg2", nx=64, ny=64, nz=80, sweeps=2)
    dev = torch.device("cuda:0")
    st = abft.from_problem(p, field_u0(p, dev), field_power(p, dev), device=dev)
    st.set_faults([Fault(1, 3, 4, 5, 20), Fault(1, 3, 4, 5, 21)])   # a repeat strikes a re-execution
    with pytest.raises(abft.AbftError):
        st.set_faults([Fault(1, 3, 4, 5, 20)] * 65)
    with pytest.raises(abft.AbftError):
        st.set_faults([Fault(1, z, 0, 0, 20) for z in range(65)])
    st.set_faults([Fault(1, z, 0, 0, 20) for z in range(64)] + [Fault(2, 0, 0, 0, 20)])
    st.destroy()


# ---- boundary conditions (P:289-292 clamp; P:407-415 periodic, zero, constant) --

BCS = [(1, 0.0), (2, 0.0), (3, 331.5)]


@pytest.mark.parametrize("bc,g", BCS)
@pytest.mark.parametrize("nx,ny,nz", [(203, 77, 9), (128, 64, 5), (5, 3, 4), (1, 1, 2)])
def test_bc_hotspot_online(bc, g, nx, ny, nz):
    p = make_problem("cfg2", nx=nx, ny=ny, nz=nz, sweeps=20, nfaults=0, bc=bc, bc_value=g)
    faults = [Fault(5, nz - 1, ny - 1, nx - 1, 29), Fault(9, 0, 0, 0, 28), Fault(13, nz // 2, ny // 2, nx // 2, 27)]
    faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())
    parity(p, faults=faults)


@pytest.mark.parametrize("bc,g", BCS)
def test_bc_fig2_five_point_2d(bc, g):
    p = make_problem("cfg1", nx=70, ny=45, sweeps=20, bc=bc, bc_value=0.25 if bc == 3 else g)
    parity(p, faults=[Fault(10, 0, 0, 69, 29), Fault(14, 0, 22, 0, 28)])


@pytest.mark.parametrize("bc,g", BCS)
def test_bc_offline_and_lazy(bc, g):
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=24, nfaults=6, mode=2, delta=6, bc=bc, bc_value=g)
    parity(p)
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=24, nfaults=6, mode=1, bc=bc, bc_value=g,
                     checksums=1)
    parity(p, faults=fault_schedule(p) + [Fault(7, 0, 0, 0, 30), Fault(9, 11, 79, 95, 29)])


@pytest.mark.parametrize("bc,g", BCS)
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_bc_generic_and_box27(bc, g, dtype):
    rng = random.Random(bc)
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    rng.shuffle(offs)
    w = [rng.uniform(0.01, 1.0) for _ in range(11)]
    pts = [(a, b, c, v / sum(w)) for (a, b, c), v in zip(offs[:11], w)]
    p = Problem("gen", 70, 33, 5, dtype, pts, [(0.002, True, 0.0)],
                eps=1e-5 if dtype == "f32" else 1e-10, mode=1, sweeps=10, init=(1.0, 2.0),
                power=(0.0, 1.0), bc=bc, bc_value=1.5 if bc == 3 else g)
    parity(p, faults=[Fault(3, 0, 0, 69, 30 if dtype == "f32" else 62), Fault(7, 4, 32, 0, 29)])
    q = make_problem("cfg5", nx=40, ny=24, nz=6, sweeps=10, nfaults=4, mode=1, bc=bc, bc_value=0.5 if bc == 3 else g)
    if dtype == "f64":
        parity(q)


@pytest.mark.parametrize("bc", [2, 3])
def test_bc_slab_group(bc, halo):
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=20, nfaults=6, mode=1, bc=bc, bc_value=330.0)
    faults = fault_schedule(p) + [Fault(9, 5, 3, 4, 30), Fault(9, 6, 70, 90, 29)]
    o = oracle_run(p, faults=faults)
    g = _group_run(p, 3, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)


@pytest.mark.parametrize("G,mode", [(2, 1), (3, 1), (2, 2), (3, 2)])
def test_bc_periodic_ring_of_slabs(G, mode, halo):
    # periodic z over several slabs closes the ring: slab 0 and the last slab
    # exchange halos (a ring of two: one neighbour on both faces)
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=12, sweeps=20, nfaults=6, mode=mode, delta=5, bc=1)
    faults = fault_schedule(p) + [Fault(9, 0, 3, 4, 30), Fault(9, 11, 70, 90, 29)]
    faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())
    o = oracle_run(p, faults=faults)
    g = _group_run(p, G, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])


# ---- correction_form 2: recompute the located cell (stencil locality)

@pytest.mark.parametrize("name,kw", [
    ("cfg1", dict(sweeps=20)),
    ("cfg2", dict(nx=203, ny=77, nz=9, sweeps=25, nfaults=4)),
    ("cfg2", dict(nx=128, ny=64, nz=5, sweeps=20, nfaults=3, bc=1)),
    ("cfg2", dict(nx=128, ny=64, nz=5, sweeps=20, nfaults=3, bc=3, bc_value=330.0)),
    ("cfg2", dict(nx=96, ny=80, nz=12, sweeps=30, nfaults=8, checksums=1)),
    ("cfg5", dict(nx=40, ny=24, nz=6, sweeps=10, nfaults=4, mode=1)),
])
def test_recompute_correction(name, kw):
    p = make_problem(name, **kw).replace(correction_form=2)
    faults = [f for f in fault_schedule(p) if f.bit >= (27 if p.dtype == "f32" else 59)]
    faults = faults + [Fault(3, 0, 0, 0, 30 if p.dtype == "f32" else 62)]
    faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())
    g, o = parity(p, faults=faults)
    ref = gpu_run(p, faults=[])
    if g["stats"]["corrected"] == len(faults):     # every flip located: exact repair
        w = np.uint32 if p.dtype == "f32" else np.uint64
        assert np.array_equal(g["u"].view(w), ref["u"].view(w))


# ---- correction_form 2 beyond one intersection: layer recompute (Q27)

from paper_1909_00709_b200 import abft  # noqa: E402

@pytest.mark.parametrize("cells", [((7, 9), (20, 31)), ((7, 9), (7, 31)), ((7, 9), (20, 9), (33, 2)),
                                   ((0, 0), (35, 39))])
@pytest.mark.parametrize("checksums", [0, 1])
def test_recompute_layer_several_flips(cells, checksums):
    p = make_problem("cfg2", nx=40, ny=36, nz=4, sweeps=6, checksums=checksums, correction_form=2)
    faults = [Fault(4, z, y, x, 29) for z in (0, 3) for y, x in cells]
    g, o = parity(p, faults=faults)
    assert g["stats"]["corrected"] == len(faults)
    assert all(r["status"] == abft.REC_RECOMPUTED for r in g["records"])
    ref = gpu_run(p, faults=[])
    assert np.array_equal(g["u"].view(np.uint32), ref["u"].view(np.uint32))


@pytest.mark.parametrize("name,kw", [
    ("cfg2", dict(nx=203, ny=77, nz=9, sweeps=8)),
    ("cfg5", dict(nx=40, ny=24, nz=6, sweeps=6, mode=1)),
])
def test_recompute_layer_ragged(name, kw):
    # ragged tiles, several layers at once (one K2 CTA each), fp64 included
    p = make_problem(name, **kw).replace(correction_form=2)
    hi = 29 if p.dtype == "f32" else 61
    faults = [Fault(3, 1, 2, 5, hi), Fault(3, 1, 2, p.nx - 1, hi), Fault(3, 4, 0, 0, hi),
              Fault(3, 4, p.ny - 1, p.nx - 1, hi), Fault(5, p.nz - 1, 3, 3, hi), Fault(5, p.nz - 1, 9, 17, hi)]
    g, o = parity(p, faults=faults)
    assert g["stats"]["corrected"] == len(faults)


def test_recompute_false_alarm_verified():
    # eps far below the prediction's rounding: error-free layers flag; the
    # recompute finds nothing to rewrite and the field is the fault-free run's
    p = make_problem("cfg5", nx=40, ny=24, nz=6, sweeps=5, mode=1, nfaults=0)
    ref = gpu_run(p, faults=[])
    g = gpu_run(p.replace(correction_form=2, eps=1e-19), faults=[])
    assert g["stats"]["detections"] > 0 and g["stats"]["corrected"] == 0
    assert g["records"] and all(r["status"] == abft.REC_VERIFIED for r in g["records"])
    assert np.array_equal(g["u"].view(np.uint64), ref["u"].view(np.uint64))


def test_recompute_layer_explicit_api():
    # sweep() / check() / correct() (CK_SUMMARY then CK_FROM_SUMMARY) reach the
    # same layer recompute as step()
    p = make_problem("cfg2", nx=72, ny=40, nz=5, sweeps=6, correction_form=2)
    faults = [Fault(2, 1, 3, 4, 29), Fault(2, 1, 30, 60, 28), Fault(4, 4, 7, 7, 30), Fault(4, 4, 7, 50, 29)]
    o = oracle_run(p, faults=faults)
    g = gpu_run(p, faults=faults, explicit=True)
    assert_field_equal(g, o, "f32")
    assert sorted((r["sweep"], r["z"], r["y"], r["x"], r["status"]) for r in g["records"]) == \
        sorted((r["sweep"], r["z"], r["y"], r["x"], r["status"]) for r in o["records"])
    assert g["stats"]["corrected"] == len(faults)


# ---- forms 0 / 1: several flips in one layer (P:663-667 pairing, Q13 / Q14) --

@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("checksums", [0, 1])
def test_multi_flip_layer_uncorrectable_and_unlocated(form, checksums):
    # per layer and sweep: two flips in different rows and columns (a and b
    # flag twice: UNCORRECTABLE), two in one row (a twice, b once:
    # UNCORRECTABLE), and on a 1024 x 8 layer a flip above eps|a| but below
    # eps|b| (only a flags: UNLOCATED under BOTH).  Under LAZY the layer is
    # examined only when b flags, so the first two still report.
    p = make_problem("cfg2", nx=96, ny=80, nz=6, sweeps=8, correction_form=form, checksums=checksums)
    faults = [Fault(3, 1, 10, 20, 29), Fault(3, 1, 50, 70, 28),          # a: 2, b: 2
              Fault(5, 4, 33, 5, 29), Fault(5, 4, 33, 90, 30),           # a: 2, b: 1
              Fault(6, 2, 7, 7, 29)]                                     # single: corrected
    g, o = parity(p, faults=faults)
    st = sorted((r["sweep"], r["z"], r["status"]) for r in o["records"])
    assert (3, 1, abft.REC_UNCORRECTABLE) in st and (5, 4, abft.REC_UNCORRECTABLE) in st
    assert (6, 2, abft.REC_CORRECTED) in st
    assert g["status"] == abft.ABFT_DETECTED_UNCORRECTABLE
    # only one vector flags: rows of 1024 cells, columns of 8 (~333 each):
    # bit 12 of a value ~333 (delta 0.125) exceeds eps|a| ~ 0.027 but not eps|b| ~ 3.4
    q = make_problem("cfg2", nx=1024, ny=8, nz=3, sweeps=4, correction_form=form, checksums=checksums)
    g, o = parity(q, faults=[Fault(2, 1, 3, 500, 12)])
    if checksums == 0:
        assert [r["status"] for r in o["records"]] == [abft.REC_UNLOCATED]
    else:
        assert o["records"] == []       # b never flagged: the lazy check does not look at a
    # b-only under LAZY: columns of 1024 cells, rows of 8
    q = make_problem("cfg2", nx=8, ny=1024, nz=3, sweeps=4, correction_form=form, checksums=checksums)
    g, o = parity(q, faults=[Fault(2, 1, 500, 3, 12)])
    assert [r["status"] for r in o["records"]] == [abft.REC_UNLOCATED]


# ---- offline partial re-execution (recovery PARTIAL, Q28) ---------

@pytest.mark.parametrize("delta", [1, 3, 6])
def test_offline_partial_reexecution_equals_oracle(delta):
    p = make_problem("cfg3", nx=96, ny=80, nz=40, sweeps=4 * delta, mode=2, delta=delta, recovery=1)
    faults = [Fault(1, 11, 7, 9, 24), Fault(delta + 1, 0, 79, 95, 30), Fault(2 * delta + 1, 39, 0, 0, 28),
              Fault(3 * delta + 1, 5, 20, 20, 24), Fault(3 * delta + 1, 30, 3, 30, 29),
              Fault(4 * delta, 20, 40, 50, 3)]
    g, o = parity(p, faults=faults)
    assert o["stats"]["rollbacks"] == 4
    ref = gpu_run(p.replace(recovery=0), faults=faults)
    assert ref["stats"]["sweeps"] == g["stats"]["sweeps"]


def test_offline_partial_keeps_undetected_error_outside_the_cone():
    p = make_problem("cfg3", nx=40, ny=32, nz=24, sweeps=4, mode=2, delta=4, recovery=1)
    faults = [Fault(1, 2, 5, 5, 29), Fault(1, 20, 9, 9, 3)]
    g, o = parity(p, faults=faults)
    only_lo = gpu_run(p, faults=[faults[1]])
    assert np.array_equal(g["u"].view(np.uint32), only_lo["u"].view(np.uint32))


@pytest.mark.parametrize("recovery", [0, 1])
def test_offline_persistent_error(recovery):
    # the same flip listed twice strikes the window's execution and its
    # re-execution: the re-check still flags, PERSISTENT records
    p = make_problem("cfg3", nx=32, ny=32, nz=10, sweeps=10, mode=2, delta=5, recovery=recovery)
    g, o = parity(p, faults=[Fault(3, 1, 5, 5, 30), Fault(3, 1, 5, 5, 30)])
    assert o["status"] == 3 and o["stats"]["persistent"] == 1


def test_offline_partial_fp64_box27():
    p = make_problem("cfg5", nx=130, ny=67, nz=30, sweeps=20, nfaults=6, recovery=1)
    g, o = parity(p)
    assert o["stats"]["rollbacks"] >= 1


@pytest.mark.parametrize("G", [2, 3, 4])
def test_offline_partial_slab_group(G, halo):
    # the cone crosses slab faces: re-execution, halos and the re-check are collective
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=24, sweeps=18, mode=2, delta=6, recovery=1)
    faults = [Fault(1, 11, 7, 9, 24), Fault(7, 0, 79, 95, 30), Fault(13, 23, 0, 0, 28), Fault(13, 5, 5, 5, 29)]
    o = oracle_run(p, faults=faults)
    g = _group_run(p, G, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])
    for s in g["stats"]:
        for k in ("sweeps", "rollbacks", "windows", "persistent"):
            assert s[k] == o["stats"][k], (k, s, o["stats"])


@pytest.mark.parametrize("checksums", [0, 1])
@pytest.mark.parametrize("G", [1, 2, 4])
def test_offline_partial_union_of_cones(G, checksums, halo):
    # the oracle pin test_partial_reexecution_is_the_union_of_the_flagged_layers_neighbourhoods
    # at GPU scale: two clusters of flagged layers (3 and 44 of 48), an
    # undetected flip half way -- several re-executed ranges per sweep, on
    # one slab and across slab faces; the layers between keep the first
    # execution, so the result equals the run with the undetected flip alone
    from tests.parity_util import assert_records_equal
    p = make_problem("cfg3", nx=96, ny=80, nz=48, sweeps=6, mode=2, delta=3, recovery=1, checksums=checksums)
    lo = Fault(1, 24, 9, 9, 3)
    faults = [Fault(1, 3, 5, 5, 29), Fault(2, 44, 20, 11, 30), lo,
              Fault(5, 40, 70, 90, 29), Fault(4, 10, 1, 2, 30), Fault(6, 25, 33, 33, 28)]
    o = oracle_run(p, faults=faults)
    assert o["stats"]["rollbacks"] == 2 and o["stats"]["persistent"] == 0
    g = _group_run(p, G, faults) if G > 1 else gpu_run(p, faults=faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    if checksums == 0:
        assert np.array_equal(g["A"], o["A"])
    assert np.array_equal(g["B"], o["B"])
    only_lo = gpu_run(p, faults=[lo])
    assert only_lo["stats"]["rollbacks"] == 0
    assert np.array_equal(g["u"].view(np.uint32), only_lo["u"].view(np.uint32))


@pytest.mark.parametrize("bc,z0", [(0, 8), (1, 1)])
def test_offline_partial_reach_on_the_unflagged_side(bc, z0):
    # the oracle pin test_partial_reach_covers_errors_on_the_unflagged_side at
    # GPU scale (several x / y tiles): an upwind z stencil moves a flip's
    # error up, so only layer z0 + 2 flags while sub-threshold errors sit in
    # z0 and z0 - 2 (periodic: wrapped to the top) -- the re-executed range
    # must reach them (Q28); the result equals the full rollback's
    pts = [(0, 0, -1, 0.98), (0, 0, 1, 1e-4)]
    p = Problem("t", 70, 40, 16, "f64", pts, [], bc=bc, eps=1e-4, mode=2, delta=3, sweeps=6,
                init=(1.0, 2.0), recovery=1)
    faults = [Fault(1, z0, 3, 4, 50), Fault(4, 12, 30, 60, 50)]
    g, o = parity(p, faults=faults)
    assert o["stats"]["rollbacks"] == 2
    full = gpu_run(p.replace(recovery=0), faults=faults)
    assert np.array_equal(g["u"].view(np.uint64), full["u"].view(np.uint64))


def test_flag_in_one_vector_only_is_unlocated():
    # P:638 / Q14: the column sum flags, the row sum does not (see the oracle pin)
    for checksums in (0, 1):
        p = make_problem("cfg2", nx=256, ny=8, nz=2, sweeps=3, checksums=checksums)
        g, o = parity(p, faults=[Fault(2, 1, 5, 100, 12)])
        if checksums == 0:
            assert [r["status"] for r in o["records"]] == [2]
        else:   # b does not flag: the lazy policy never looks at a
            assert o["records"] == []
