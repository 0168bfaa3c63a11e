"""Multi-process (world_size 2 and 3, gloo on CPU) checks of the z-slab
decomposition's host logic (paper_1909_00709_b200/dist.py):
the partition, the halo plan (which layers and which checksum rows cross a
face), deadlock-free exchange ordering and max-over-ranks timing.  The
per-slab compute is the ORACLE on an extended slab [halo, slab, halo]; the
claim checked is the one the GPU path relies on: per-layer
arithmetic does not depend on the partition, so slabs + halos reproduce the
single domain bitwise -- field, actual checksums (Eqs. 2-3) and predicted
checksums (Theorem 1) of every layer, every sweep.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from abft_inputs import Fault, field_power, field_u0, make_problem
from oracle import oracle as O
from paper_1909_00709_b200 import dist as D


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reference(p, u0, P, nsweeps, faults):
    """single domain: per sweep (u, A, B, PA, PB) with the oracle"""
    op = O.OProblem(p, [P])
    u = u0
    A, B = O.checksums(op, u)
    out = []
    for s in range(1, nsweeps + 1):
        un = O.sweep(op, u, s, [f for f in faults if f.sweep == s])
        PA, PB = O.predict(op, A, B, u)
        A, B = O.checksums(op, un)
        out.append((un, A, B, PA, PB))
        u = un
    return out


def _worker(rank, world, port, nz, nsweeps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_problem("cfg3", nx=24, ny=20, nz=nz, sweeps=nsweeps)
        u0 = field_u0(p).numpy()
        P = field_power(p).numpy()
        faults = [Fault(2, nz // 2, 7, 9, 29), Fault(3, 0, 0, 23, 30), Fault(3, nz - 1, 19, 0, 28)]
        ref = _reference(p, u0, P, nsweeps, faults)

        z0, zc = D.slab(nz, world, rank)
        lo, hi = D.neighbours(rank, world)
        plan = D.halo_plan(rank, world, zc)
        # extended slab: buffer layers 0..zc+1, halo layers at 0 and zc+1
        ue = np.zeros((zc + 2, p.ny, p.nx), np.float32)
        ue[1:zc + 1] = u0[z0:z0 + zc]
        Pe = P[[min(max(z, 0), nz - 1) for z in range(z0 - 1, z0 + zc + 1)]]
        pe = p.replace(nz=zc + 2)
        ope = O.OProblem(pe, [Pe])
        Ae, Be = O.checksums(ope, ue)

        def halo():
            def send(peer, layer):
                dist.send(torch.from_numpy(ue[layer].copy()), peer)
                dist.send(torch.from_numpy(np.concatenate([Ae[layer], Be[layer]])), peer)

            def recv(peer, layer):
                t = torch.empty((p.ny, p.nx), dtype=torch.float32)
                dist.recv(t, peer)
                ue[layer] = t.numpy()
                v = torch.empty(p.nx + p.ny, dtype=torch.float64)
                dist.recv(v, peer)
                Ae[layer], Be[layer] = v[:p.nx].numpy(), v[p.nx:].numpy()

            D.exchange(rank, plan, send, recv)
            # global faces: the clamp of P:289-292 reuses the edge layer
            if lo is None:
                ue[0], Ae[0], Be[0] = ue[1], Ae[1], Be[1]
            if hi is None:
                ue[zc + 1], Ae[zc + 1], Be[zc + 1] = ue[zc], Ae[zc], Be[zc]

        halo()
        for s in range(1, nsweeps + 1):
            mine = [Fault(f.sweep, f.z - z0 + 1, f.y, f.x, f.bit) for f in faults
                    if f.sweep == s and z0 <= f.z < z0 + zc]
            un = O.sweep(ope, ue, s, mine)
            PA, PB = O.predict(ope, Ae, Be, ue)
            An, Bn = O.checksums(ope, un)
            ru, rA, rB, rPA, rPB = ref[s - 1]
            sl = slice(1, zc + 1)
            assert np.array_equal(un[sl].view(np.uint32), ru[z0:z0 + zc].view(np.uint32)), (rank, s)
            assert np.array_equal(An[sl], rA[z0:z0 + zc]) and np.array_equal(Bn[sl], rB[z0:z0 + zc])
            assert np.array_equal(PA[sl], rPA[z0:z0 + zc]) and np.array_equal(PB[sl], rPB[z0:z0 + zc])
            ue[sl], Ae[sl], Be[sl] = un[sl], An[sl], Bn[sl]
            halo()
        # bench timing rule: the slowest rank defines the step
        assert D.max_over_ranks(float(rank + 1), world) == float(world)
        assert D.sum_over_ranks(float(zc), world) == float(nz)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz", [(2, 8), (2, 7), (3, 11)])
def test_slab_halo_protocol_reproduces_single_domain(world, nz):
    mp.spawn(_worker, args=(world, _port(), nz, 4), nprocs=world, join=True)


def _partial_worker(rank, world, port, nz, L):
    """One dirty offline window of L sweeps recovered by slabs: the flagged
    layers reduced over ranks, the re-execution plan of dist.py (ranges, cones
    per sweep, local pieces), layers outside the cones poisoned -- the result
    must be the single-domain oracle's partial re-execution bitwise."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = make_problem("cfg3", nx=24, ny=20, nz=nz, sweeps=L, mode=2, delta=L, recovery=1)
        u0 = field_u0(p).numpy()
        P = field_power(p).numpy()
        faults = [Fault(1, 2, 7, 9, 29), Fault(2, nz - 4, 3, 3, 30), Fault(1, nz // 2, 10, 10, 2)]
        ref = O.run(O.OProblem(p, [P]), u0, L, faults)          # single domain, recovery PARTIAL
        assert ref["stats"]["rollbacks"] == 1 and ref["stats"]["persistent"] == 0
        first = O.run(O.OProblem(p.replace(mode=0), [P]), u0, L, faults)["u"]   # the first execution
        flagged_ref = sorted(r["z"] for r in ref["records"])

        z0, zc = D.slab(nz, world, rank)
        flagged = D.flagged_over_ranks([z for z in flagged_ref if z0 <= z < z0 + zc], nz, world)
        assert flagged == flagged_ref
        ranges = D.reexecution_ranges(flagged, L, nz)
        assert len(ranges) == 2                                  # two clusters, far apart
        r = 2 * (L - 1)
        inside = lambda z, rs: any(lo <= z <= hi for lo, hi in rs)
        assert all(inside(z, ranges) == any(abs(z - f) <= r for f in flagged) for z in range(nz))

        lo, hi = D.neighbours(rank, world)
        plan = D.halo_plan(rank, world, zc)
        ue = np.zeros((zc + 2, p.ny, p.nx), np.float32)
        ue[1:zc + 1] = u0[z0:z0 + zc]
        Pe = P[[min(max(z, 0), nz - 1) for z in range(z0 - 1, z0 + zc + 1)]]
        ope = O.OProblem(p.replace(nz=zc + 2, mode=0), [Pe])

        def halo():
            def send(peer, layer):
                dist.send(torch.from_numpy(ue[layer].copy()), peer)

            def recv(peer, layer):
                t = torch.empty((p.ny, p.nx), dtype=torch.float32)
                dist.recv(t, peer)
                ue[layer] = t.numpy()

            D.exchange(rank, plan, send, recv)
            if lo is None:
                ue[0] = ue[1]
            if hi is None:
                ue[zc + 1] = ue[zc]

        halo()
        for k in range(1, L + 1):
            cs = D.cones(ranges, k, L, nz)
            assert all(inside(z, cs) == any(lo_ - (L - k) <= z <= hi_ + (L - k) for lo_, hi_ in ranges)
                       for z in range(nz))
            un = O.sweep(ope, ue, k, [])                         # transient faults do not strike again
            nxt = np.full_like(ue, np.nan)                       # layers outside the cones: never read
            for za, zb in D.local_pieces(cs, z0, zc):
                nxt[1 + za:1 + zb] = un[1 + za:1 + zb]
            ue = nxt
            halo()
        out = first[z0:z0 + zc].copy()
        for za, zb in D.local_pieces(ranges, z0, zc):
            out[za:zb] = ue[1 + za:1 + zb]
        assert np.array_equal(out.view(np.uint32), ref["u"][z0:z0 + zc].view(np.uint32)), rank
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz", [(2, 32), (3, 31)])
def test_partial_reexecution_plan_over_slabs(world, nz):
    mp.spawn(_partial_worker, args=(world, _port(), nz, 3), nprocs=world, join=True)


def test_reexecution_ranges_and_cones():
    assert D.widen([(3, 3), (5, 5), (20, 21)], 1, 24) == [(2, 6), (19, 22)]
    assert D.widen([(0, 0), (23, 23)], 4, 24) == [(0, 4), (19, 23)]
    assert D.reexecution_ranges([3, 44], 3, 48) == [(0, 7), (40, 47)]
    assert D.reexecution_ranges([3, 11], 3, 48) == [(0, 15)]              # neighbourhoods meet
    assert D.reexecution_ranges([10], 1, 48) == [(10, 10)]                # L = 1: the layer alone
    assert D.reexecution_ranges([3, 30], 3, 48, periodic=True) == [(0, 47)]
    assert D.reexecution_ranges([10, 30], 3, 48, periodic=True) == [(6, 14), (26, 34)]
    assert D.cones([(0, 7), (40, 47)], 1, 3, 48) == [(0, 9), (38, 47)]
    assert D.cones([(6, 14), (18, 20)], 1, 3, 48) == [(4, 22)]            # cones merge, ranges do not
    assert D.local_pieces([(0, 9), (38, 47)], 8, 32) == [(0, 2), (30, 32)]
    assert D.local_pieces([(0, 9)], 16, 8) == []


def test_reexecution_plan_against_brute_force():
    # random flagged sets: the ranges are exactly the layers within 2 (L - 1)
    # of a flag, ascending, disjoint and not adjacent; sweep k's cones are
    # exactly the layers within L - k of a range; the slabs' pieces tile them
    rng = np.random.default_rng(7)
    for _ in range(200):
        nz = int(rng.integers(1, 70))
        L = int(rng.integers(1, 7))
        flagged = sorted(set(int(z) for z in rng.integers(0, nz, size=int(rng.integers(1, 6)))))
        rs = D.reexecution_ranges(flagged, L, nz)
        want = {z for z in range(nz) if any(abs(z - f) <= 2 * (L - 1) for f in flagged)}
        assert {z for lo, hi in rs for z in range(lo, hi + 1)} == want
        assert all(a[1] + 1 < b[0] for a, b in zip(rs, rs[1:])) and all(lo <= hi for lo, hi in rs)
        for k in range(1, L + 1):
            cs = D.cones(rs, k, L, nz)
            cw = {z for z in range(nz) if any(lo - (L - k) <= z <= hi + (L - k) for lo, hi in rs)}
            assert {z for lo, hi in cs for z in range(lo, hi + 1)} == cw
            world = int(rng.integers(1, min(nz, 5) + 1))
            got = set()
            for r in range(world):
                z0, zc = D.slab(nz, world, r)
                for za, zb in D.local_pieces(cs, z0, zc):
                    assert 0 <= za < zb <= zc
                    got |= {z0 + z for z in range(za, zb)}
            assert got == cw
        assert D.cones(rs, L, L, nz) == rs


def test_partition_and_plan():
    for nz, world in [(1024, 8), (11, 3), (7, 7), (1000, 3)]:
        parts = [D.slab(nz, world, r) for r in range(world)]
        assert parts[0][0] == 0 and sum(c for _, c in parts) == nz
        assert all(a[0] + a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    assert D.halo_plan(0, 1, 5) == []
    assert D.halo_plan(0, 2, 5) == [(1, 5, 6)]
    assert D.halo_plan(1, 2, 3) == [(0, 1, 0)]
    assert D.halo_plan(1, 3, 3) == [(0, 1, 0), (2, 3, 4)]
    with pytest.raises(ValueError):
        D.slab(3, 4, 0)
    assert D.weak_nz(1024, 8) == 8192


def test_bench_reference_arm_under_torchrun_two_ranks():
    # the driver's N>1 launch: rank 0 alone prints the reference line, rank 1 exits 0
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--impl",
           "reference", "--gpus", "2", "--config", "cfg1", "--steps", "2", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
