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
