"""One process per slab over CUDA IPC (abft_stencil_ipc_export / _link,
SURVEY NEXT-3): 2-4 processes, each owning a z-slab on cuda:0 (the only GPU
here; on a node each would own its own GPU and the stores would cross
NVLink), halos stored by the kernels into the neighbours' mapped buffers,
sweeps ordered by IPC events, offline verdicts reduced through the shared
progress slots.  The gathered result must equal the oracle of the undivided
domain bitwise (fp32) -- field, a, b, records -- online, lazy, offline with a
collective rollback, and offline with a partial re-execution whose cone
crosses slab faces.  The processes wait on each other only through stream
events (no kernel spins on another process), so sharing one GPU is safe.
"""
import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from abft_inputs import Fault, fault_schedule, field_power, field_u0, make_problem
from tests.parity_util import assert_records_equal, oracle_run

pytestmark = pytest.mark.gpu


def setup_module(module):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, pkw, faults, out_dir):
    import torch.distributed as dist
    from paper_1909_00709_b200 import abft, dist as D
    from paper_1909_00709_b200.ipc import IpcContext
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        name = pkw.pop("name")
        p = make_problem(name, **pkw)
        z0, zc = D.slab(p.nz, world, rank)
        ctx = IpcContext(rank, world)
        P = field_power(p, dev, z0, zc)
        st = abft.from_problem(p, field_u0(p, dev, z0, zc), P, device=dev,
                               stream=torch.cuda.Stream(dev), z_begin=z0, z_count=zc, rank=rank,
                               nranks=world)
        st.set_faults([Fault(*f) for f in faults])
        assert ctx.link(st)
        status = st.step(p.sweeps)
        u = st.read_field().cpu().numpy()
        A, B = st.checksums()
        res = dict(status=max(status, st.status()), stats=st.stats(), records=st.records(),
                   launches=st.launches)
        st.destroy()
        ctx.close()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u, A=A.numpy(), B=B.numpy())
        with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
            json.dump(res, f)
    finally:
        dist.destroy_process_group()


def _ipc_run(world, pkw, faults):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_rank_main, args=(world, _port(), dict(pkw), [tuple(vars(f).values()) for f in faults], d),
                           nprocs=world, join=True, start_method="spawn")
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
        meta = [json.load(open(os.path.join(d, f"r{r}.json"))) for r in range(world)]
    return dict(u=np.concatenate([x["u"] for x in parts]), A=np.concatenate([x["A"] for x in parts]),
                B=np.concatenate([x["B"] for x in parts]),
                records=sum((m["records"] for m in meta), []), stats=[m["stats"] for m in meta],
                status=max(m["status"] for m in meta), launches=[m["launches"] for m in meta])


CASES = {
    "online": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=30, nfaults=8, mode=1),
    "lazy": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=30, nfaults=8, mode=1, checksums=1),
    "offline": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=28, nfaults=8, mode=2, delta=7),
    "partial": dict(name="cfg3", nx=96, ny=80, nz=24, sweeps=18, mode=2, delta=6, recovery=1),
    # two clusters of flagged layers far apart: the union of their cones is
    # re-executed, an undetected flip between them is kept (Q28)
    "partial_union": dict(name="cfg3", nx=96, ny=80, nz=48, sweeps=6, mode=2, delta=3, recovery=1),
    # offline under policy LAZY: b alone predicted, summed, compared (Q29)
    "offline_lazy": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=28, nfaults=8, mode=2, delta=7,
                         checksums=1),
    "partial_lazy": dict(name="cfg3", nx=96, ny=80, nz=24, sweeps=18, mode=2, delta=6, recovery=1,
                         checksums=1),
    "periodic": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=20, nfaults=6, mode=1, bc=1),
    "periodic_offline": dict(name="cfg3", nx=96, ny=80, nz=12, sweeps=20, nfaults=6, mode=2, delta=5,
                             bc=1, recovery=1),
}


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_ipc_processes_equal_oracle(world, case):
    pkw = CASES[case]
    p = make_problem(pkw["name"], **{k: v for k, v in pkw.items() if k != "name"})
    if case == "partial_union":
        faults = [Fault(1, 3, 5, 5, 29), Fault(2, 44, 20, 11, 30), Fault(1, 24, 9, 9, 3),
                  Fault(5, 40, 70, 90, 29), Fault(4, 10, 1, 2, 30)]
    elif case.startswith("partial"):
        faults = [Fault(1, 11, 7, 9, 24), Fault(7, 0, 79, 95, 30), Fault(13, 23, 0, 0, 28),
                  Fault(13, 5, 5, 5, 29)]
    else:
        faults = fault_schedule(p) + [Fault(9, 5, 3, 4, 30), Fault(9, 6, 70, 90, 29),
                                      Fault(11, p.nz - 1, 79, 95, 30)]
        faults = list({(f.sweep, f.z, f.y, f.x): f for f in faults}.values())
    o = oracle_run(p, faults=faults)
    g = _ipc_run(world, pkw, faults)
    assert np.array_equal(g["u"].view(np.uint32), o["u"].view(np.uint32))
    assert_records_equal(g, o)
    assert np.array_equal(g["A"], o["A"]) and np.array_equal(g["B"], o["B"])
    assert g["status"] == o["status"]
    for s in g["stats"]:
        for k in ("sweeps", "rollbacks", "windows", "persistent"):
            assert s[k] == o["stats"][k], (k, s, o["stats"])
    for k in ("detections", "corrected", "located"):
        assert sum(s[k] for s in g["stats"]) == o["stats"][k]


def test_ipc_fp64_box27_offline_partial():
    pkw = dict(name="cfg5", nx=70, ny=33, nz=9, sweeps=15, nfaults=6, recovery=1)
    p = make_problem("cfg5", **{k: v for k, v in pkw.items() if k != "name"})
    faults = fault_schedule(p)
    o = oracle_run(p, faults=faults)
    g = _ipc_run(3, pkw, faults)
    rel = np.abs(g["u"] - o["u"]) / np.abs(o["u"])
    assert rel.max() <= 1e-12
    assert_records_equal(g, o, exact_values=False, rtol=1e-12)
