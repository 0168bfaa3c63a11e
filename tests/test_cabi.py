"""CPU checks of the C-ABI boundary: the shared library loads, exports every
function include/abft_stencil.h declares, its structs match the header's
layout, and configuration validation (no device needed) behaves as the
header documents.  No compute call is made here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from abft_inputs import make_problem
from paper_1909_00709_b200 import abft

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "abft_stencil.h")


@pytest.fixture(scope="module")
def L():
    from paper_1909_00709_b200 import build
    build.build()
    return abft.lib()


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(abft_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_binding_exports():
    assert set(_declared()) == set(abft.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in _declared():
        assert hasattr(L, name), name


def test_struct_sizes_match_header_layout(tmp_path):
    # the ctypes mirrors against the header itself, compiled with gcc
    src = tmp_path / "sz.c"
    names = ["abft_point", "abft_source", "abft_fault", "abft_record", "abft_stats", "abft_config",
             "abft_ipc_slot"]
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "abft_stencil.h"\nint main(void){'
                   + "".join(f'printf("%zu\\n", sizeof({n}));' for n in names)
                   + 'printf("%zu\\n", offsetof(abft_config, recovery));return 0;}\n')
    exe = tmp_path / "sz"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got[:-1] == [C.sizeof(getattr(abft, n)) for n in names]
    assert got[-1] == abft.abft_config.recovery.offset


def test_strerror(L):
    assert abft.abft_strerror(0) == "ok"
    assert "invalid" in abft.abft_strerror(-1)
    assert "persistent" in abft.abft_strerror(3)


def _cfg(**kw):
    p = make_problem("cfg2", nx=64, ny=32, nz=4)
    base = dict(nx=p.nx, ny=p.ny, nz=p.nz, dtype="f32", points=p.points, sources=[],
                epsilon=1e-5)
    base.update(kw)
    return abft.make_config(**base)


def test_workspace_size_sane(L):
    c, keep = _cfg()
    fb, ab = abft.abft_stencil_workspace_size(c)
    assert fb >= 64 * 32 * 6 * 4 and fb % 256 == 0
    assert ab > 3 * 6 * (64 + 32) * 8
    c2, k2 = _cfg(nx=65)   # ragged: the row pitch is padded to 128 bytes
    fb2, _ = abft.abft_stencil_workspace_size(c2)
    assert fb2 >= 96 * 32 * 6 * 4


@pytest.mark.parametrize("kw,code", [
    (dict(nx=0), abft.ABFT_EINVAL),
    (dict(ny=-1), abft.ABFT_EINVAL),
    (dict(epsilon=0.0), abft.ABFT_EINVAL),
    (dict(epsilon=float("nan")), abft.ABFT_EINVAL),
    (dict(points=[]), abft.ABFT_EINVAL),
    (dict(points=[(0, 0, 0, 0.5), (0, 0, 0, 0.5)]), abft.ABFT_EINVAL),
    (dict(points=[(2, 0, 0, 1.0)]), abft.ABFT_EUNSUPPORTED),
    (dict(points=[(0, 0, 0, float("inf"))]), abft.ABFT_EINVAL),
    (dict(mode=2, delta=0), abft.ABFT_EINVAL),
    (dict(mode=7), abft.ABFT_EINVAL),
    (dict(bc=abft.ABFT_BC_CONSTANT, bc_value=float("inf")), abft.ABFT_EINVAL),
    (dict(bc=9), abft.ABFT_EINVAL),
    (dict(checksum_policy=2), abft.ABFT_EINVAL),
    (dict(recovery=2), abft.ABFT_EINVAL),
    (dict(z_begin=1, z_count=2), abft.ABFT_EINVAL),
    (dict(nranks=2, rank=1, z_count=2), abft.ABFT_EINVAL),   # rank 1 cannot own layer 0
    (dict(nranks=2, rank=0, z_count=4), abft.ABFT_EINVAL),   # rank 0 of 2 owns every layer
])
def test_workspace_size_validates(L, kw, code):
    c, keep = _cfg(**kw)
    with pytest.raises(abft.AbftError) as e:
        abft.abft_stencil_workspace_size(c)
    assert e.value.status == code


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_every_boundary_condition_accepted(L, bc):
    c, keep = _cfg(bc=bc, bc_value=2.5)
    fb, ab = abft.abft_stencil_workspace_size(c)
    assert fb > 0 and ab > 0


def test_multi_rank_slab_config_accepted(L):
    c, keep = _cfg(nranks=2, rank=1, z_begin=2, z_count=2, nccl_unique_id=b"\0" * 128)
    fb, ab = abft.abft_stencil_workspace_size(c)
    assert fb >= 64 * 32 * 4 * 4


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("nz,world", [(4, 1), (4, 2), (7, 3), (9, 4), (16, 8)])
def test_library_halo_plan_matches_dist(L, nz, world, periodic):
    """The library's NCCL exchange plan (abft_stencil_halo_plan, used by
    exchange_nccl) equals the host plan dist.halo_plan that the gloo tests run;
    a periodic domain over several ranks closes the ring."""
    from paper_1909_00709_b200 import dist
    for rank in range(world):
        z0, zc = dist.slab(nz, world, rank)
        c, keep = _cfg(nz=nz, nranks=world, rank=rank, z_begin=z0, z_count=zc,
                       nccl_unique_id=b"\0" * 128 if world > 1 else None,
                       bc=abft.ABFT_BC_PERIODIC if periodic else abft.ABFT_BC_CLAMP)
        plan = dist.halo_plan(rank, world, zc, periodic)
        assert abft.abft_stencil_halo_plan(c) == plan
        if periodic and world > 1:
            assert [p for p, _, _ in plan] == [(rank - 1) % world, (rank + 1) % world]


def test_stencil_refuses_cpu_device(L):
    import torch
    c, keep = _cfg()
    with pytest.raises(RuntimeError):
        abft.Stencil(c, keep, torch.zeros(4, 32, 64), device="cpu")
