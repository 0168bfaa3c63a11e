"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the ABFT method (no sweep, checksum,
interpolation, detection or correction).  It only states the problems
(BASELINE.json configs cfg1..cfg5) and draws their random
data and fault schedules from a counter-based splitmix64 generator, so that
the oracle (oracle/) and the GPU path (paper_1909_00709_b200/) consume
bit-identical inputs without sharing any method code.

Generator recipe:
  * stream k of seed s is  r_i = mix64((s ^ k) + (i + 1) * 0x9E3779B97F4A7C15)
    (splitmix64 finaliser), i = linear index in (z, y, x) order;
  * k = 1: initial field u0, k = 2: HotSpot power P, k = 3: cfg5 weights,
    k = 4: fault schedule;
  * fp32 U[0,1) = (r >> 40) * 2^-24, fp64 U[0,1) = (r >> 11) * 2^-53,
    U[lo,hi) = lo + (hi - lo) * U evaluated in fp64, then rounded to dtype.

The Rodinia HotSpot3D inputs the paper used (§V-A) are not in
the container; the HotSpot-like configs below stand in for them with the tile
shapes of Table 1 and BASELINE.json's coefficients.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

__all__ = [
    "Problem", "Fault", "splitmix64", "uniform", "field_u0", "field_power",
    "make_problem", "CONFIGS", "fault_schedule", "flat_index",
]

_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    """Two's-complement view of a uint64 constant as int64."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor holding uint64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(seed: int, stream: int, start: int, count: int,
               device="cpu") -> torch.Tensor:
    """r_i for i in [start, start+count) of stream `stream`; int64 bit patterns."""
    key = _s64((seed ^ stream) & ((1 << 64) - 1))
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    z = i * _s64(_GAMMA) + key
    z = (z ^ _lsr(z, 30)) * _s64(_M1)
    z = (z ^ _lsr(z, 27)) * _s64(_M2)
    return z ^ _lsr(z, 31)


def splitmix64_numpy(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """Same stream with numpy uint64 (well-defined wrap-around); used to pin
    the torch implementation in tests."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = i * np.uint64(_GAMMA) + np.uint64((seed ^ stream) & ((1 << 64) - 1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, stream: int, n: int, dtype: str, lo: float = 0.0,
            hi: float = 1.0, device="cpu", chunk: int = 1 << 26, start: int = 0) -> torch.Tensor:
    """draws [start, start+n) of U[lo,hi) of `dtype` ('f32' | 'f64'), linear-index order."""
    tdt = torch.float32 if dtype == "f32" else torch.float64
    out = torch.empty(n, dtype=tdt, device=device)
    for s in range(0, n, chunk):
        c = min(chunk, n - s)
        r = splitmix64(seed, stream, start + s, c, device)
        if dtype == "f32":
            u = _lsr(r, 40).to(torch.float64) * (2.0 ** -24)
        else:
            u = _lsr(r, 11).to(torch.float64) * (2.0 ** -53)
        if lo != 0.0 or hi != 1.0:
            u = lo + (hi - lo) * u
        out[s:s + c] = u.to(tdt)
        del r, u
    return out


@dataclasses.dataclass
class Fault:
    """One scheduled single-bit flip: at sweep `sweep`
    (1-based), cell (z, y, x) in GLOBAL coordinates, bit `bit`."""
    sweep: int
    z: int
    y: int
    x: int
    bit: int


@dataclasses.dataclass
class Problem:
    """The problem as the paper states it (Eq. 1 + BC + threshold + period):
    stencil set S as ordered (di, dj, dk, w) points,
    constant term C as ordered sources coef * (field | scalar), boundary
    condition, detection threshold eps, offline period delta
    (PAPER.md:696)."""
    name: str
    nx: int
    ny: int
    nz: int
    dtype: str                          # 'f32' | 'f64'
    points: List[Tuple[int, int, int, float]]
    sources: List[Tuple[float, bool, float]]   # (coef, has_field, scalar)
    bc: int = 0                         # 0 clamp, 1 periodic, 2 zero, 3 constant
    bc_value: float = 0.0
    eps: float = 1e-5
    mode: int = 1                       # 0 none, 1 online, 2 offline
    delta: int = 1
    sweeps: int = 1
    correction_form: int = 0            # 0 re-summed Eq. 8, 1 literal Eq. 8
    checksums: int = 0                  # 0 a and b every sweep, 1 b every sweep + a on detection
    recovery: int = 0                   # offline: 0 full rollback, 1 re-execute the flagged layers' light cone
    init: Tuple[float, float] = (0.0, 1.0)
    power: Optional[Tuple[float, float]] = None
    fault_recipe: str = "none"
    nfaults: int = 0
    seed: int = 0

    @property
    def cells(self) -> int:
        return self.nx * self.ny * self.nz

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


def flat_index(p: Problem, z: int, y: int, x: int) -> int:
    return (z * p.ny + y) * p.nx + x


# --- stencils ------------------------------------------------------------
# cfg1: PAPER.md:289-294 (fig.sweep) term order: centre, west, east, south, north
FIVE_POINT_FIG2 = [(0, 0, 0, 0.6), (-1, 0, 0, 0.1), (1, 0, 0, 0.1),
                   (0, 1, 0, 0.1), (0, -1, 0, 0.1)]
# cfg2-4: BASELINE.json configs[1] term order cc*c, cw*w, ce*e, cn*n, cs*s, ct*t, cb*b
HS_CW = HS_CE = HS_CN = HS_CS = 0.1
HS_CT = HS_CB = 0.05
HS_CC = 0.5            # 1 - sum of neighbour weights (BASELINE.json configs[1])
HS_SDC = 0.001
HS_AMB = 80.0
HOTSPOT7 = [(0, 0, 0, HS_CC), (-1, 0, 0, HS_CW), (1, 0, 0, HS_CE),
            (0, -1, 0, HS_CN), (0, 1, 0, HS_CS), (0, 0, 1, HS_CT), (0, 0, -1, HS_CB)]
HOTSPOT_SOURCES = [(HS_SDC, True, 0.0), (HS_CT, False, HS_AMB)]


def box27_weights(seed: int = 0) -> List[Tuple[int, int, int, float]]:
    """cfg5: 27-point box, w = r / sum(r), r U[0,1) fp64 (stream 3), canonical
    order dk outer, dj middle, di inner, each ascending."""
    r = uniform(seed, 3, 27, "f64").tolist()
    s = 0.0
    for v in r:
        s += v
    pts = []
    k = 0
    for dk in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                pts.append((di, dj, dk, r[k] / s))
                k += 1
    return pts


def _cfg(name: str) -> Problem:
    if name == "cfg1":
        return Problem("cfg1", 64, 64, 1, "f32", FIVE_POINT_FIG2, [], eps=1e-5,
                       mode=1, sweeps=20, init=(0.0, 1.0), fault_recipe="cfg1", nfaults=1)
    if name == "cfg2":
        return Problem("cfg2", 512, 512, 8, "f32", HOTSPOT7, HOTSPOT_SOURCES, eps=1e-5,
                       mode=1, sweeps=100, init=(323.0, 343.0), power=(0.0, 1.0),
                       fault_recipe="every10", nfaults=10)
    if name == "cfg3":
        return Problem("cfg3", 512, 512, 64, "f32", HOTSPOT7, HOTSPOT_SOURCES, eps=1e-5,
                       mode=1, delta=10, sweeps=1000, init=(323.0, 343.0), power=(0.0, 1.0),
                       fault_recipe="uniform_noreplace", nfaults=20)
    if name == "cfg4":
        return Problem("cfg4", 1024, 1024, 1024, "f32", HOTSPOT7, HOTSPOT_SOURCES, eps=1e-5,
                       mode=1, sweeps=200, init=(323.0, 343.0), power=(0.0, 1.0),
                       fault_recipe="per_slab_block", nfaults=32)
    if name == "cfg5":
        return Problem("cfg5", 2048, 2048, 1024, "f64", box27_weights(0), [], eps=1e-10,
                       mode=2, delta=5, sweeps=100, init=(0.0, 1.0),
                       fault_recipe="uniform_replace", nfaults=50)
    raise KeyError(name)


CONFIGS = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


def make_problem(name: str, **overrides) -> Problem:
    """A BASELINE.json config (cfg1..cfg5) with optional overrides (reduced
    sizes for parity tests keep the config's stencil, sources, eps, mode)."""
    return _cfg(name).replace(**overrides)


def field_u0(p: Problem, device="cpu", z0: int = 0, zc: Optional[int] = None) -> torch.Tensor:
    """Initial field, layers [z0, z0 + zc) of the global domain (a z-slab)."""
    zc = p.nz - z0 if zc is None else zc
    lo, hi = p.init
    n = zc * p.ny * p.nx
    return uniform(p.seed, 1, n, p.dtype, lo, hi, device,
                   start=z0 * p.ny * p.nx).view(zc, p.ny, p.nx)


def field_power(p: Problem, device="cpu", z0: int = 0,
                zc: Optional[int] = None) -> Optional[torch.Tensor]:
    """HotSpot power field (source of C), layers [z0, z0 + zc)."""
    if p.power is None:
        return None
    zc = p.nz - z0 if zc is None else zc
    lo, hi = p.power
    n = zc * p.ny * p.nx
    return uniform(p.seed, 2, n, p.dtype, lo, hi, device,
                   start=z0 * p.ny * p.nx).view(zc, p.ny, p.nx)


class _Draw:
    """Sequential draws from stream 4 (fault schedule)."""

    def __init__(self, seed: int):
        self.seed = seed
        self.i = 0

    def u64(self) -> int:
        v = int(splitmix64(self.seed, 4, self.i, 1)[0].item()) & ((1 << 64) - 1)
        self.i += 1
        return v

    def below(self, n: int) -> int:
        return self.u64() % n


def fault_schedule(p: Problem, sweeps: Optional[int] = None, slab_planes: int = 128,
                   block: int = 50) -> List[Fault]:
    """Seeded fault schedule of the config.
    At most one flip per (sweep, plane); collisions are re-drawn."""
    n_sweeps = p.sweeps if sweeps is None else sweeps
    d = _Draw(p.seed)
    bits = 64 if p.dtype == "f64" else 32
    out: List[Fault] = []
    used = set()

    def cell(z_lo: int, z_hi: int):
        z = z_lo + d.below(z_hi - z_lo)
        y = d.below(p.ny)
        x = d.below(p.nx)
        return z, y, x

    def add(s, z, y, x, b):
        used.add((s, z))
        out.append(Fault(s, z, y, x, b))

    r = p.fault_recipe
    if r == "none" or p.nfaults == 0 or n_sweeps == 0:
        return []
    if r == "cfg1":                      # 1 flip at sweep 10, bit 0..30
        s = min(10, n_sweeps)
        z, y, x = cell(0, p.nz)
        add(s, z, y, x, d.below(31))
    elif r == "every10":                 # at sweeps 10, 20, ..., bits 0..31
        for k in range(p.nfaults):
            s = 10 * (k + 1)
            if s > n_sweeps:
                break
            z, y, x = cell(0, p.nz)
            add(s, z, y, x, d.below(bits))
    elif r == "uniform_noreplace":       # sweeps without replacement in 1..n
        chosen = set()
        while len(chosen) < min(p.nfaults, n_sweeps):
            chosen.add(1 + d.below(n_sweeps))
        for s in sorted(chosen):
            z, y, x = cell(0, p.nz)
            add(s, z, y, x, d.below(bits))
    elif r == "per_slab_block":          # 1 per `slab_planes`-plane slab per `block` sweeps
        nslab = max(1, math.ceil(p.nz / slab_planes))
        nblk = max(1, math.ceil(n_sweeps / block))
        for b in range(nblk):
            for k in range(nslab):
                lo_s = b * block + 1
                hi_s = min((b + 1) * block, n_sweeps)
                s = lo_s + d.below(hi_s - lo_s + 1)
                z, y, x = cell(k * slab_planes, min(p.nz, (k + 1) * slab_planes))
                add(s, z, y, x, d.below(bits))
    elif r == "uniform_replace":         # sweeps uniform with replacement; (s, z) unique
        while len(out) < p.nfaults:
            s = 1 + d.below(n_sweeps)
            z, y, x = cell(0, p.nz)
            b = d.below(bits)
            if (s, z) in used:
                continue
            add(s, z, y, x, b)
    else:
        raise KeyError(r)
    out.sort(key=lambda f: (f.sweep, f.z, f.y, f.x))
    return out
