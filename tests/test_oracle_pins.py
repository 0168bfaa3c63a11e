"""Pins of the CPU oracle against what the paper and mathematics fix
(not against the oracle itself).  CPU only.

Each test names the PAPER.md passage (P:<line>) or closed form it checks.
A plausible slip anywhere in oracle/abft_oracle.c (dropped alpha/beta term,
wrong sign, transposed axis, wrong neighbour direction, wrong BC, wrong
injection point, wrong correction algebra, rollback not restoring) fails at
least one test here.
"""
import math
import os
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

from abft_inputs import (Fault, Problem, fault_schedule, field_power, field_u0,
                         make_problem, splitmix64, splitmix64_numpy, uniform)
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold_lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.split("#")[0].strip() for l in f if l.split("#")[0].strip()]


# ----------------------------------------------------------- generators

def test_splitmix64_known_values():
    want = [int(v, 16) for v in _gold_lines("splitmix64_seed0.txt")]
    got = splitmix64(0, 0, 0, len(want)).numpy().view(np.uint64).tolist()
    assert got == want


def test_splitmix64_torch_equals_numpy_wraparound():
    a = splitmix64(12345, 4, 1000, 4096).numpy().view(np.uint64)
    b = splitmix64_numpy(12345, 4, 1000, 4096)
    assert (a == b).all()


def test_uniform_f32_grid_and_range():
    u = uniform(0, 1, 100000, "f32", 323.0, 343.0).numpy()
    assert u.dtype == np.float32 and u.min() >= 323.0 and u.max() < 343.0
    v = uniform(0, 1, 1000, "f32").numpy().astype(np.float64)
    assert np.all(v * 2 ** 24 == np.floor(v * 2 ** 24))     # multiples of 2^-24


def test_fault_schedules_follow_recipes():
    f1 = fault_schedule(make_problem("cfg1"))
    assert len(f1) == 1 and f1[0].sweep == 10 and 0 <= f1[0].bit <= 30
    f2 = fault_schedule(make_problem("cfg2"))
    assert [f.sweep for f in f2] == list(range(10, 101, 10))
    f3 = fault_schedule(make_problem("cfg3"))
    assert len(f3) == 20 and len({f.sweep for f in f3}) == 20
    f4 = fault_schedule(make_problem("cfg4"))
    assert len(f4) == 32
    for f in f4:   # one per 128-plane slab per 50-sweep block
        assert sum(1 for g in f4 if g.z // 128 == f.z // 128 and
                   (g.sweep - 1) // 50 == (f.sweep - 1) // 50) == 1
    f5 = fault_schedule(make_problem("cfg5"))
    assert len(f5) == 50 and len({(f.sweep, f.z) for f in f5}) == 50
    assert max(f.bit for f in f5) <= 63


# ------------------------------------------------------------ fault hook

def test_flip_ieee_layout():
    for line in _gold_lines("ieee_flip.txt"):
        dt, val, bit, want = line.split()
        if dt == "f32":
            a = np.array([float(val)], np.float32)
            O.flip(a, 0, int(bit))
            assert a.view(np.uint32)[0] == int(want, 16)
        else:
            a = np.array([float(val)], np.float64)
            O.flip(a, 0, int(bit))
            assert a.view(np.uint64)[0] == int(want, 16)


def test_flip_is_an_involution():
    rng = np.random.default_rng(0)
    a = rng.random(64).astype(np.float32)
    b = a.copy()
    for k in range(64):
        O.flip(b, k, k % 32)
        assert b[k] != a[k] or np.isnan(b[k])
        O.flip(b, k, k % 32)
    assert (a.view(np.uint32) == b.view(np.uint32)).all()


# -------------------------------------------------------- checksums Eqs. 2-3

def test_checksums_worked_example():
    g = {l.split(":")[0]: l.split(":")[1] for l in _gold_lines("checksum_2x2.txt")}
    rows = [[float(v) for v in r.split()] for r in g["grid_rows_y"].split("|")]
    p = Problem("t", 2, 2, 1, "f32", [(0, 0, 0, 1.0)], [])
    A, B = O.checksums(O.OProblem(p), np.array(rows, np.float32))
    assert A[0].tolist() == [float(v) for v in g["a"].split()]
    assert B[0].tolist() == [float(v) for v in g["b"].split()]


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_checksums_brute_force(dtype):
    p = Problem("t", 13, 7, 3, dtype, [(0, 0, 0, 1.0)], [])
    rng = np.random.default_rng(1)
    u = rng.random((3, 7, 13)).astype(np.float32 if dtype == "f32" else np.float64)
    A, B = O.checksums(O.OProblem(p), u)
    for z in range(3):
        for x in range(13):
            want = math.fsum(float(u[z, y, x]) for y in range(7))
            assert abs(A[z, x] - want) <= 1e-15 * abs(want)
            if dtype == "f32":
                assert A[z, x] == want          # exact: fp64 sum of few fp32 values
        for y in range(7):
            want = math.fsum(float(u[z, y, x]) for x in range(13))
            assert abs(B[z, y] - want) <= 1e-15 * abs(want)
        assert abs(math.fsum(A[z]) - math.fsum(B[z])) < 1e-12   # both = plane total


# ---------------------------------------------------------------- sweep Eq. 1

def _exact_sweep(u, pts, bc, nz, ny, nx, g=0):
    """Brute-force Eq. 1 in exact rational arithmetic (tiny grids)."""
    def r(c, n):
        if 0 <= c < n:
            return c
        if bc == 0:
            return 0 if c < 0 else n - 1
        if bc == 1:
            return c % n
        return None
    out = np.empty((nz, ny, nx), dtype=object)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                s = Fraction(0)
                for (di, dj, dk, w) in pts:
                    zz, yy, xx = r(z + dk, nz), r(y + dj, ny), r(x + di, nx)
                    v = Fraction(g) if None in (zz, yy, xx) else Fraction(float(u[zz, yy, xx]))
                    s += Fraction(w) * v
                out[z, y, x] = s
    return out


def test_sweep_identity_is_copy():
    p = Problem("t", 9, 5, 2, "f32", [(0, 0, 0, 1.0)], [])
    u = np.random.default_rng(2).random((2, 5, 9)).astype(np.float32)
    out = O.sweep(O.OProblem(p), u)
    assert (out.view(np.uint32) == u.view(np.uint32)).all()


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
def test_sweep_dyadic_exact_brute_force(bc):
    # dyadic weights, integer data < 2^10: every fp32 operation is exact, so the
    # oracle must equal exact rational Eq. 1 incl. the BC of P:289-292.
    pts = [(0, 0, 0, 0.25), (-1, 0, 0, 0.125), (1, 0, 0, 0.0625), (0, 1, 0, 0.125),
           (0, -1, 0, 0.1875), (0, 0, 1, 0.125), (0, 0, -1, 0.125)]
    g = 7.0 if bc == 3 else 0.0
    p = Problem("t", 6, 5, 4, "f32", pts, [], bc=bc, bc_value=g)
    u = np.random.default_rng(3).integers(0, 1024, (4, 5, 6)).astype(np.float32)
    out = O.sweep(O.OProblem(p), u)
    want = _exact_sweep(u, pts, bc, 4, 5, 6, g)
    assert all(Fraction(float(out[i])) == want[i] for i in np.ndindex(out.shape))


def test_sweep_four_point_paper_example_checkerboard():
    # S = {(0,-1,.25), (-1,0,.25), (1,0,.25), (0,1,.25)}: with periodic BC
    # every neighbour of a +1 cell of a checkerboard is -1, so the sweep negates it.
    line = [l for l in _gold_lines("paper_parameters.txt") if l.startswith("four_point")][0]
    pts = []
    for t in line.split(":", 1)[1].split():
        i, j, w = t.strip("()").split(",")
        pts.append((int(i), int(j), 0, float(w)))
    p = Problem("t", 8, 6, 1, "f32", pts, [], bc=1)
    x, y = np.meshgrid(np.arange(8), np.arange(6))
    u = np.where((x + y) % 2 == 0, 1.0, -1.0).astype(np.float32)[None]
    out = O.sweep(O.OProblem(p), u)
    assert (out == -u).all()


def test_sweep_uniform_fixed_point_and_vertical_direction():
    # weights summing to 1, C = 0: a uniform field is a fixed point
    pts = [(0, 0, 0, 0.5), (-1, 0, 0, 0.125), (1, 0, 0, 0.125), (0, -1, 0, 0.125),
           (0, 1, 0, 0.125)]
    p = Problem("t", 5, 4, 2, "f32", pts, [])
    u = np.full((2, 4, 5), 3.25, np.float32)
    assert (O.sweep(O.OProblem(p), u) == u).all()
    # t = z+1 and b = z-1 (HotSpot, Q22): u = f(z) layered; only (0,0,+1) weighted
    p = Problem("t", 3, 3, 4, "f32", [(0, 0, 1, 1.0)], [])
    u = np.arange(4, dtype=np.float32)[:, None, None] * np.ones((4, 3, 3), np.float32)
    out = O.sweep(O.OProblem(p), u)
    assert out[:, 0, 0].tolist() == [1.0, 2.0, 3.0, 3.0]    # clamped at the top


def test_sweep_sources_hotspot_closed_form():
    # uniform T, weights summing to 1: out = T + sdc*P + ct*amb exactly in the
    # FMA chain when T*w terms are exact (T = 256, dyadic weights 0.5/0.125/...)
    pts = [(0, 0, 0, 0.5), (-1, 0, 0, 0.125), (1, 0, 0, 0.125), (0, -1, 0, 0.0625),
           (0, 1, 0, 0.0625), (0, 0, 1, 0.0625), (0, 0, -1, 0.0625)]
    srcs = [(0.5, True, 0.0), (0.25, False, 8.0)]
    p = Problem("t", 4, 4, 3, "f32", pts, srcs)
    P = np.full((3, 4, 4), 2.0, np.float32)
    u = np.full((3, 4, 4), 256.0, np.float32)
    out = O.sweep(O.OProblem(p, [P]), u)
    assert (out == 256.0 + 0.5 * 2.0 + 0.25 * 8.0).all()


def test_constant_sums_fp32_use_dtype_rounded_operands():
    # c_x, c_y of Theorem 1 ("pre-computed" P:392) for an fp32 problem:
    # the constant C_{x,y} of Eq. 1 as the sweep applies it, i.e. with the
    # coefficients and the scalar rounded to the field dtype (Q23).  Exact
    # rational brute force: every product of two fp32 values is exact in
    # fp64, so the oracle's fp64 sums may differ from the exact sum only by
    # their own rounding (<= ny ulps); an oracle that used the unrounded
    # fp64 coefficients (0.001, 0.05) would be off by ~1e-8 relative.
    nz, ny, nx = 3, 6, 8
    p = Problem("t", nx, ny, nz, "f32", [(0, 0, 0, 1.0)],
                [(0.001, True, 0.0), (0.05, False, 80.0)])
    P = np.random.default_rng(5).random((nz, ny, nx)).astype(np.float32)
    cA, cB = O.constant_sums(O.OProblem(p, [P]))
    f = lambda v: Fraction(float(np.float32(v)))
    C = [[[f(0.001) * Fraction(float(P[z, y, x])) + f(0.05) * f(80.0) for x in range(nx)]
          for y in range(ny)] for z in range(nz)]
    for z in range(nz):
        for x in range(nx):
            ex = sum(C[z][y][x] for y in range(ny))
            assert abs(Fraction(cA[z, x]) - ex) <= ex * Fraction(1, 2 ** 49)
        for y in range(ny):
            ex = sum(C[z][y][x] for x in range(nx))
            assert abs(Fraction(cB[z, y]) - ex) <= ex * Fraction(1, 2 ** 49)
    # the unrounded coefficients are measurably different (the pin can fail)
    raw = sum(Fraction(0.001) * Fraction(float(P[0, y, 0])) + Fraction(0.05) * Fraction(80.0)
              for y in range(ny))
    assert abs(Fraction(cA[0, 0]) - raw) > raw * Fraction(1, 10 ** 9)


# ------------------------------------------------------ Theorem 1 (prediction)

def _fsum_checksums(u):
    nz, ny, nx = u.shape
    A = np.array([[math.fsum(float(v) for v in u[z, :, x]) for x in range(nx)] for z in range(nz)])
    B = np.array([[math.fsum(float(v) for v in u[z, y, :]) for y in range(ny)] for z in range(nz)])
    return A, B


def _random_stencil(rng, k, symmetric=False):
    offs = [(di, dj, dk) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    rng.shuffle(offs)
    sel = offs[:k]
    return [(di, dj, dk, float(rng.uniform(0.01, 0.3))) for (di, dj, dk) in sel]


@pytest.mark.parametrize("bc", [0, 1, 2, 3])
@pytest.mark.parametrize("seed", range(4))
def test_theorem1_prediction_equals_brute_force_checksums(bc, seed):
    # Theorem 1: interpolated a', b' == checksums of the swept grid,
    # for arbitrary (asymmetric) radius-1 stencils, every BC, 3D (Q6), fp64.
    rng = random.Random(seed)
    pts = _random_stencil(rng, rng.randint(3, 27))
    p = Problem("t", 7, 6, 5, "f64", pts, [(0.3, True, 0.0), (0.2, False, 1.5)],
                bc=bc, bc_value=0.75)
    nrng = np.random.default_rng(seed)
    u = nrng.random((5, 6, 7))
    P = nrng.random((5, 6, 7))
    op = O.OProblem(p, [P])
    A, B = O.checksums(op, u)
    PA, PB = O.predict(op, A, B, u)
    u1 = O.sweep(op, u)
    A1, B1 = _fsum_checksums(u1)
    assert np.max(np.abs(PA - A1) / np.abs(A1)) < 1e-12
    assert np.max(np.abs(PB - B1) / np.abs(B1)) < 1e-12


def test_theorem1_negative_control_dropped_boundary_terms():
    # Dropping alpha/beta (u := 0 in the ledger) must break Theorem 1 for an
    # asymmetric clamp stencil -- shows the pin above is sensitive --
    # while for a mirror-symmetric clamp stencil or periodic BC the simplified
    # Eqs. 6-7 (alpha = beta = 0) hold.
    nrng = np.random.default_rng(7)
    u = nrng.random((3, 8, 9))
    zeros = np.zeros_like(u)
    asym = [(0, 0, 0, 0.4), (-1, 0, 0, 0.3), (1, 0, 0, 0.1), (0, 1, 0, 0.15), (0, -1, 0, 0.05)]
    sym = [(0, 0, 0, 0.6), (-1, 0, 0, 0.1), (1, 0, 0, 0.1), (0, 1, 0, 0.1), (0, -1, 0, 0.1)]
    for pts, bc, must_hold in [(asym, 0, False), (sym, 0, True), (asym, 1, True)]:
        op = O.OProblem(Problem("t", 9, 8, 3, "f64", pts, [], bc=bc))
        A, B = O.checksums(op, u)
        PA, PB = O.predict(op, A, B, zeros)
        A1, B1 = _fsum_checksums(O.sweep(op, u))
        gap = max(np.max(np.abs(PA - A1) / A1), np.max(np.abs(PB - B1) / B1))
        assert (gap < 1e-12) == must_hold, (pts, bc, gap)


def test_theorem1_dyadic_exact_equality():
    # dyadic workload: every operation exact => predicted == actual exactly
    pts = [(0, 0, 0, 0.5), (-1, 0, 0, 0.125), (1, 0, 0, 0.0625), (0, -1, 0, 0.125),
           (0, 1, 0, 0.0625), (0, 0, 1, 0.0625), (0, 0, -1, 0.0625)]
    p = Problem("t", 16, 16, 4, "f32", pts, [])
    op = O.OProblem(p)
    u = np.random.default_rng(5).integers(0, 1024, (4, 16, 16)).astype(np.float32)
    A, B = O.checksums(op, u)
    PA, PB = O.predict(op, A, B, u)
    A1, B1 = O.checksums(op, O.sweep(op, u))
    assert (PA == A1).all() and (PB == B1).all()


# ------------------------------------------------------ detection (Thm 2)

def test_flag_rule_closed_cases():
    # fig.detect: flagged iff |pred/act - 1| > eps (fp64, Q7, Q24)
    assert O.flag(1.0 + 2e-5, 1.0, 1e-5) == 1
    assert O.flag(1.0 + 5e-6, 1.0, 1e-5) == 0
    assert O.flag(1.0 - 2e-5, 1.0, 1e-5) == 1
    assert O.flag(0.0, 0.0, 1e-5) == 0
    assert O.flag(1e-300, 0.0, 1e-5) == 1
    assert O.flag(float("nan"), 1.0, 1e-5) == 1
    assert O.flag(1.0, float("nan"), 1e-5) == 1
    assert O.flag(1.0, float("inf"), 1e-5) == 1
    assert O.flag(-3.0, 3.0, 1e-5) == 1


def _cfg1_like(**kw):
    return make_problem("cfg1", **kw)


@pytest.mark.parametrize("name,kw", [
    ("cfg1", {}),
    ("cfg2", dict(nx=64, ny=48, nz=6, sweeps=40)),
    ("cfg3", dict(nx=40, ny=33, nz=5, sweeps=30, mode=2, delta=10)),
    ("cfg5", dict(nx=24, ny=20, nz=6, sweeps=20, mode=1)),
    ("cfg5", dict(nx=24, ny=20, nz=6, sweeps=20)),
])
def test_no_false_positives_error_free(name, kw):
    # Theorem 2 and "no false-positives" at eps
    p = make_problem(name, **kw)
    op = O.OProblem(p, [field_power(p).numpy()] if p.power else [])
    r = O.run(op, field_u0(p).numpy(), p.sweeps)
    assert r["stats"]["detections"] == 0 and r["status"] == 0 and r["records"] == []


def _clean_states(p, op, u0, s):
    q = p.replace(mode=0)
    oq = O.OProblem(q, op._fields)
    return O.run(oq, u0, s)["u"]


@pytest.mark.parametrize("checksums", [0, 1])
def test_detection_closed_form_and_location_cfg1(checksums):
    # For one flip at sweep s: delta = flipped - clean is exact; since the
    # prediction equals the clean checksum up to ~1e-8, the B (row) entry is
    # flagged iff |delta| > eps*|S + delta| (S clean row sum), same for A.
    # Every flip flagged in both vectors must be located at the injected cell
    # and corrected (Eq. 8).  checksums=1 (detect on b,
    # compute and compare a only then): a record iff b is flagged.
    p = _cfg1_like().replace(checksums=checksums)
    op = O.OProblem(p)
    u0 = field_u0(p).numpy()
    s = 10
    clean = _clean_states(p, op, u0, s)
    rng = random.Random(11)
    checked = 0
    for trial in range(120):
        y, x, bit = rng.randrange(64), rng.randrange(64), rng.randrange(31)
        cv = np.array([clean[0, y, x]], np.float32)
        fv = cv.copy()
        O.flip(fv, 0, bit)
        d = float(fv[0]) - float(cv[0])
        Srow = math.fsum(float(v) for v in clean[0, y, :])
        Scol = math.fsum(float(v) for v in clean[0, :, x])
        mb = abs(d) / abs(Srow + d) if math.isfinite(d) else math.inf
        ma = abs(d) / abs(Scol + d) if math.isfinite(d) else math.inf
        if 0.9 * p.eps < mb < 1.1 * p.eps or 0.9 * p.eps < ma < 1.1 * p.eps:
            continue                               # ambiguous band
        r = O.run(op, u0, s, [Fault(s, 0, y, x, bit)])
        expect_b, expect_a = mb > p.eps, ma > p.eps
        if checksums == 1 and not expect_b:
            assert r["records"] == []
        elif not (expect_a or expect_b):
            assert r["records"] == []
        else:
            rec = r["records"][0]
            assert rec["sweep"] == s and rec["z"] == 0
            assert (rec["nflag_b"] == 1) == expect_b and (rec["nflag_a"] == 1) == expect_a
            if expect_a and expect_b:
                assert (rec["y"], rec["x"]) == (y, x) and rec["status"] == O.REC_CORRECTED
                assert abs(rec["corrected"] - float(cv[0])) <= 1e-5 * abs(float(cv[0]))
                # fig.correction: corrected = (vx + vy) / 2, in the dtype
                assert rec["corrected"] == float(np.float32((rec["vx"] + rec["vy"]) / 2.0))
                assert rec["vx"] != rec["vy"] or rec["corrected"] == np.float32(rec["vx"])
        checked += 1
    assert checked > 80


def test_lazy_checksum_policy_equals_both_when_b_flags():
    # P:271-273 / P:496-497: computing a only for layers whose b flags changes
    # nothing when every flip is large enough to flag b (bits >= 24 of values
    # in [323, 343) in 64-wide rows): same field bitwise, same records.
    p = make_problem("cfg2", nx=64, ny=48, nz=5, sweeps=30)
    u0 = field_u0(p).numpy()
    P = field_power(p).numpy()
    rng = random.Random(5)
    faults = [Fault(s, rng.randrange(5), rng.randrange(48), rng.randrange(64), rng.randint(24, 30))
              for s in range(3, 30, 4)]
    r0 = O.run(O.OProblem(p, [P]), u0, p.sweeps, faults)
    r1 = O.run(O.OProblem(p.replace(checksums=1), [P]), u0, p.sweeps, faults)
    assert r0["stats"]["corrected"] == len(faults)
    assert (r0["u"].view(np.uint32) == r1["u"].view(np.uint32)).all()
    assert r0["records"] == r1["records"]
    assert np.array_equal(r0["B"], r1["B"]) and np.array_equal(r0["A"], r1["A"])


def test_paper_bits_0_12_undetected_high_bits_detected():
    # flips in bits 0..12 are never detected (64x64, eps = 1e-5);
    # bits 13..31 are mostly detected and corrected.
    par = {l.split(":")[0]: l.split(":")[1].strip() for l in _gold_lines("paper_parameters.txt")}
    lo, hi = (int(v) for v in par["undetected_bits_fp32"].split("-"))
    p = _cfg1_like(sweeps=6)
    op = O.OProblem(p)
    u0 = field_u0(p).numpy()
    rng = random.Random(3)
    for bit in list(range(lo, hi + 1)) + list(range(20, 32)):
        det = 0
        for t in range(12):
            f = Fault(rng.randint(1, 6), 0, rng.randrange(64), rng.randrange(64), bit)
            r = O.run(op, u0, 6, [f])
            det += r["stats"]["detections"]
        if bit <= hi:
            assert det == 0, bit
        else:
            assert det == 12, bit


# ------------------------------------------------------------- correction

def test_correction_dyadic_is_bitwise_exact():
    # dyadic workload: predicted == actual exactly (sweeps 1-4), so the
    # re-summed Eq. 8 restores the clean value bitwise and the whole run equals
    # the fault-free run bitwise.
    pts = [(0, 0, 0, 0.5), (-1, 0, 0, 0.125), (1, 0, 0, 0.125), (0, -1, 0, 0.125),
           (0, 1, 0, 0.125)]
    p = Problem("t", 32, 32, 2, "f32", pts, [], eps=1e-5, mode=1, sweeps=4)
    op = O.OProblem(p)
    u0 = np.random.default_rng(9).integers(0, 1024, (2, 32, 32)).astype(np.float32)
    ref = O.run(op, u0, 4)
    rng = random.Random(4)
    for t in range(40):
        f = Fault(rng.randint(1, 4), rng.randrange(2), rng.randrange(32), rng.randrange(32),
                  rng.randint(13, 30))
        r = O.run(op, u0, 4, [f])
        if r["stats"]["corrected"] == 1:
            assert (r["u"].view(np.uint32) == ref["u"].view(np.uint32)).all()
            assert r["stats"]["detections"] == 1     # repaired checksums: no later flags


@pytest.mark.parametrize("name,kw", [
    ("cfg1", dict(sweeps=12)),
    ("cfg2", dict(nx=40, ny=33, nz=5, sweeps=12)),
    ("cfg2", dict(nx=40, ny=33, nz=5, sweeps=12, bc=1)),
    ("cfg2", dict(nx=40, ny=33, nz=5, sweeps=12, bc=3, bc_value=330.0)),
    ("cfg5", dict(nx=20, ny=17, nz=5, sweeps=10, mode=1)),
])
def test_correction_by_recompute_restores_the_fault_free_run(name, kw):
    # correction_form 2 (stencil locality): u^(t) is
    # intact, so recomputing the located cell with Eq. 1 restores it exactly:
    # every run whose flips are all located equals the fault-free run bitwise
    # (field and checksums), whatever bit was flipped -- including the exponent
    # flips that defeat the checksum estimate of Eq. 8.
    p = make_problem(name, **kw).replace(correction_form=2)
    fields = [field_power(p).numpy()] if p.power else []
    op = O.OProblem(p, fields)
    u0 = field_u0(p).numpy()
    ref = O.run(op, u0, p.sweeps)
    rng = random.Random(8)
    hi = 31 if p.dtype == "f32" else 63
    done = 0
    for t in range(30):
        f = Fault(rng.randint(1, p.sweeps), rng.randrange(p.nz), rng.randrange(p.ny), rng.randrange(p.nx),
                  rng.randint(hi - 12, hi))
        r = O.run(op, u0, p.sweeps, [f])
        if r["stats"]["corrected"] == 1 and r["stats"]["detections"] == 1:
            w = np.uint32 if p.dtype == "f32" else np.uint64
            assert (r["u"].view(w) == ref["u"].view(w)).all()
            assert np.array_equal(r["A"], ref["A"]) or p.dtype == "f64"
            done += 1
    assert done >= 15


@pytest.mark.parametrize("cells", [
    ((7, 9), (20, 31)),            # two rows, two columns: 2x2 flagged, no single intersection
    ((7, 9), (7, 31)),             # one row, two columns
    ((7, 9), (20, 9), (33, 2)),    # one column twice + a third cell
])
@pytest.mark.parametrize("checksums", [0, 1])
def test_recompute_repairs_several_flips_in_one_layer(cells, checksums):
    # correction_form 2 when the flags do not intersect in one cell (Q27):
    # recomputing layer z from the intact u^(t) (locality)
    # finds exactly the flipped cells, restores the fault-free field bitwise,
    # and the re-summed a, b are the exact column / row sums (Eqs. 2-3; fp32
    # HotSpot data sum exactly in fp64).  Forms 0 / 1 leave such a layer
    # "uncorrectable" / "unlocated" (Q13, Q14).
    p = make_problem("cfg2", nx=40, ny=36, nz=4, sweeps=6, checksums=checksums)
    op = O.OProblem(p, [field_power(p).numpy()])
    u0 = field_u0(p).numpy()
    ref = O.run(op, u0, p.sweeps)
    faults = [Fault(4, 2, y, x, 29) for y, x in cells]
    r0 = O.run(op, u0, p.sweeps, faults)
    assert r0["stats"]["corrected"] == 0 and r0["stats"]["uncorrectable"] + r0["stats"]["unlocated"] == 1
    p2 = p.replace(correction_form=2)
    r = O.run(O.OProblem(p2, [field_power(p2).numpy()]), u0, p.sweeps, faults)
    assert (r["u"].view(np.uint32) == ref["u"].view(np.uint32)).all()
    rec = [(x["sweep"], x["z"], x["y"], x["x"]) for x in r["records"]]
    assert sorted(rec) == sorted((4, 2, y, x) for y, x in cells)
    assert all(x["status"] == O.REC_RECOMPUTED for x in r["records"])
    assert r["stats"]["detections"] == 1 and r["stats"]["corrected"] == len(cells)
    u = r["u"].astype(np.float64)
    assert np.array_equal(r["A"], u.sum(axis=1)) and np.array_equal(r["B"], u.sum(axis=2))


def test_recompute_false_alarm_leaves_the_field():
    # a threshold far below the prediction's rounding error flags error-free
    # layers; form 2 recomputes them, finds no differing cell ("verified") and
    # the field is the fault-free run's, bitwise.
    p = make_problem("cfg5", nx=20, ny=17, nz=4, sweeps=5, mode=1, nfaults=0)
    op = O.OProblem(p)
    u0 = field_u0(p).numpy()
    ref = O.run(op, u0, p.sweeps, [])
    tight = p.replace(correction_form=2, eps=1e-19)
    r = O.run(O.OProblem(tight), u0, p.sweeps, [])
    assert r["stats"]["detections"] > 0 and r["stats"]["corrected"] == 0
    assert r["records"] and all(x["status"] == O.REC_VERIFIED for x in r["records"])
    assert (r["u"].view(np.uint64) == ref["u"].view(np.uint64)).all()


def test_correction_literal_form_fails_on_exponent_flip():
    # "if the bit-flips occur in the last bits of the exponent, the error
    # causes an overflow in the checksums" -- the literal fig.correction form
    # a' - (a - u) loses the value when u ~ 1e38; the re-summed form (Q11) not.
    p = _cfg1_like(sweeps=10)
    u0 = field_u0(p).numpy()
    clean = _clean_states(p, O.OProblem(p), u0, 10)[0, 20, 30]
    f = [Fault(10, 0, 20, 30, 30)]
    lit = O.run(O.OProblem(p.replace(correction_form=1)), u0, 10, f)["records"][0]
    res = O.run(O.OProblem(p), u0, 10, f)["records"][0]
    assert abs(res["corrected"] - clean) / clean < 1e-5
    assert not abs(lit["corrected"] - clean) / clean < 1e-2


# ---------------------------------------------------------------- offline

def test_offline_rollback_erases_error_bitwise():
    # P:913 / P:867: checkpoint + recompute "completely" erases detected errors.
    p = make_problem("cfg3", nx=48, ny=40, nz=6, sweeps=30, mode=2, delta=10, nfaults=3)
    P = field_power(p).numpy()
    op = O.OProblem(p, [P])
    u0 = field_u0(p).numpy()
    ref = O.run(op, u0, 30)
    faults = [Fault(4, 2, 7, 9, 27), Fault(15, 5, 39, 0, 30), Fault(30, 0, 0, 47, 31)]
    r = O.run(op, u0, 30, faults)
    assert r["stats"]["rollbacks"] == 3 and r["status"] == 0
    assert (r["u"].view(np.uint32) == ref["u"].view(np.uint32)).all()
    assert {(x["sweep"], x["z"]) for x in r["records"]} >= {(10, 2), (20, 5), (30, 0)}


def test_offline_persistent_error():
    # a fault that strikes again during the recomputation (second armed copy)
    p = make_problem("cfg3", nx=32, ny=32, nz=4, sweeps=10, mode=2, delta=5)
    op = O.OProblem(p, [field_power(p).numpy()])
    f = [Fault(3, 1, 5, 5, 30), Fault(3, 1, 5, 5, 30)]
    r = O.run(op, field_u0(p).numpy(), 10, f)
    assert r["status"] == 3 and r["stats"]["persistent"] == 1
    assert any(x["status"] == O.REC_PERSISTENT for x in r["records"])


def test_offline_interpolation_matches_direct_after_delta_sweeps():
    # algo.offline.inteprolation: applying Theorem 1 delta times to
    # the checkpoint checksums reproduces the direct checksums (fp64, 27-pt).
    p = make_problem("cfg5", nx=12, ny=10, nz=5, sweeps=8)
    op = O.OProblem(p)
    u = field_u0(p).numpy()
    A, B = O.checksums(op, u)
    for t in range(8):
        A, B = O.predict(op, A, B, u)
        u = O.sweep(op, u)
    A1, B1 = _fsum_checksums(u)
    assert np.max(np.abs(A - A1) / A1) < 1e-12 and np.max(np.abs(B - B1) / B1) < 1e-12


# ------------------------------------- offline partial re-execution (Q28)

def _offline(p, faults, recovery):
    q = p.replace(recovery=recovery)
    op = O.OProblem(q, [field_power(q).numpy()] if q.power else [])
    return O.run(op, field_u0(q).numpy(), q.sweeps, faults)


@pytest.mark.parametrize("delta", [1, 3, 6])
def test_partial_reexecution_of_detected_errors_restores_the_fault_free_run(delta):
    # stencil locality: re-executing only the light
    # cone of the flagged layers erases every detected error, so the result
    # is the fault-free run bitwise -- like the full rollback.  Flips
    # at a window's first sweep spread over the whole window; bit 24 of a
    # value ~333 (delta ~1e3) flags its own layer while the layers it reaches
    # 3+ sweeps later stay below eps: a cone of the flagged layers alone
    # (no 2(L - 1) margin) would leave those errors in place.
    p = make_problem("cfg3", nx=48, ny=40, nz=24, sweeps=4 * delta, mode=2, delta=delta)
    ref = _offline(p, [], 0)
    faults = [Fault(1, 11, 7, 9, 24), Fault(delta + 1, 0, 39, 47, 30),
              Fault(2 * delta + 1, 23, 0, 0, 28), Fault(3 * delta + 1, 5, 20, 20, 24),
              Fault(3 * delta + 1, 17, 3, 30, 29)]
    for recovery in (0, 1):
        r = _offline(p, faults, recovery)
        assert r["stats"]["rollbacks"] == 4 and r["stats"]["persistent"] == 0 and r["status"] == 0
        assert r["stats"]["sweeps"] == 8 * delta
        assert (r["u"].view(np.uint32) == ref["u"].view(np.uint32)).all()
        assert np.array_equal(r["A"], ref["A"]) and np.array_equal(r["B"], ref["B"])


def test_partial_reexecution_keeps_layers_no_detected_error_reached():
    # a detected flip in layer 2 and, in the same window, an undetected
    # low-bit flip in layer 20: the full rollback erases both; the partial
    # re-execution (window of 4 sweeps: cone 2 * 3 layers around layer 2)
    # re-executes layers 0..8 only, so the result equals the run with the
    # undetected flip alone
    p = make_problem("cfg3", nx=40, ny=32, nz=24, sweeps=4, mode=2, delta=4)
    hi, lo = Fault(1, 2, 5, 5, 29), Fault(1, 20, 9, 9, 3)
    full = _offline(p, [hi, lo], 0)
    part = _offline(p, [hi, lo], 1)
    only_lo = _offline(p, [lo], 0)
    clean = _offline(p, [], 0)
    assert only_lo["stats"]["rollbacks"] == 0          # the low bit goes undetected
    assert (full["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()
    assert (part["u"].view(np.uint32) == only_lo["u"].view(np.uint32)).all()
    assert not (part["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()


def test_partial_reexecution_is_the_union_of_the_flagged_layers_neighbourhoods():
    # two detected flips far apart (layers 3 and 44) and, in the same window,
    # an undetected low-bit flip half way (layer 24), outside both
    # neighbourhoods (window of 3 sweeps: 2 * 2 layers around each flagged
    # layer, flags at most 2 layers from a flip): only the layers near the
    # detected flips are re-executed, so the result equals the run with the
    # undetected flip alone -- one interval from the lowest to the highest
    # flagged layer would have erased it as the full rollback does
    p = make_problem("cfg3", nx=40, ny=32, nz=48, sweeps=3, mode=2, delta=3)
    hi = [Fault(1, 3, 5, 5, 29), Fault(2, 44, 20, 11, 30)]
    lo = Fault(1, 24, 9, 9, 3)
    full = _offline(p, hi + [lo], 0)
    part = _offline(p, hi + [lo], 1)
    only_lo = _offline(p, [lo], 0)
    clean = _offline(p, [], 0)
    assert only_lo["stats"]["rollbacks"] == 0          # the low bit goes undetected
    assert part["stats"]["rollbacks"] == 1 and part["stats"]["persistent"] == 0
    zs = sorted({r["z"] for r in part["records"]})
    assert zs and min(zs) <= 5 and max(zs) >= 42 and not any(8 <= z <= 39 for z in zs)
    assert (full["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()
    assert (part["u"].view(np.uint32) == only_lo["u"].view(np.uint32)).all()
    assert not (part["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()
    # with every flip detected the union is bitwise the full rollback
    both = _offline(p, hi, 1)
    assert (both["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()
    assert (both["A"] == clean["A"]).all() and (both["B"] == clean["B"]).all()


# ------------------------------- offline, detection by b alone (Q29)

@pytest.mark.parametrize("checksums", [0, 1])
def test_offline_window_detection_closed_form(checksums):
    # Offline windows of one sweep (Delta = 1), one flip at sweep s: the
    # prediction is Theorem 1 applied to the verified checksums of u^{s-1}
    # (the clean row / column sums up to ~1e-8), the actual window-end sums
    # differ from the clean ones by exactly d = flipped - clean.  So b[y]
    # flags iff |d| > eps |S_row + d| and a[x] iff |d| > eps |S_col + d|.
    # checksums = 1 (one vector compared, the second computed only
    # "to enable correction" -- which offline never does): a window is dirty
    # iff b flags, its record has nflag_a = 0 and x = -1; both policies roll
    # the window back, so the result is the fault-free run.
    p = _cfg1_like().replace(mode=2, delta=1, checksums=checksums)
    op = O.OProblem(p)
    u0 = field_u0(p).numpy()
    s = 10
    clean = _clean_states(p, op, u0, s)
    ref = O.run(op, u0, s)
    rng = random.Random(29)
    checked = 0
    for trial in range(80):
        y, x, bit = rng.randrange(64), rng.randrange(64), rng.randrange(31)
        cv = np.array([clean[0, y, x]], np.float32)
        fv = cv.copy()
        O.flip(fv, 0, bit)
        d = float(fv[0]) - float(cv[0])
        Srow = math.fsum(float(v) for v in clean[0, y, :])
        Scol = math.fsum(float(v) for v in clean[0, :, x])
        mb = abs(d) / abs(Srow + d) if math.isfinite(d) else math.inf
        ma = abs(d) / abs(Scol + d) if math.isfinite(d) else math.inf
        if 0.9 * p.eps < mb < 1.1 * p.eps or 0.9 * p.eps < ma < 1.1 * p.eps:
            continue                               # ambiguous band
        r = O.run(op, u0, s, [Fault(s, 0, y, x, bit)])
        expect_b, expect_a = mb > p.eps, ma > p.eps
        dirty = expect_b if checksums == 1 else (expect_a or expect_b)
        first = [q for q in r["records"] if q["status"] == O.REC_WINDOW_DIRTY]
        assert r["stats"]["rollbacks"] == int(dirty) and r["status"] == 0
        if dirty:
            (rec,) = first
            assert rec["sweep"] == s and rec["z"] == 0
            assert rec["nflag_b"] == int(expect_b) and rec["y"] == (y if expect_b else -1)
            assert rec["nflag_a"] == (0 if checksums == 1 else int(expect_a))
            assert rec["x"] == (x if (expect_a and checksums == 0) else -1)
            assert (r["u"].view(np.uint32) == ref["u"].view(np.uint32)).all()
        else:
            assert first == []
        checked += 1
    assert checked > 50


def test_offline_b_only_equals_both_when_b_flags():
    # every flip large enough to flag its b entry (bits 24-30 of values in
    # [323, 343)): comparing b alone rolls back exactly the windows BOTH
    # rolls back, so the field and the checksums are bitwise BOTH's -- the
    # fault-free run -- and the records differ only in the a fields
    p = make_problem("cfg3", nx=40, ny=32, nz=8, sweeps=20, mode=2, delta=5)
    P = field_power(p).numpy()
    u0 = field_u0(p).numpy()
    rng = random.Random(31)
    faults = [Fault(s, rng.randrange(8), rng.randrange(32), rng.randrange(40), rng.randint(24, 30))
              for s in (2, 5, 9, 13, 14, 18)]
    both = O.run(O.OProblem(p, [P]), u0, p.sweeps, faults)
    bonly = O.run(O.OProblem(p.replace(checksums=1), [P]), u0, p.sweeps, faults)
    clean = O.run(O.OProblem(p, [P]), u0, p.sweeps)
    assert both["stats"]["rollbacks"] == 4 and bonly["stats"] == both["stats"]
    for r in (both, bonly):
        assert (r["u"].view(np.uint32) == clean["u"].view(np.uint32)).all()
        assert np.array_equal(r["A"], clean["A"]) and np.array_equal(r["B"], clean["B"])
    strip = lambda q: {k: v for k, v in q.items() if k not in ("nflag_a", "x")}
    assert [strip(q) for q in bonly["records"]] == [strip(q) for q in both["records"]]
    assert all(q["nflag_a"] == 0 and q["x"] == -1 for q in bonly["records"])
    assert all(q["nflag_b"] >= 1 for q in bonly["records"])


# ------------------------- exact-arithmetic pins of the fp32 rounding (Q23)

def _r32(q: Fraction) -> float:
    """q rounded once to the nearest fp32 (ties to even) -- IEEE 754's
    definition of a correctly rounded operation, in exact rational arithmetic
    (independent of the hardware and of the oracle)."""
    if q == 0:
        return 0.0
    s, a = (-1 if q < 0 else 1), abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    ulp = Fraction(2) ** (max(e, -126) - 23)
    m = a / ulp
    n = m.numerator // m.denominator
    rem = m - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return float(s * n * ulp)


def _f(v) -> Fraction:
    return Fraction(float(np.float32(v)))


def test_r32_rounding_helper_matches_numpy():
    # the helper above against numpy's fp64 -> fp32 cast (exact inputs)
    rng = np.random.default_rng(3)
    for v in list(rng.normal(size=200) * 1e3) + [1 + 2 ** -24, 1 + 3 * 2 ** -24, 2 ** -140 * 1.3]:
        assert _r32(Fraction(float(v))) == float(np.float32(v))


@pytest.mark.parametrize("srcs,base,span", [
    ([(0.001, True, 0.0), (0.05, False, 80.0)], 323.0, 20.0),    # HotSpot (cfg2-4)
    ([(0.7, True, 0.0), (0.3, False, 1.7)], 0.0, 1.0),           # sources of the size of the field
])
def test_fp32_sweep_is_the_fused_canonical_chain(srcs, base, span):
    # Q23: an fp32 cell is acc = w_0 v_0, acc = fma(w_p, v_p,
    # acc) over the points in order, then acc = fma(coef_q, src_q, acc): each
    # step ONE rounding of the exact w*v + acc.  Evaluated here in exact
    # rationals with _r32, cell by cell (HotSpot weights, non-dyadic, clamp);
    # the unfused chain (w*v rounded, then the add rounded) differs in many
    # cells, so the pin can fail.
    pts = [(0, 0, 0, 0.4), (-1, 0, 0, 0.1), (1, 0, 0, 0.1), (0, -1, 0, 0.1), (0, 1, 0, 0.1),
           (0, 0, -1, 0.05), (0, 0, 1, 0.05)]
    nz, ny, nx = 3, 5, 6
    p = Problem("t", nx, ny, nz, "f32", pts, srcs)
    rng = np.random.default_rng(11)
    u = (base + span * rng.random((nz, ny, nx))).astype(np.float32)
    P = rng.random((nz, ny, nx)).astype(np.float32)
    out = O.sweep(O.OProblem(p, [P]), u)
    cl = lambda c, n: min(max(c, 0), n - 1)
    unfused_differs = [0, 0]   # chain, sources
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                acc = accu = None
                for di, dj, dk, w in pts:
                    v = Fraction(float(u[cl(z + dk, nz), cl(y + dj, ny), cl(x + di, nx)]))
                    t = _f(w) * v
                    acc = _r32(t) if acc is None else _r32(t + Fraction(acc))
                    accu = _r32(t) if accu is None else _r32(Fraction(_r32(t)) + Fraction(accu))
                unfused_differs[0] += accu != acc
                accs = acc
                for (cf, fld, sc) in srcs:
                    sv = Fraction(float(P[z, y, x])) if fld else _f(sc)
                    acc = _r32(_f(cf) * sv + Fraction(acc))
                    accs = _r32(Fraction(_r32(_f(cf) * sv)) + Fraction(accs))
                assert float(out[z, y, x]) == acc, (z, y, x)
                unfused_differs[1] += accs != acc
    assert unfused_differs[0] > 0 and (base > 0 or unfused_differs[1] > 0)


def test_constant_sums_fp32_round_the_scalar_too():
    # c_x, c_y of an fp32 problem whose scalar source is not an
    # fp32 value (80.3): C is built from the dtype-rounded scalar, as the sweep
    # applies it (Q23); exact rational brute force as in the pin above.
    nz, ny, nx = 2, 5, 7
    p = Problem("t", nx, ny, nz, "f32", [(0, 0, 0, 1.0)], [(0.001, True, 0.0), (0.05, False, 80.3)])
    P = np.random.default_rng(6).random((nz, ny, nx)).astype(np.float32)
    cA, cB = O.constant_sums(O.OProblem(p, [P]))
    C = [[[_f(0.001) * Fraction(float(P[z, y, x])) + _f(0.05) * _f(80.3) for x in range(nx)]
          for y in range(ny)] for z in range(nz)]
    for z in range(nz):
        for x in range(nx):
            ex = sum(C[z][y][x] for y in range(ny))
            assert abs(Fraction(cA[z, x]) - ex) <= ex * Fraction(1, 2 ** 49)
        for y in range(ny):
            ex = sum(C[z][y][x] for x in range(nx))
            assert abs(Fraction(cB[z, y]) - ex) <= ex * Fraction(1, 2 ** 49)
    raw = sum(_f(0.001) * Fraction(float(P[0, y, 0])) + _f(0.05) * Fraction(80.3) for y in range(ny))
    assert abs(Fraction(cA[0, 0]) - raw) > raw * Fraction(1, 10 ** 10)


@pytest.mark.parametrize("bc", [0, 1, 3])
def test_theorem1_fp32_exact_linear_update(bc):
    # Theorem 1 is an identity of the linear update: a'_x equals
    # the column sum of sum_q w_q u(neighbour) + C EXACTLY, for the weights the
    # sweep uses -- fp32-rounded for an fp32 problem (Q23).  The right side is
    # brute force in exact rationals (the stencil applied cell by cell, every
    # ghost read through the BC, then summed); the oracle's fp64 prediction may
    # differ from it only by its own rounding (~1e-15), while unrounded fp64
    # weights (0.1 vs fp32 0.1) would be off by ~1e-9.
    pts = [(0, 0, 0, 0.35), (-1, 0, 0, 0.1), (1, 0, 0, 0.15), (0, -1, 0, 0.1), (0, 1, 0, 0.05),
           (1, 1, 0, 0.1), (0, 0, -1, 0.05), (-1, 0, 1, 0.1)]
    srcs = [(0.001, True, 0.0), (0.05, False, 80.0)]
    nz, ny, nx = 3, 5, 6
    g = 330.5
    p = Problem("t", nx, ny, nz, "f32", pts, srcs, bc=bc, bc_value=g)
    rng = np.random.default_rng(12 + bc)
    u = (323 + 20 * rng.random((nz, ny, nx))).astype(np.float32)
    P = rng.random((nz, ny, nx)).astype(np.float32)
    op = O.OProblem(p, [P])
    A, B = O.checksums(op, u)
    PA, PB = O.predict(op, A, B, u)

    def val(z, y, x):
        if bc == 1:
            return Fraction(float(u[z % nz, y % ny, x % nx]))
        if bc == 0:
            return Fraction(float(u[min(max(z, 0), nz - 1), min(max(y, 0), ny - 1), min(max(x, 0), nx - 1)]))
        if 0 <= z < nz and 0 <= y < ny and 0 <= x < nx:
            return Fraction(float(u[z, y, x]))
        return _f(g)
    lin = [[[sum(_f(w) * val(z + dk, y + dj, x + di) for di, dj, dk, w in pts)
             + _f(0.001) * Fraction(float(P[z, y, x])) + _f(0.05) * _f(80.0)
             for x in range(nx)] for y in range(ny)] for z in range(nz)]
    for z in range(nz):
        for x in range(nx):
            ex = sum(lin[z][y][x] for y in range(ny))
            assert abs(Fraction(PA[z, x]) - ex) <= ex * Fraction(1, 10 ** 13), (z, x)
        for y in range(ny):
            ex = sum(lin[z][y][x] for x in range(nx))
            assert abs(Fraction(PB[z, y]) - ex) <= ex * Fraction(1, 10 ** 13), (z, y)


# ----------------------- forms 0 / 1 with several flags (Q13, Q14)

def test_several_flags_in_a_layer_record_first_row_and_column_uncorrectable():
    # several errors in one layer pair up ambiguously -- forms 0 / 1
    # do not correct them (Q13: |X| >= 2 or |Y| >= 2 is "uncorrectable"), and
    # the record names the first flagged row and column (lowest
    # index) with the flag counts; the field keeps both flipped values.
    p = make_problem("cfg2", nx=40, ny=36, nz=4, sweeps=6)
    op = O.OProblem(p, [field_power(p).numpy()])
    u0 = field_u0(p).numpy()
    ref = O.run(op, u0, 4)
    for form in (0, 1):
        q = p.replace(correction_form=form)
        r = O.run(O.OProblem(q, [field_power(q).numpy()]), u0, 4,
                  [Fault(4, 2, 20, 31, 29), Fault(4, 2, 7, 9, 29)])
        assert r["status"] == 1 and r["stats"]["uncorrectable"] == 1 and r["stats"]["corrected"] == 0
        (rec,) = r["records"]
        assert rec["status"] == O.REC_UNCORRECTABLE
        assert (rec["sweep"], rec["z"], rec["y"], rec["x"]) == (4, 2, 7, 9)
        assert (rec["nflag_a"], rec["nflag_b"]) == (2, 2)
        diff = np.argwhere(r["u"].view(np.uint32) != ref["u"].view(np.uint32))
        assert sorted(map(tuple, diff)) == [(2, 7, 9), (2, 20, 31)]


def test_flag_in_one_vector_only_is_unlocated():
    # fig.abft.error scenario 2 (Q14): a flip that moves its column sum
    # (ny = 8 terms) past eps but not its row sum (nx = 256 terms) flags a
    # alone: detected, not located.  delta = 2^(12 - 15) = 0.125 on a value in
    # [256, 512): column |d| / S ~ 0.125 / 2640 > 1e-5 > row 0.125 / 84480.
    p = make_problem("cfg2", nx=256, ny=8, nz=2, sweeps=3)
    op = O.OProblem(p, [field_power(p).numpy()])
    r = O.run(op, field_u0(p).numpy(), 3, [Fault(2, 1, 5, 100, 12)])
    (rec,) = r["records"]
    assert rec["status"] == O.REC_UNLOCATED and r["stats"]["unlocated"] == 1 and r["status"] == 1
    assert (rec["nflag_a"], rec["nflag_b"]) == (1, 0) and rec["x"] == 100


def test_literal_form_corrects_and_repairs_a_mantissa_flip():
    # fig.correction as listed (form 1) on a mantissa flip: the
    # corrected value is the clean one within the checksum's rounding, and the
    # repaired a, b (a += c - u) are the true sums of the repaired
    # layer, so no later sweep flags (one detection in the whole run).
    p = make_problem("cfg2", nx=48, ny=40, nz=3, sweeps=6).replace(correction_form=1)
    op = O.OProblem(p, [field_power(p).numpy()])
    u0 = field_u0(p).numpy()
    clean = _clean_states(p, op, u0, 3)[1, 17, 23]
    r = O.run(op, u0, 6, [Fault(3, 1, 17, 23, 20)])
    assert r["stats"]["detections"] == 1 and r["stats"]["corrected"] == 1
    (rec,) = r["records"]
    assert (rec["y"], rec["x"]) == (17, 23)
    assert abs(rec["corrected"] - clean) / clean < 1e-6
    A1, B1 = _fsum_checksums(r["u"])
    assert np.max(np.abs(r["A"] - A1) / A1) < 1e-9 and np.max(np.abs(r["B"] - B1) / B1) < 1e-9


# ------------------- partial re-execution: the 2 (L - 1) reach is needed (Q28)

@pytest.mark.parametrize("bc,z0", [(0, 8), (1, 1)])
def test_partial_reach_covers_errors_on_the_unflagged_side(bc, z0):
    # An upwind stencil in z (u^s[z] = 0.98 u[z-1] + 1e-4 u[z+1]): a mantissa
    # flip in layer z0 at a window's first sweep travels up, so after the
    # window (L = 3 sweeps) only layer z0 + 2 flags, while the back-leak has
    # put sub-threshold (fp64-visible) errors in layers z0 and z0 - 2.  Those
    # lie 4 = 2 (L - 1) layers below the flagged one: the re-executed range
    # must reach them for the partial re-execution to equal the full rollback
    # bitwise (P:743-745 via Q28); a reach of L - 1 would leave z0 - 2
    # contaminated.  Periodic z (bc 1, z0 = 1): the reach wraps to the top
    # layer, so every layer is re-executed.
    pts = [(0, 0, -1, 0.98), (0, 0, 1, 1e-4)]
    p = Problem("t", 8, 8, 16, "f64", pts, [], bc=bc, eps=1e-4, mode=2, delta=3, sweeps=3,
                init=(1.0, 2.0))
    op = O.OProblem(p)
    u0 = field_u0(p).numpy()
    f = [Fault(1, z0, 3, 4, 50)]
    clean = O.run(O.OProblem(p.replace(mode=0)), u0, 1)["u"]
    first = O.run(O.OProblem(p.replace(mode=0)), u0, 3, f)["u"]
    ref = O.run(O.OProblem(p.replace(mode=0)), u0, 3)["u"]
    bad = sorted({int(z) for z, _, _ in np.argwhere(first != ref)})
    assert bad == sorted({(z0 - 2) % 16, z0, z0 + 2}), bad
    assert clean[z0, 3, 4] != 0
    full = O.run(op, u0, 3, f)
    part = O.run(O.OProblem(p.replace(recovery=1)), u0, 3, f)
    assert [(r["z"], r["status"]) for r in full["records"]] == [(z0 + 2, O.REC_WINDOW_DIRTY)]
    for r in (full, part):
        assert r["stats"]["rollbacks"] == 1 and r["status"] == 0
        assert (r["u"].view(np.uint64) == ref.view(np.uint64)).all()
