#!/usr/bin/env python
"""GPU fault-injection campaign: the paper's experiments (Section V,
PAPER.md:748-951) on the B200 path, through the C-ABI.

    python campaign.py [--exp e1,e2,e3] [--reps R] [--out FILE]

E1 (fig.overhead / fig.error): HotSpot tiles 64x64x8 / 512x512x8,
   128 / 256 iterations, No-ABFT vs Online vs Offline (period 16), error-free
   and with one bit-flip at a random iteration 1..128, cell and bit 0..31:
   mean time per run and mean / median / max l2 error (Eq. 9) against
   the error-free run.
E2 (fig.biterror): 64x64x8, 128 iterations, for every bit position
   0..31, R flips at random iteration and cell: l2 error quartiles per mode,
   detection and correction rates, for Eq. 8 re-summed, Eq. 8 literal and the
   locality recompute (correction_form 2).  The paper's findings:
   bits 0-12 never detected, exponent flips break the literal Eq. 8
   correction, offline rollback erases every detected flip.
E3 (fig.interval): offline detection period 1..128 on both tiles,
   error-free and with one flip: mean time per run.
Offline runs come twice: with the full rollback of a dirty window (the
paper's) and with the partial re-execution of the flagged layers'
light cone (recovery PARTIAL, "exploit stencil locality to reduce the
re-execution cost"; Q28) -- the 512x512x64 tile (cfg3's)
shows what the locality saves when the layers outnumber the cone.

Every run is seeded (abft_inputs); the l2 norm is computed on the device in
fp64.  Prints one JSON object per experiment and writes them to --out.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import random
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from abft_inputs import Fault, field_power, field_u0, make_problem  # noqa: E402

TILES = {"64x64x8": dict(nx=64, ny=64, nz=8, sweeps=128),
         "512x512x8": dict(nx=512, ny=512, nz=8, sweeps=256),
         "512x512x64": dict(nx=512, ny=512, nz=64, sweeps=128)}
MODES = {"none": 0, "online": 1, "offline": 2, "offline_partial": 2}


def problem(tile: str, mode: str, **kw):
    """HotSpot3D-like tile of BASELINE.json configs[1] at the paper's sizes (Table 1,
    P:793; 512x512x64 = configs[2]).  offline_partial: recovery PARTIAL (Q28)."""
    return make_problem("cfg2", **TILES[tile], mode=MODES[mode], delta=kw.pop("delta", 16),
                        recovery=1 if mode == "offline_partial" else 0, **kw)


class Runner:
    """Runs one protected execution on cuda:0 through the C-ABI and returns the
    final field, the records and the device time."""

    def __init__(self, dev=None):
        from paper_1909_00709_b200 import abft
        self.abft = abft
        self.dev = torch.device(dev or "cuda:0")
        self.stream = torch.cuda.Stream(self.dev)
        self._inputs = {}

    def inputs(self, p):
        key = (p.nx, p.ny, p.nz, p.seed)
        if key not in self._inputs:
            self._inputs[key] = (field_u0(p, self.dev), field_power(p, self.dev))
        return self._inputs[key]

    def run(self, p, faults=(), policy=0):
        u0, P = self.inputs(p)
        with torch.cuda.stream(self.stream):
            st = self.abft.from_problem(p, u0, P, device=self.dev, stream=self.stream,
                                        checksum_policy=policy)
            st.set_faults(list(faults))
            # a step with no flip in its range runs as a CUDA graph: capture it
            # before the timed region (abft_stencil_plan; a no-op otherwise)
            st.plan(p.sweeps)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            status = st.step(p.sweeps)
            e1.record(self.stream)
            u = st.read_field()
            recs = st.records()
            stats = st.stats()
            st.destroy()
        torch.cuda.synchronize()
        return dict(u=u, records=recs, stats=stats, status=status, ms=e0.elapsed_time(e1))


def l2(a: torch.Tensor, b: torch.Tensor) -> float:
    """Eq. 9: sqrt(sum (v_ref - v_comp)^2), fp64; inf if non-finite."""
    d = a.to(torch.float64) - b.to(torch.float64)
    v = float(torch.sqrt(torch.sum(d * d)).item())
    return v if math.isfinite(v) else float("inf")


def random_flip(p, rng: random.Random, bit=None, max_sweep=128) -> Fault:
    """random iteration 0..127 (sweeps are 1-based), cell, bit 0..31."""
    return Fault(rng.randint(1, min(max_sweep, p.sweeps)), rng.randrange(p.nz), rng.randrange(p.ny),
                 rng.randrange(p.nx), rng.randrange(32) if bit is None else bit)


def _q(v):
    v = sorted(v)
    if not v:
        return {}
    fin = [x for x in v if math.isfinite(x)]

    def pct(q):
        k = (len(v) - 1) * q
        lo, hi = int(math.floor(k)), int(math.ceil(k))
        return v[lo] + (v[hi] - v[lo]) * (k - lo) if math.isfinite(v[hi]) else v[hi]
    return {"mean": statistics.fmean(fin) if len(fin) == len(v) else float("inf"),
            "q1": pct(0.25), "median": pct(0.5), "q3": pct(0.75), "max": v[-1]}


def exp_e1(R: Runner, reps: int, seed: int = 1, policy: int = 0):
    out = {"exp": "E1 overhead and l2 error, error-free vs one random bit-flip (P:770-838)",
           "policy": policy, "tiles": {}}
    for tile in TILES:
        rng = random.Random(seed)
        ref = R.run(problem(tile, "none"))["u"]
        flips = [random_flip(problem(tile, "none"), rng) for _ in range(reps)]
        res = {}
        for mode in MODES:
            p = problem(tile, mode)
            clean = [R.run(p, policy=policy) for _ in range(3)]
            faulty = [R.run(p, [f], policy=policy) for f in flips]
            res[mode] = {
                "ms_error_free": statistics.median(r["ms"] for r in clean),
                "ms_one_flip_mean": statistics.fmean(r["ms"] for r in faulty),
                "l2_error_free": l2(ref, clean[0]["u"]),
                "l2_one_flip": _q([l2(ref, r["u"]) for r in faulty]),
                "detected": sum(1 for r in faulty if r["stats"]["detections"] > 0),
                "corrected": sum(1 for r in faulty if r["stats"]["corrected"] > 0),
                "rollbacks": sum(r["stats"]["rollbacks"] for r in faulty),
            }
        base = res["none"]["ms_error_free"]
        for mode in ("online", "offline", "offline_partial"):
            res[mode]["overhead_error_free_pct"] = 100.0 * (res[mode]["ms_error_free"] / base - 1.0)
        out["tiles"][tile] = dict(sweeps=TILES[tile]["sweeps"], reps=reps, modes=res)
    return out


def exp_e2(R: Runner, reps: int, seed: int = 2, policy: int = 0, forms=(0, 1, 2)):
    tile = "64x64x8"
    out = {"exp": "E2 error vs bit position, 64x64x8, 128 iterations (P:852-915)", "policy": policy,
           "reps_per_bit": reps, "bits": {}}
    ref = R.run(problem(tile, "none"))["u"]
    for bit in range(32):
        rng = random.Random(seed * 1000 + bit)
        flips = [random_flip(problem(tile, "none"), rng, bit=bit) for _ in range(reps)]
        row = {}
        for mode in MODES:
            for form in (forms if mode == "online" else (0,)):
                p = problem(tile, mode, correction_form=form)
                rs = [R.run(p, [f], policy=policy) for f in flips]
                key = mode if mode != "online" else {0: "online", 1: "online_literal_eq8",
                                                     2: "online_recompute"}[form]
                row[key] = {"l2": _q([l2(ref, r["u"]) for r in rs]),
                            "detected": sum(1 for r in rs if r["stats"]["detections"] > 0),
                            "corrected": sum(1 for r in rs if r["stats"]["corrected"] > 0)}
        out["bits"][bit] = row
    return out


def exp_e3(R: Runner, reps: int, seed: int = 3, policy: int = 0,
           periods=(1, 2, 4, 8, 16, 32, 64, 128)):
    out = {"exp": "E3 offline detection period (P:917-951)", "tiles": {}}
    for tile in TILES:
        rng = random.Random(seed)
        flips = [random_flip(problem(tile, "none"), rng, bit=rng.randint(20, 30)) for _ in range(reps)]
        base = statistics.median(R.run(problem(tile, "none"))["ms"] for _ in range(3))
        rows = {}
        for d in periods:
            p = problem(tile, "offline", delta=d)
            clean = statistics.median(R.run(p)["ms"] for _ in range(3))
            faulty = [R.run(p, [f]) for f in flips]
            part = [R.run(problem(tile, "offline_partial", delta=d), [f]) for f in flips]
            rows[d] = {"ms_error_free": clean, "overhead_error_free_pct": 100.0 * (clean / base - 1.0),
                       "ms_one_flip_mean": statistics.fmean(r["ms"] for r in faulty),
                       "ms_one_flip_mean_partial": statistics.fmean(r["ms"] for r in part),
                       "rollbacks_mean": statistics.fmean(r["stats"]["rollbacks"] for r in faulty)}
        out["tiles"][tile] = dict(no_abft_ms=base, periods=rows)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exp", default="e1,e2,e3")
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--policy", type=int, default=0, help="0 both checksums, 1 lazy (P:271-273)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "campaign.json"))
    a = ap.parse_args()
    if not torch.cuda.is_available():
        raise SystemExit("campaign.py runs on the GPU path only")
    R = Runner()
    results = []
    for e in a.exp.split(","):
        t0 = time.time()
        r = {"e1": exp_e1, "e2": exp_e2, "e3": exp_e3}[e](R, a.reps, policy=a.policy)
        r["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(r), flush=True)
        results.append(r)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
