#!/usr/bin/env python
"""Benchmark of the ABFT-protected stencil hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

One "step" is one protected sweep of the whole workload: K1 (Eq. 1 sweep +
actual checksums, Eqs. 2-3) and K2 (Theorem 1 prediction, compare, locate,
correct) over every z-layer, with the config's scheduled bit-flips.  The
default workload is BASELINE.json configs[3] (cfg4): HotSpot3D 7-point,
1024^3 fp32, online ABFT, 200 sweeps, one flip per 128-layer slab per 50
sweeps, z-partitioned over N GPUs (one process per GPU; the kernels store the
halo into the neighbours' buffers over CUDA IPC, or NCCL send/recv).  Inputs
(4 GiB per array) are larger than L2, so no flush is needed between steps.

Prints ONE JSON line (rank 0).  `value` = protected GCell-updates/s of the
whole job (max time over ranks); `e2e` = the same through the C-ABI with
host buffers (pinned H2D of u0 and P, init, K sweeps, D2H of the field);
`roofline` = the dominant kernel K1 against the measured HBM copy peak;
`cpu_baseline` = the CPU oracle on a bounded sample (rank 0, N = 1).
`--impl reference` times the oracle as it stands (the reference arm).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
try:
    _CORES = len(os.sched_getaffinity(0))
except AttributeError:
    _CORES = os.cpu_count() or 1
os.environ.setdefault("OMP_NUM_THREADS", str(_CORES))

import torch  # noqa: E402

from abft_inputs import fault_schedule, field_power, field_u0, make_problem  # noqa: E402
from paper_1909_00709_b200 import dist as D  # noqa: E402

METRIC = "protected GCell-updates/s at 1/2/4/8 B200, %HBM roofline, ABFT overhead %"
UNIT = "GCell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-layers", type=int, default=0, help="oracle sample layers (0 = auto)")
    ap.add_argument("--strong", action="store_true",
                    help="split the config's domain over the ranks (default: weak scaling, "
                         "every rank owns a slab of the config's size)")
    ap.add_argument("--nz-per-gpu", type=int, default=0,
                    help="weak scaling: layers per rank (0 = the config's nz; cfg5: 128, its "
                         "per-GPU slab at G=8)")
    ap.add_argument("--policy", default="lazy", choices=["lazy", "both"],
                    help="checksum policy of the headline run (the other is measured too)")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured", mp
    except Exception:
        return 6650.0, "fallback", {}


class Clocks:
    """nvidia-smi sampling during the timed regions (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: str):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "-i", index,
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.windows = []

    def mark(self):
        return time.time()

    def window(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [l.strip().split(", ") for l in self.f.read().splitlines() if l.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for k, n in enumerate(names):
                    if r[5 + k].strip().lower() == "active":
                        reasons.add(n)
        # samples under load: the upper half of the clock distribution while timing
        load = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def timed(stream, fn):
    """device time (ms) of fn() on `stream` with CUDA events, synchronised both sides."""
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def _coll_device():
    import torch.distributed as dist
    return "cuda" if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(v: float, world: int) -> float:
    return D.max_over_ranks(v, world, device=_coll_device())


def sum_over_ranks(v: float, world: int) -> float:
    return D.sum_over_ranks(v, world, device=_coll_device())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def shift(faults, k):
    from abft_inputs import Fault
    return [Fault(f.sweep + k, f.z, f.y, f.x, f.bit) for f in faults]


def stencil_name(p) -> str:
    if len(p.points) == 7 and p.sources:
        return "HotSpot3D 7-point"
    if len(p.points) == 27:
        return "27-point box"
    return f"{len(p.points)}-point"


# ----------------------------------------------------------------- ours
def run_ours(a):
    from paper_1909_00709_b200 import abft
    world, rank, local = dist_env()
    if a.gpus != world and world > 1:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE {world}")
    # ABFT_BENCH_SHARE_GPU=1 (a check of the multi-rank path on a one-GPU box,
    # not a measurement): every rank on cuda:0, gloo for the host collectives
    share = os.environ.get("ABFT_BENCH_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    # N > 1: the z-slab halo moves over CUDA IPC by default -- the kernels store
    # it into the neighbours' mapped buffers (fused halo, NVLink); with
    # ABFT_TRANSPORT=nccl the library posts NCCL send/recv after each sweep
    # instead, every handle of this process sharing one communicator (the
    # library caches it by the unique id broadcast once here)
    transport = os.environ.get("ABFT_TRANSPORT", "ipc") if world > 1 else "none"
    ipc_ctx, nccl_id = None, None
    if transport == "ipc":
        from paper_1909_00709_b200.ipc import IpcContext
        ipc_ctx = IpcContext(rank, world)
    elif transport == "nccl":
        import torch.distributed as dist
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    # online single slab: the checks of sweep s run beside sweep s + 1
    # (abft_schedule AUTO, the default); ABFT_SCHEDULE=1 measures the serial order
    sched = int(os.environ.get("ABFT_SCHEDULE", "0"))

    def handle_kw():
        return dict(z_begin=z0, z_count=zc, rank=rank, nranks=world, nccl_unique_id=nccl_id,
                    schedule=sched)

    def new_handle(*args, **kw):
        nonlocal transport, nccl_id
        st = abft.from_problem(*args, **kw, **handle_kw())
        if transport == "ipc" and not ipc_ctx.link(st):   # collective, lockstep on every rank
            # IPC unavailable on some rank (no peer mapping): NCCL for the rest of the run
            st.destroy()
            import torch.distributed as dist
            obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            transport, nccl_id = "nccl", obj[0]
            st = abft.from_problem(*args, **kw, **handle_kw())
        return st
    p = make_problem(a.config)
    if not a.strong:            # weak scaling: each rank owns a slab of the config's size
        per = a.nz_per_gpu or (128 if a.config == "cfg5" else p.nz)
        p = p.replace(nz=per * world)
    pmode = p.mode              # online (cfg1-4) or offline (cfg5: period 5)
    z0, zc = D.slab(p.nz, world, rank)
    pol = abft.ABFT_CK_LAZY if a.policy == "lazy" else abft.ABFT_CK_BOTH
    pol_other = abft.ABFT_CK_BOTH if pol == abft.ABFT_CK_LAZY else abft.ABFT_CK_LAZY
    cells_local = p.nx * p.ny * zc
    cells_global = p.cells
    K, W = a.steps, a.warmup
    stream = torch.cuda.Stream(dev)
    u0 = field_u0(p, dev, z0, zc)
    P = field_power(p, dev, z0, zc)
    faults = fault_schedule(p, K)
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    idx = vis.split(",")[local] if vis and vis.split(",")[local].isdigit() else str(local)
    clocks = Clocks(idx)

    def protected_run(mode, with_faults, prof=False, policy=pol, prob=None):
        st = new_handle(prob or p, u0, P, device=dev, stream=stream, mode=mode, checksum_policy=policy)
        if with_faults:
            st.set_faults(shift(faults, W))
        st.step(W)
        # single slab, error-free range: capture the CUDA graph of step(K) now
        # (abft_stencil_plan; a no-op otherwise) -- the e2e job below pays it inside
        st.plan(K)
        barrier(world)
        if prof:
            st.profile(True)
        l0 = st.launches
        t0 = clocks.mark()
        ms = timed(stream, lambda: st.step(K))
        clocks.window(t0, clocks.mark())
        out = dict(ms=ms, launches=st.launches - l0)
        if prof:
            out["prof"] = st.profile_read()
        out["stats"] = st.stats()
        out["status"] = st.status()
        st.destroy()
        return out

    # the schedule the library chose for this problem (abft_stencil_field_buffers:
    # three buffers online = the checks of sweep s run beside sweep s + 1)
    cfg_probe, _keep = abft.problem_config(p, P, z_begin=z0, z_count=zc, rank=rank, nranks=world,
                                           schedule=sched)
    nbuf = C.c_int32(0)
    abft.lib().abft_stencil_field_buffers(C.byref(cfg_probe), C.byref(nbuf))
    sched_label = ("pipelined: checks of sweep s beside sweep s + 1" if pmode == 1 and nbuf.value == 3
                   else "serial: checks of sweep s before sweep s + 1")
    with torch.cuda.stream(stream):
        rA = protected_run(pmode, True)               # headline: flips on
        rE = protected_run(pmode, True, policy=pol_other)
        # offline: the same flipped run re-executing only the flagged layers'
        # light cone on a dirty window (recovery PARTIAL, DESIGN Q28)
        # instead of the whole window (bitwise the same result)
        rP = protected_run(pmode, True, prob=p.replace(recovery=1)) if pmode == 2 else None
        # overhead (t_protected / t_unprotected - 1, error-free runs): the
        # three error-free runs interleaved, 7 rounds, median of each (clocks
        # drift under the power cap; interleaving exposes every run to it alike)
        reps = {"B": [], "C": [], "D": []}
        for _ in range(7):
            reps["C"].append(protected_run(abft.ABFT_MODE_NONE, False))      # unprotected
            reps["B"].append(protected_run(pmode, False))                    # protected
            reps["D"].append(protected_run(pmode, False, policy=pol_other))
        rB, rC, rD = (sorted(reps[k], key=lambda r: r["ms"])[3] for k in ("B", "C", "D"))
        # per-kernel device times (CUDA events around every launch) in separate
        # runs, so the events do not perturb the overhead timings above
        rB["prof"] = protected_run(pmode, False, prof=True)["prof"]
        rC["prof"] = protected_run(abft.ABFT_MODE_NONE, False, prof=True)["prof"]
        rD["prof"] = protected_run(pmode, False, prof=True, policy=pol_other)["prof"]
    ck = clocks.stop()
    tA = max_over_ranks(rA["ms"], world)
    tB = max_over_ranks(rB["ms"], world)
    tC = max_over_ranks(rC["ms"], world)
    tD = max_over_ranks(rD["ms"], world)
    tE = max_over_ranks(rE["ms"], world)
    tP = max_over_ranks(rP["ms"], world) if rP is not None else None
    value = cells_global * K / (tA * 1e-3) / 1e9
    # roofline of the dominant kernel K1 (protected, checksums fused): algorithmic
    # bytes = (field read + source read + field write) * cells of the launch
    esz = 4 if p.dtype == "f32" else 8
    nfield = sum(1 for s in p.sources if s[1])
    bytes_cell = (2 + nfield) * esz
    prof = rB["prof"]
    k1_ms = prof["k1_ms"] / max(1, prof["k1_launches"])
    k2_ms = prof["k2_ms"] / max(1, K)      # K2 (+ K3 under the lazy policy) per sweep
    k1_gbs = bytes_cell * cells_local / (k1_ms * 1e-3) / 1e9
    k1_ms_unprot = rC["prof"]["k1_ms"] / max(1, rC["prof"]["k1_launches"])
    k1_ms_other = rD["prof"]["k1_ms"] / max(1, rD["prof"]["k1_launches"])
    k2_ms_other = rD["prof"]["k2_ms"] / max(1, K)
    peak, peak_kind, mp = peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            want = "offline" if pmode == 2 else a.policy
            for e in (tj if isinstance(tj, list) else [tj]):
                if e.get("config") == a.config and e.get("policy", "lazy") == want:
                    traffic = e.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    launches = sum_over_ranks(rA["launches"], world)

    # end to end through the C-ABI with host buffers
    e2e = None
    e2e_ok, e2e_err = 0.0, "another rank failed"
    if not a.no_e2e:
        try:   # pinned host copies of the inputs and the result (12 GiB per cfg4 rank)
            u0h = u0.cpu().pin_memory()
            Ph = P.cpu().pin_memory() if P is not None else None
            outh = torch.empty_like(u0h).pin_memory()
            Pd = torch.empty_like(P) if P is not None else None
            e2e_ok = 1.0
        except RuntimeError as ex:
            e2e_err = str(ex).splitlines()[0][:120]
        # every rank runs the e2e job or none does (it contains collectives)
        e2e_ok = -max_over_ranks(-e2e_ok, world)
        if e2e_ok < 1.0:
            e2e = {"value": None, "unit": UNIT, "unavailable": "pinned host buffers: " + e2e_err}
    if not a.no_e2e and e2e_ok >= 1.0:

        def job():
            if Pd is not None:
                Pd.copy_(Ph, non_blocking=True)
            st = new_handle(p, u0h, Pd, device=dev, stream=stream, checksum_policy=pol)
            st.set_faults(faults)
            st.step(K)
            st.read_field(outh)
            s = st.stats()
            st.destroy()
            return s

        with torch.cuda.stream(stream):
            job()   # warm the caching allocator
            barrier(world)
            te = timed(stream, job)
        te = max_over_ranks(te, world)
        h2d = u0h.numel() * esz + (Ph.numel() * esz if Ph is not None else 0)
        d2h = outh.numel() * esz + 72 + 80 * 4096
        e2e = {"value": cells_global * K / (te * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(h2d, world) / K),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h, world) / K),
               "ms_total": te, "what": "pinned H2D of u0 and P, init (K0), K protected sweeps, "
                                       "D2H of the field + stats; bytes are job totals / K"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(p, a.cpu_layers)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": round(tA / K, 5),
            "higher_is_better": True, "scaling": "strong" if a.strong else "weak",
            "vs_baseline": None,
            "dtype": "f32" if p.dtype == "f32" else "f64",
            "data": "synthetic (seeded splitmix64; Rodinia HotSpot3D inputs not available)",
            "config": {"workload": f"{a.config}: {stencil_name(p)} {p.nx}x{p.ny}x{p.nz} "
                                   f"{p.dtype}, {'online' if pmode == 1 else 'offline (period %d)' % p.delta}"
                                   f" ABFT, {K} sweeps, {len(faults)} scheduled bit-flips",
                       "checksum_policy": ("lazy offline: b alone predicted every sweep, summed and compared at "
                                           "each window end (no correction offline, so a is never needed; "
                                           "PAPER.md:271-273, 496-497; DESIGN.md Q29)" if pmode == 2 else
                                           "lazy: b every sweep, a for layers whose b flags "
                                           "(PAPER.md:271-273, 496-497)") if pol == abft.ABFT_CK_LAZY
                       else ("both offline: a and b at each window end" if pmode == 2 else
                             "both: a and b every sweep in the K1 pass"),
                       "nx": p.nx, "ny": p.ny, "nz": p.nz, "z_per_gpu": zc,
                       "parallelism": (f"z-slab x{world} ({'CUDA IPC fused halo' if transport == 'ipc' else 'NCCL halo'})"
                                       if world > 1 else "1 GPU"),
                       "schedule": sched_label,
                       "l2": "inputs larger than L2 (4 GiB per array); no flush",
                       "k1_grid": list(prof["grid"]), "k1_threads": prof["threads"],
                       "k1_smem": prof["smem"], "k1_layers_per_cta": prof["zchunk"]},
            "abft_overhead_pct": round((tB / tC - 1.0) * 100.0, 3),
            "abft_overhead_with_flips_pct": round((tA / tC - 1.0) * 100.0, 3),
            "other_policy": {"policy": "both" if pol == abft.ABFT_CK_LAZY else "lazy",
                             "abft_overhead_pct": round((tD / tC - 1.0) * 100.0, 3),
                             "abft_overhead_with_flips_pct": round((tE / tC - 1.0) * 100.0, 3),
                             "protected_gcells_with_flips": round(cells_global * K / (tE * 1e-3) / 1e9, 3),
                             "k1_ms": round(k1_ms_other, 5), "check_ms_per_sweep": round(k2_ms_other, 5),
                             "detections": rE["stats"]},
            "offline_partial_recovery": None if tP is None else {
                "what": "the headline's flipped run with recovery PARTIAL: a dirty window re-executes "
                        "only the flagged layers' light cone (P:743-745, DESIGN.md Q28)",
                "protected_gcells_with_flips": round(cells_global * K / (tP * 1e-3) / 1e9, 3),
                "abft_overhead_with_flips_pct": round((tP / tC - 1.0) * 100.0, 3),
                "detections": rP["stats"]},
            "unprotected_gcells": round(cells_global * K / (tC * 1e-3) / 1e9, 3),
            "error_free_protected_gcells": round(cells_global * K / (tB * 1e-3) / 1e9, 3),
            "hbm_roofline_frac_step": round(value * 1e9 * bytes_cell / (peak * 1e9) / world, 4),
            "roofline": {"bound": "hbm", "achieved": round(k1_gbs, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(k1_gbs / peak, 4), "traffic": traffic,
                         "kernel": ("k1_sweep<%s,%s,%s,INJ=0> (protected)" % (
                             "float" if p.dtype == "f32" else "double", stencil_name(p),
                             "K1_CK_B" if pol == abft.ABFT_CK_LAZY else "K1_CK_AB")) if pmode == 1
                         else "k1_sweep (offline: K1_CK_NONE within a window, K1_CK_AB at its end)",
                         "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "algorithmic_bytes_per_launch": bytes_cell * cells_local,
                         "k1_ms": round(k1_ms, 5), "k1_unprotected_ms": round(k1_ms_unprot, 5),
                         "check_ms_per_sweep": round(k2_ms, 5)},
            "detections": rA["stats"], "status": rA["status"],
            "gpu_launches": int(launches),
            "clocks": ck,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ipc_ctx is not None:
        ipc_ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# -------------------------------------------------------------- CPU oracle
def _oracle_sample(p, layers, sweeps):
    """The oracle as it stands on a z-sample of the workload (same generator)."""
    from oracle import oracle as O
    sub = p.replace(nz=layers)
    u0 = field_u0(sub).numpy()
    P = field_power(sub)
    op = O.OProblem(sub, [P.numpy()] if P is not None else [])
    t0 = time.perf_counter()
    O.run(op, u0, sweeps, [])
    dt = time.perf_counter() - t0
    return sub.cells * sweeps, dt


def cpu_baseline(p, layers=0):
    sweeps = 2
    if layers <= 0:   # calibrate to ~15 s of CPU work (>= 2 layers per thread: OpenMP over layers)
        n, dt = _oracle_sample(p, min(p.nz, 2 * int(os.environ["OMP_NUM_THREADS"])), 1)
        rate = n / dt
        layers = int(max(2, min(p.nz, 15.0 * rate / (p.nx * p.ny * sweeps))))
    n, dt = _oracle_sample(p, layers, sweeps)
    return {"value": round(n / dt / 1e9, 6), "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]),
            "kind": "oracle",
            "sample": f"{p.nx}x{p.ny}x{layers} layers of {p.name}, {sweeps} online sweeps, "
                      f"{dt:.1f} s wall (C oracle, OpenMP over layers)"}


def run_reference(a):
    world, rank, local = dist_env()
    if rank != 0:
        return
    p = make_problem(a.config)
    layers = a.cpu_layers if a.cpu_layers > 0 else 4
    from oracle import oracle as O
    sub = p.replace(nz=layers)
    u0 = field_u0(sub).numpy()
    P = field_power(sub)
    op = O.OProblem(sub, [P.numpy()] if P is not None else [])
    for _ in range(a.warmup):
        O.run(op, u0, 1, [])
    t0 = time.perf_counter()
    for _ in range(a.steps):
        O.run(op, u0, 1, [])
    dt = time.perf_counter() - t0
    v = sub.cells * a.steps / dt / 1e9
    sample = (f"each step: one online protected sweep of {p.nx}x{p.ny}x{layers} layers of "
              f"{p.name} (C oracle as it stands, incl. its per-call checksum init)")
    line = {"metric": METRIC, "value": round(v, 6), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(dt / a.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": p.dtype,
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{p.name} (sampled, see cpu_baseline.sample)"},
            "cpu_baseline": {"value": round(v, 6), "unit": UNIT,
                             "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(v, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
