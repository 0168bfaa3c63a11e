"""Python binding of libabft_stencil.so (include/abft_stencil.h).

Argument marshalling only: every step of the protected sweep runs in the
sm_100a kernels behind the C-ABI.  PyTorch is used for device memory and
streams.  There is no fallback: if the shared library is missing or the
device is not a CUDA GPU, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, List, Optional, Sequence, Tuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libabft_stencil.so")
if os.environ.get("ABFT_LIB"):   # A/B experiments against another build (tools/)
    LIB_PATH = os.environ["ABFT_LIB"]

ABFT_OK, ABFT_DETECTED_UNCORRECTABLE, ABFT_PERSISTENT_ERROR = 0, 1, 3
ABFT_EINVAL, ABFT_ENOSPACE, ABFT_ECUDA, ABFT_ENCCL, ABFT_EUNSUPPORTED, ABFT_ETIMEOUT = -1, -2, -3, -4, -5, -6
ABFT_F32, ABFT_F64 = 0, 1
ABFT_BC_CLAMP, ABFT_BC_PERIODIC, ABFT_BC_ZERO, ABFT_BC_CONSTANT = 0, 1, 2, 3
ABFT_MODE_NONE, ABFT_MODE_ONLINE, ABFT_MODE_OFFLINE = 0, 1, 2
ABFT_SCHED_AUTO, ABFT_SCHED_SERIAL = 0, 1
ABFT_CK_BOTH, ABFT_CK_LAZY = 0, 1
ABFT_RECOVER_ROLLBACK, ABFT_RECOVER_PARTIAL = 0, 1
REC_CORRECTED, REC_UNLOCATED, REC_UNCORRECTABLE, REC_WINDOW_DIRTY, REC_PERSISTENT, REC_RECOMPUTED, REC_VERIFIED = 1, 2, 3, 4, 5, 6, 7

EXPORTS = ("abft_stencil_workspace_size", "abft_stencil_init", "abft_stencil_step",
           "abft_stencil_sweep", "abft_stencil_check", "abft_stencil_correct",
           "abft_stencil_set_faults", "abft_stencil_field", "abft_stencil_read_field",
           "abft_stencil_checksums", "abft_stencil_stats", "abft_stencil_records",
           "abft_stencil_status", "abft_stencil_sweep_count", "abft_stencil_launch_count",
           "abft_stencil_destroy", "abft_strerror", "abft_stencil_profile",
           "abft_stencil_profile_read", "abft_stencil_group", "abft_stencil_step_group",
           "abft_stencil_halo_plan", "abft_stencil_ipc_export", "abft_stencil_ipc_link",
           "abft_stencil_plan", "abft_stencil_field_buffers")
IPC_BLOB_BYTES = 1024
IPC_ZWORDS = 256


class abft_point(C.Structure):
    _fields_ = [("di", C.c_int32), ("dj", C.c_int32), ("dk", C.c_int32), ("pad", C.c_int32),
                ("w", C.c_double)]


class abft_source(C.Structure):
    _fields_ = [("coef", C.c_double), ("field", C.c_void_p), ("scalar", C.c_double)]


class abft_config(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz_global", C.c_int64),
                ("z_begin", C.c_int64), ("z_count", C.c_int64),
                ("dtype", C.c_int32), ("bc", C.c_int32), ("bc_value", C.c_double),
                ("npoints", C.c_int32), ("nsources", C.c_int32),
                ("points", C.POINTER(abft_point)), ("sources", C.POINTER(abft_source)),
                ("epsilon", C.c_double), ("mode", C.c_int32), ("delta", C.c_int32),
                ("correction_form", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("checksum_policy", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("recovery", C.c_int32), ("schedule", C.c_int32)]


class abft_fault(C.Structure):
    _fields_ = [("sweep", C.c_int64), ("z", C.c_int64), ("y", C.c_int64), ("x", C.c_int64),
                ("bit", C.c_int32), ("pad", C.c_int32)]


class abft_record(C.Structure):
    _fields_ = [("sweep", C.c_int64), ("z", C.c_int64), ("y", C.c_int64), ("x", C.c_int64),
                ("observed", C.c_double), ("corrected", C.c_double), ("vx", C.c_double),
                ("vy", C.c_double), ("status", C.c_int32), ("nflag_a", C.c_int32),
                ("nflag_b", C.c_int32), ("pad", C.c_int32)]


class abft_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("sweeps", "detections", "located", "corrected",
                                         "unlocated", "uncorrectable", "rollbacks", "windows",
                                         "persistent")]


class abft_ipc_slot(C.Structure):
    _fields_ = [("seq", C.c_int64), ("wseq", C.c_int64), ("wdone", C.c_int64),
                ("val", (C.c_int32 * 3) * 2), ("z_begin", C.c_int32), ("z_count", C.c_int32),
                ("zbits", (C.c_uint32 * IPC_ZWORDS) * 2)]


class AbftError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn}: {abft_strerror(status)} ({status})")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load the in-tree shared library (build it with
    `python -m paper_1909_00709_b200.build`).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run python -m paper_1909_00709_b200.build "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        cfgp = C.POINTER(abft_config)
        L.abft_stencil_workspace_size.argtypes = [cfgp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.abft_stencil_init.argtypes = [cfgp, C.POINTER(vp), vp, vp, vp, C.POINTER(vp)]
        L.abft_stencil_step.argtypes = [vp, i32]
        L.abft_stencil_plan.argtypes = [vp, i32]
        L.abft_stencil_field_buffers.argtypes = [cfgp, C.POINTER(i32)]
        L.abft_stencil_sweep.argtypes = [vp]
        L.abft_stencil_check.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.abft_stencil_correct.argtypes = [vp, C.POINTER(i64)]
        L.abft_stencil_set_faults.argtypes = [vp, C.POINTER(abft_fault), i32]
        L.abft_stencil_field.argtypes = [vp, C.POINTER(vp), C.POINTER(i64)]
        L.abft_stencil_read_field.argtypes = [vp, vp]
        L.abft_stencil_checksums.argtypes = [vp, vp, vp]
        L.abft_stencil_stats.argtypes = [vp, C.POINTER(abft_stats)]
        L.abft_stencil_records.argtypes = [vp, C.POINTER(abft_record), i32, C.POINTER(i64)]
        L.abft_stencil_status.argtypes = [vp]
        L.abft_stencil_sweep_count.argtypes = [vp]
        L.abft_stencil_sweep_count.restype = i64
        L.abft_stencil_launch_count.argtypes = [vp]
        L.abft_stencil_launch_count.restype = i64
        L.abft_stencil_destroy.argtypes = [vp]
        L.abft_stencil_profile.argtypes = [vp, i32]
        L.abft_stencil_profile_read.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(i64),
                                                C.POINTER(C.c_double), C.POINTER(i64),
                                                C.POINTER(i32)]
        L.abft_stencil_halo_plan.argtypes = [cfgp, C.POINTER(i32)]
        L.abft_stencil_group.argtypes = [C.POINTER(vp), i32]
        L.abft_stencil_step_group.argtypes = [C.POINTER(vp), i32, i32]
        L.abft_stencil_ipc_export.argtypes = [vp, vp]
        L.abft_stencil_ipc_link.argtypes = [vp, vp, vp, vp]
        L.abft_strerror.argtypes = [C.c_int]
        L.abft_strerror.restype = C.c_char_p
        _lib = L
    return _lib


def abft_strerror(status: int) -> str:
    return lib().abft_strerror(status).decode()


def _ok(fn: str, status: int, allow_positive: bool = False) -> int:
    if status < 0 or (status > 0 and not allow_positive):
        raise AbftError(fn, status)
    return status


def _dtype_code(dt) -> int:
    if dt in ("f32", torch.float32, ABFT_F32):
        return ABFT_F32
    if dt in ("f64", torch.float64, ABFT_F64):
        return ABFT_F64
    raise ValueError(dt)


def make_config(nx: int, ny: int, nz: int, dtype, points: Sequence[Tuple[int, int, int, float]],
                sources: Sequence[Tuple[float, Optional[torch.Tensor], float]] = (),
                bc: int = ABFT_BC_CLAMP, bc_value: float = 0.0, epsilon: float = 1e-5,
                mode: int = ABFT_MODE_ONLINE, delta: int = 1, correction_form: int = 0,
                z_begin: int = 0, z_count: Optional[int] = None, rank: int = 0,
                nranks: int = 1, nccl_unique_id: Optional[bytes] = None,
                checksum_policy: int = 0, recovery: int = 0, schedule: int = 0):
    """abft_config for the problem as the paper states it (Eq. 1: stencil points
    (di, dj, dk, w) in evaluation order + constant-term sources
    (coef, device field or None, scalar); BC; threshold; offline period).
    Returns (config, keepalive) -- keep `keepalive` referenced while the
    config is in use."""
    pts = (abft_point * len(points))()
    for k, (di, dj, dk, w) in enumerate(points):
        pts[k].di, pts[k].dj, pts[k].dk, pts[k].w = di, dj, dk, float(w)
    srcs = (abft_source * max(1, len(sources)))()
    for k, (coef, field, scalar) in enumerate(sources):
        srcs[k].coef = float(coef)
        srcs[k].scalar = float(scalar)
        srcs[k].field = field.data_ptr() if field is not None else None
    c = abft_config()
    c.nx, c.ny, c.nz_global = nx, ny, nz
    c.z_begin = z_begin
    c.z_count = nz - z_begin if z_count is None else z_count
    c.dtype = _dtype_code(dtype)
    c.bc, c.bc_value = bc, bc_value
    c.npoints, c.nsources = len(points), len(sources)
    c.points = C.cast(pts, C.POINTER(abft_point))
    c.sources = C.cast(srcs, C.POINTER(abft_source))
    c.epsilon, c.mode, c.delta, c.correction_form = epsilon, mode, delta, correction_form
    c.rank, c.nranks = rank, nranks
    c.checksum_policy = checksum_policy
    c.recovery = recovery
    c.schedule = schedule
    idbuf = None
    if nccl_unique_id is not None:
        idbuf = C.create_string_buffer(bytes(nccl_unique_id), 128)
        c.nccl_unique_id = C.cast(idbuf, C.c_void_p)
    return c, (pts, srcs, idbuf)


def abft_stencil_halo_plan(cfg: abft_config) -> List[Tuple[int, int, int]]:
    """[(peer, send_layer, recv_layer)] per face that has a neighbour, lower first."""
    plan = (C.c_int32 * 6)()
    _ok("abft_stencil_halo_plan", lib().abft_stencil_halo_plan(C.byref(cfg), plan))
    return [(plan[3 * f], plan[3 * f + 1], plan[3 * f + 2]) for f in (0, 1) if plan[3 * f] >= 0]


def abft_stencil_workspace_size(cfg: abft_config) -> Tuple[int, int]:
    fb, ab = C.c_size_t(0), C.c_size_t(0)
    _ok("abft_stencil_workspace_size",
        lib().abft_stencil_workspace_size(C.byref(cfg), C.byref(fb), C.byref(ab)))
    return fb.value, ab.value


class Stencil:
    """One handle of the C-ABI on one CUDA device, owning its torch buffers.

    u0: this rank's slab [z_count, ny, nx] (torch tensor on the device or in
    host memory, of the field dtype).  The field / aux buffers are allocated
    with torch on `device`."""

    def __init__(self, cfg: abft_config, keepalive, u0: torch.Tensor, device=None,
                 stream: Optional[torch.cuda.Stream] = None):
        self.cfg, self._keep = cfg, keepalive
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise RuntimeError("abft_stencil runs on CUDA devices only (no CPU fallback)")
        self.dtype = torch.float32 if cfg.dtype == ABFT_F32 else torch.float64
        self.shape = (cfg.z_count, cfg.ny, cfg.nx)
        fb, ab = abft_stencil_workspace_size(cfg)
        # offline: the checkpoint; pipelined online schedule: u^{s-1} for the
        # checks running beside the next sweep
        nb = C.c_int32(2)
        with torch.cuda.device(self.device):
            _ok("abft_stencil_field_buffers", lib().abft_stencil_field_buffers(C.byref(cfg), C.byref(nb)))
        nbuf = nb.value
        self.fields = [torch.empty(fb, dtype=torch.uint8, device=self.device) for _ in range(nbuf)]
        self.aux = torch.empty(ab, dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        if tuple(u0.shape) != self.shape or u0.dtype != self.dtype:
            raise ValueError(f"u0 must be {self.shape} {self.dtype}")
        self._u0 = u0.contiguous()
        # u0 and the source fields may still be in flight on any torch stream
        # (init is not a hot path): the handle's stream starts after them; the
        # allocator keeps the buffers until the handle's stream is done
        torch.cuda.synchronize(self.device)
        cur = torch.cuda.current_stream(self.device)
        if self.stream != cur:
            for t in self.fields + [self.aux] + ([self._u0] if self._u0.is_cuda else []):
                t.record_stream(self.stream)
        bufs = (C.c_void_p * 3)(*([t.data_ptr() for t in self.fields] + [None] * (3 - nbuf)))
        h = C.c_void_p()
        # the library binds the handle to the current device (every later call
        # runs on that device, whatever is current then)
        with torch.cuda.device(self.device):
            _ok("abft_stencil_init",
                lib().abft_stencil_init(C.byref(cfg), bufs, C.c_void_p(self.aux.data_ptr()),
                                        C.c_void_p(self._u0.data_ptr()),
                                        C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h
        self._faults = None

    # -- run ---------------------------------------------------------------
    def step(self, n: int) -> int:
        return _ok("abft_stencil_step", lib().abft_stencil_step(self.h, n), allow_positive=True)

    def plan(self, n: int) -> None:
        """abft_stencil_plan: capture the graph of step(n) from the current state."""
        _ok("abft_stencil_plan", lib().abft_stencil_plan(self.h, n))

    def sweep(self) -> None:
        _ok("abft_stencil_sweep", lib().abft_stencil_sweep(self.h))

    def check(self) -> Tuple[int, int]:
        a, b = C.c_int64(0), C.c_int64(0)
        _ok("abft_stencil_check", lib().abft_stencil_check(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def correct(self) -> int:
        n = C.c_int64(0)
        _ok("abft_stencil_correct", lib().abft_stencil_correct(self.h, C.byref(n)))
        return n.value

    def set_faults(self, faults: Iterable) -> None:
        fl = list(faults)
        arr = (abft_fault * max(1, len(fl)))()
        for k, f in enumerate(fl):
            arr[k].sweep, arr[k].z, arr[k].y, arr[k].x, arr[k].bit = f.sweep, f.z, f.y, f.x, f.bit
        self._faults = arr
        _ok("abft_stencil_set_faults", lib().abft_stencil_set_faults(self.h, arr, len(fl)))

    # -- read-back -----------------------------------------------------------
    def read_field(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.shape, dtype=self.dtype, device=self.device)
        assert out.is_contiguous() and tuple(out.shape) == self.shape and out.dtype == self.dtype
        _ok("abft_stencil_read_field", lib().abft_stencil_read_field(self.h, C.c_void_p(out.data_ptr())))
        return out

    def field_ptr(self) -> Tuple[int, int]:
        p, pitch = C.c_void_p(), C.c_int64(0)
        _ok("abft_stencil_field", lib().abft_stencil_field(self.h, C.byref(p), C.byref(pitch)))
        return p.value, pitch.value

    def checksums(self, device: bool = False) -> Tuple[torch.Tensor, torch.Tensor]:
        dev = self.device if device else "cpu"
        A = torch.empty((self.shape[0], self.shape[2]), dtype=torch.float64, device=dev)
        B = torch.empty((self.shape[0], self.shape[1]), dtype=torch.float64, device=dev)
        _ok("abft_stencil_checksums",
            lib().abft_stencil_checksums(self.h, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr())))
        return A, B

    def stats(self) -> dict:
        s = abft_stats()
        _ok("abft_stencil_stats", lib().abft_stencil_stats(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in abft_stats._fields_}

    def records(self, cap: int = 4096) -> List[dict]:
        arr = (abft_record * cap)()
        n = C.c_int64(0)
        _ok("abft_stencil_records", lib().abft_stencil_records(self.h, arr, cap, C.byref(n)))
        out = []
        for k in range(min(n.value, cap)):
            r = arr[k]
            out.append(dict(sweep=r.sweep, z=r.z, y=r.y, x=r.x, observed=r.observed,
                            corrected=r.corrected, vx=r.vx, vy=r.vy, status=r.status,
                            nflag_a=r.nflag_a, nflag_b=r.nflag_b))
        return out

    def profile(self, enable: bool = True) -> None:
        _ok("abft_stencil_profile", lib().abft_stencil_profile(self.h, int(enable)))

    def profile_read(self) -> dict:
        t1, t2 = C.c_double(0), C.c_double(0)
        n1, n2 = C.c_int64(0), C.c_int64(0)
        geo = (C.c_int32 * 6)()
        _ok("abft_stencil_profile_read",
            lib().abft_stencil_profile_read(self.h, C.byref(t1), C.byref(n1), C.byref(t2),
                                            C.byref(n2), geo))
        return dict(k1_ms=t1.value, k1_launches=n1.value, k2_ms=t2.value, k2_launches=n2.value,
                    grid=(geo[0], geo[1], geo[2]), threads=geo[3], smem=geo[4], zchunk=geo[5])

    def status(self) -> int:
        return _ok("abft_stencil_status", lib().abft_stencil_status(self.h), allow_positive=True)

    @property
    def sweeps(self) -> int:
        return lib().abft_stencil_sweep_count(self.h)

    @property
    def launches(self) -> int:
        return lib().abft_stencil_launch_count(self.h)

    def destroy(self) -> None:
        if getattr(self, "h", None):
            lib().abft_stencil_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def ipc_export(st: Stencil) -> bytes:
    """abft_stencil_ipc_export: this slab's IPC description for its neighbours."""
    buf = C.create_string_buffer(IPC_BLOB_BYTES)
    _ok("abft_stencil_ipc_export", lib().abft_stencil_ipc_export(st.h, buf))
    return buf.raw


def ipc_link(st: Stencil, lo_blob: Optional[bytes], hi_blob: Optional[bytes], shm_addr: int) -> None:
    """abft_stencil_ipc_link: map the neighbours' buffers and events; shm_addr
    is the address of nranks abft_ipc_slot shared by every process of the job."""
    lo = C.create_string_buffer(lo_blob, IPC_BLOB_BYTES) if lo_blob is not None else None
    hi = C.create_string_buffer(hi_blob, IPC_BLOB_BYTES) if hi_blob is not None else None
    _ok("abft_stencil_ipc_link", lib().abft_stencil_ipc_link(st.h, lo, hi, C.c_void_p(shm_addr)))


def _handles(stencils):
    return (C.c_void_p * len(stencils))(*[s.h.value if isinstance(s.h, C.c_void_p) else s.h
                                          for s in stencils])


def group(stencils: Sequence[Stencil]) -> None:
    """abft_stencil_group: link the slab handles of one process (rank order)."""
    hs = _handles(stencils)
    _ok("abft_stencil_group", lib().abft_stencil_group(hs, len(stencils)))
    for s in stencils:
        s._group = stencils


def step_group(stencils: Sequence[Stencil], n: int) -> int:
    hs = _handles(stencils)
    return _ok("abft_stencil_step_group", lib().abft_stencil_step_group(hs, len(stencils), n),
               allow_positive=True)


def problem_config(p, power: Optional[torch.Tensor] = None, **kw):
    """abft_config from an object with the attributes of abft_inputs.Problem
    (duck-typed; this package does not import the generators)."""
    srcs = []
    for (coef, has_field, scalar) in p.sources:
        if has_field and power is None:
            raise ValueError("problem has a field source: pass `power`")
        srcs.append((coef, power if has_field else None, scalar))
    args = dict(bc=p.bc, bc_value=p.bc_value, epsilon=p.eps, mode=p.mode, delta=p.delta,
                correction_form=p.correction_form, checksum_policy=getattr(p, "checksums", 0),
                recovery=getattr(p, "recovery", 0))
    args.update(kw)
    return make_config(p.nx, p.ny, p.nz, p.dtype, p.points, srcs, **args)


def from_problem(p, u0: torch.Tensor, power: Optional[torch.Tensor] = None, device=None,
                 stream=None, **kw) -> Stencil:
    cfg, keep = problem_config(p, power, **kw)
    st = Stencil(cfg, keep, u0, device=device, stream=stream)
    st._power = power
    if power is not None and power.is_cuda and st.stream != torch.cuda.current_stream(st.device):
        power.record_stream(st.stream)   # read by every sweep on the handle's stream
    return st
