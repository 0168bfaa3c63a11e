"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It never imports the CUDA
package (paper_1909_00709_b200) and the CUDA package never imports it.
See abft_oracle.h for the functions and their PAPER.md citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

OR_F32, OR_F64 = 0, 1
REC_CORRECTED, REC_UNLOCATED, REC_UNCORRECTABLE, REC_WINDOW_DIRTY, REC_PERSISTENT, REC_RECOMPUTED, REC_VERIFIED = 1, 2, 3, 4, 5, 6, 7


class Point(C.Structure):
    _fields_ = [("di", C.c_int32), ("dj", C.c_int32), ("dk", C.c_int32), ("pad", C.c_int32),
                ("w", C.c_double)]


class Source(C.Structure):
    _fields_ = [("coef", C.c_double), ("field", C.c_void_p), ("scalar", C.c_double)]


class FaultS(C.Structure):
    _fields_ = [("sweep", C.c_int64), ("z", C.c_int64), ("y", C.c_int64), ("x", C.c_int64),
                ("bit", C.c_int32), ("armed", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("sweep", C.c_int64), ("z", C.c_int64), ("y", C.c_int64), ("x", C.c_int64),
                ("observed", C.c_double), ("corrected", C.c_double), ("vx", C.c_double),
                ("vy", C.c_double), ("status", C.c_int32), ("nflag_a", C.c_int32),
                ("nflag_b", C.c_int32), ("pad", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("sweeps", "detections", "located", "corrected",
                                         "unlocated", "uncorrectable", "rollbacks", "windows",
                                         "persistent")]


class ProblemS(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dtype", C.c_int32), ("bc", C.c_int32), ("bc_value", C.c_double),
                ("npoints", C.c_int32), ("nsources", C.c_int32),
                ("points", C.POINTER(Point)), ("sources", C.POINTER(Source)),
                ("eps", C.c_double), ("mode", C.c_int32), ("delta", C.c_int32),
                ("correction_form", C.c_int32), ("checksums", C.c_int32),
                ("recovery", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile liboracle.so with the oracle's Makefile (gcc -ffp-contract=off)."""
    if force or not os.path.exists(_SO) or \
            os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "abft_oracle.c")):
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "liboracle.so"],
                       check=True)
    return _SO


_lib_handle = None


def lib():
    global _lib_handle
    if _lib_handle is None:
        build()
        L = C.CDLL(_SO)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        P = C.POINTER(ProblemS)
        L.or_flip.argtypes = [vp, i64, i32, i32]
        L.or_sweep.argtypes = [P, vp, vp, i64, C.POINTER(FaultS), i64]
        L.or_checksums.argtypes = [P, vp, vp, vp]
        L.or_constant_sums.argtypes = [P, vp, vp]
        L.or_predict.argtypes = [P, vp, vp, vp, vp, vp, vp, vp]
        L.or_flag.argtypes = [C.c_double, C.c_double, C.c_double]
        L.or_flag.restype = i32
        L.or_run.argtypes = [P, vp, vp, vp, i64, i64, C.POINTER(FaultS), i64,
                             C.POINTER(Record), i64, C.POINTER(i64), C.POINTER(Stats)]
        L.or_run.restype = i32
        _lib_handle = L
    return _lib_handle


def _np_dtype(dtype: str):
    return np.float32 if dtype == "f32" else np.float64


class OProblem:
    """Marshals an abft_inputs.Problem (+ its source fields) into or_problem.
    Keeps every referenced buffer alive."""

    def __init__(self, prob, fields: Sequence[Optional[np.ndarray]] = ()):
        self.prob = prob
        self.npdt = _np_dtype(prob.dtype)
        pts = (Point * len(prob.points))()
        for k, (di, dj, dk, w) in enumerate(prob.points):
            pts[k].di, pts[k].dj, pts[k].dk, pts[k].w = di, dj, dk, w
        self._fields = []
        srcs = (Source * max(1, len(prob.sources)))()
        fi = iter(fields)
        for k, (coef, has_field, scalar) in enumerate(prob.sources):
            srcs[k].coef = coef
            srcs[k].scalar = scalar
            if has_field:
                f = np.ascontiguousarray(next(fi), dtype=self.npdt)
                assert f.size == prob.cells
                self._fields.append(f)
                srcs[k].field = f.ctypes.data
            else:
                srcs[k].field = None
        self._pts, self._srcs = pts, srcs
        s = ProblemS()
        s.nx, s.ny, s.nz = prob.nx, prob.ny, prob.nz
        s.dtype = OR_F32 if prob.dtype == "f32" else OR_F64
        s.bc, s.bc_value = prob.bc, prob.bc_value
        s.npoints, s.nsources = len(prob.points), len(prob.sources)
        s.points = C.cast(pts, C.POINTER(Point))
        s.sources = C.cast(srcs, C.POINTER(Source))
        s.eps, s.mode, s.delta = prob.eps, prob.mode, prob.delta
        s.correction_form = prob.correction_form
        s.checksums = getattr(prob, "checksums", 0)
        s.recovery = getattr(prob, "recovery", 0)
        self.s = s

    @property
    def ref(self):
        return C.byref(self.s)

    def field(self, a) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(a), dtype=self.npdt)
        assert a.size == self.prob.cells
        return a


def _faults(faults) -> "C.Array":
    arr = (FaultS * max(1, len(faults)))()
    for k, f in enumerate(faults):
        arr[k].sweep, arr[k].z, arr[k].y, arr[k].x = f.sweep, f.z, f.y, f.x
        arr[k].bit, arr[k].armed = f.bit, 1
    return arr


def flip(a: np.ndarray, idx: int, bit: int) -> None:
    """In-place single bit-flip of element idx of a contiguous array."""
    assert a.flags.c_contiguous
    lib().or_flip(a.ctypes.data, idx, OR_F32 if a.dtype == np.float32 else OR_F64, bit)


def sweep(op: OProblem, u: np.ndarray, sweep_idx: int = 1, faults=()) -> np.ndarray:
    u = op.field(u)
    out = np.empty_like(u)
    fa = _faults(list(faults))
    lib().or_sweep(op.ref, u.ctypes.data, out.ctypes.data, sweep_idx, fa, len(faults))
    return out.reshape(op.prob.nz, op.prob.ny, op.prob.nx)


def checksums(op: OProblem, u: np.ndarray):
    u = op.field(u)
    p = op.prob
    A = np.empty((p.nz, p.nx), np.float64)
    B = np.empty((p.nz, p.ny), np.float64)
    lib().or_checksums(op.ref, u.ctypes.data, A.ctypes.data, B.ctypes.data)
    return A, B


def constant_sums(op: OProblem):
    p = op.prob
    cA = np.empty((p.nz, p.nx), np.float64)
    cB = np.empty((p.nz, p.ny), np.float64)
    lib().or_constant_sums(op.ref, cA.ctypes.data, cB.ctypes.data)
    return cA, cB


def predict(op: OProblem, A, B, uprev, cA=None, cB=None):
    p = op.prob
    uprev = op.field(uprev)
    if cA is None:
        cA, cB = constant_sums(op)
    A = np.ascontiguousarray(A, np.float64)
    B = np.ascontiguousarray(B, np.float64)
    cA = np.ascontiguousarray(cA, np.float64)
    cB = np.ascontiguousarray(cB, np.float64)
    PA = np.empty((p.nz, p.nx), np.float64)
    PB = np.empty((p.nz, p.ny), np.float64)
    lib().or_predict(op.ref, A.ctypes.data, B.ctypes.data, uprev.ctypes.data,
                     cA.ctypes.data, cB.ctypes.data, PA.ctypes.data, PB.ctypes.data)
    return PA, PB


def flag(pred: float, act: float, eps: float) -> int:
    return int(lib().or_flag(pred, act, eps))


def run(op: OProblem, u0, nsweeps: int, faults=(), sweep0: int = 0,
        cap: int = 1 << 16) -> Dict:
    """Full protected run (online / offline / none per the problem's mode)."""
    p = op.prob
    u = op.field(u0).copy()
    A = np.empty((p.nz, p.nx), np.float64)
    B = np.empty((p.nz, p.ny), np.float64)
    fa = _faults(list(faults))
    recs = (Record * cap)()
    nrec = C.c_int64(0)
    st = Stats()
    status = lib().or_run(op.ref, u.ctypes.data, A.ctypes.data, B.ctypes.data, sweep0, nsweeps,
                          fa, len(faults), recs, cap, C.byref(nrec), C.byref(st))
    records = []
    for k in range(min(nrec.value, cap)):
        r = recs[k]
        records.append(dict(sweep=r.sweep, z=r.z, y=r.y, x=r.x, observed=r.observed,
                            corrected=r.corrected, vx=r.vx, vy=r.vy, status=r.status,
                            nflag_a=r.nflag_a, nflag_b=r.nflag_b))
    stats = {n: getattr(st, n) for n, _ in Stats._fields_}
    return dict(u=u.reshape(p.nz, p.ny, p.nx), A=A, B=B, records=records, nrec=nrec.value,
                stats=stats, status=int(status))
