"""Builds libabft_stencil.so in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_1909_00709_b200.build [--force]

Objects compile in parallel; the shared library lands next to this file so
it travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libabft_stencil.so")
BUILD = os.path.join(HERE, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations or []) if spec else []:
        inc = os.path.join(base, "nccl", "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (expected under site-packages/nvidia/nccl/include)")


def flags() -> list:
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-fmad=false",
                   "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include()]


def _sources():
    # heaviest translation units first (the K1 instantiations), so the
    # parallel build's critical path is as short as possible
    srcs = glob.glob(os.path.join(CSRC, "*.cu"))
    return sorted(srcs, key=lambda f: ("_s3_" not in os.path.basename(f),
                                       not os.path.basename(f).startswith("k2"),
                                       not os.path.basename(f).startswith("k1"), f))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.inc")) + \
        [os.path.join(ROOT, "include", "abft_stencil.h"), __file__]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    fl = flags()

    shared = [d for d in _deps() if not d.endswith(".cu")]
    newest_shared = max(os.path.getmtime(d) for d in shared)

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and \
                os.path.getmtime(obj) >= max(newest_shared, os.path.getmtime(src)):
            return obj   # incremental: source and every shared header older than the object
        cmd = [NVCC] + fl + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        with open(obj + ".log", "w") as f:
            f.write(r.stdout + r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    cmd = [NVCC] + ARCH + ["-shared", "-o", OUT + ".tmp"] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
