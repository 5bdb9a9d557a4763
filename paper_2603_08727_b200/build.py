"""Builds libarkv.so in-tree for sm_100a with nvcc (static cudart, -lineinfo).

    python -m paper_2603_08727_b200.build [--force] [--tuning]

--tuning builds libarkv_tuning.so with -DARKV_TUNING_KNOBS (the A/B measurement knobs of
csrc/kernels.h read their environment variables); the product library is libarkv.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libarkv.so")
OBJ = os.path.join(HERE, "build_obj")
LIB_TUNING = os.path.join(HERE, "libarkv_tuning.so")
OBJ_TUNING = os.path.join(HERE, "build_obj_tuning")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE, "--expt-relaxed-constexpr"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found")
    return p


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    srcs = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force: bool = False, verbose: bool = False, tuning: bool = False) -> str:
    lib, obj_dir = (LIB_TUNING, OBJ_TUNING) if tuning else (LIB, OBJ)
    extra = ["-DARKV_TUNING_KNOBS"] if tuning else []
    if not force and not _stale(lib):
        return lib
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cc = nvcc()

    def comp(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        # ARKV_NVCC_FLAGS: extra defines for A/B builds of compile-time switches (measurement only)
        cmd = [cc, *ARCH, *FLAGS, *extra, *os.environ.get("ARKV_NVCC_FLAGS", "").split(), "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(comp, srcs))
    tmp = lib + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, tuning="--tuning" in sys.argv))
