"""Build the native library libswdb.so in-tree with nvcc for sm_100a.

    python -m paper_1702_07195_b200.build [--force]

Sources: csrc/api.cu (C-ABI), csrc/kernels.cu (sm_100a kernels),
csrc/prep.cpp (host pre-processor).  The result,
paper_1702_07195_b200/libswdb.so, is git-ignored but travels to the GPU box
with the gpurun snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libswdb.so")
BUILD = os.path.join(PKG, "build")

SOURCES = ["api.cu", "kernels.cu", "prep.cpp"]
HEADERS = ["kernels.cuh", "swdb_internal.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "-I" + os.path.join(ROOT, "include")]
if os.environ.get("SW_ABLATE"):   # performance experiments only (wrong results)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_ABLATE=" + os.environ["SW_ABLATE"]]
if os.environ.get("SW_ARITH"):    # cell arithmetic (kernels.cuh): 2 biased unsigned (default), 1 biased signed, 0 relu
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_ARITH=" + os.environ["SW_ARITH"]]
if os.environ.get("SW_ROWAHEAD"):  # row order of the biased cell loop (experiment)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_ROWAHEAD=" + os.environ["SW_ROWAHEAD"]]
if os.environ.get("SW_UNROLL"):    # columns per unrolled block (experiment)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_UNROLL=" + os.environ["SW_UNROLL"]]
if os.environ.get("SW_BRING"):    # boundary prefetch ring in every boundary-reading kernel (experiment)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_BRING=" + os.environ["SW_BRING"]]
if os.environ.get("SW_S32ROWS"):  # rows per lane of the 32-bit kernel (experiment)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_S32ROWS=" + os.environ["SW_S32ROWS"]]
for _k in ("SW_QPTAIL", "SW_TAILADDR", "SW_ROWS_TRACE"):   # profile tail layout experiments (kernels.cuh)
    if os.environ.get(_k):
        NVCC_FLAGS = NVCC_FLAGS + [f"-D{_k}=" + os.environ[_k]]
if os.environ.get("SW_DEFS"):     # experiment macros: SW_DEFS="SW_X=1 SW_Y=0"
    NVCC_FLAGS = NVCC_FLAGS + ["-D" + d for d in os.environ["SW_DEFS"].split()]
if os.environ.get("SW_PTXAS"):    # experiment: extra ptxas options, SW_PTXAS="-O2 --allow-expensive-optimizations=true"
    NVCC_FLAGS = NVCC_FLAGS + ["-Xptxas", ",".join(os.environ["SW_PTXAS"].split())]
if os.environ.get("SW_DEBUG"):    # device-side bounds checks (slow; debug builds)
    NVCC_FLAGS = NVCC_FLAGS + ["-DSW_DEBUG=1"]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


STAMP = LIB + ".flags"


def _flags_stamp() -> str:
    return " ".join(NVCC_FLAGS)


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    # a library built with another flag set (an experiment variant) is stale
    try:
        with open(STAMP) as f:
            if f.read() != _flags_stamp():
                return True
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "swdb.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src):
        obj = os.path.join(BUILD, src + ".o")
        cmd = [nvcc] + NVCC_FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(_flags_stamp())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
