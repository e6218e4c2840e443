"""Build the in-tree CUDA library (sm_100a) with nvcc.

    python -m paper_2303_11767_b200.build [--force] [-v]

Output: paper_2303_11767_b200/libdgswe_b200.so (git-ignored; travels to the
GPU box with the gpurun snapshot).  The CUDA runtime is linked statically.
The kernels of each polynomial degree live in their own translation unit
(csrc/deg_p*.cu), compiled in parallel, then linked with the ABI unit.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(os.path.dirname(HERE), "build", "dgswe_obj")
OUT = os.path.join(HERE, "libdgswe_b200.so")
SOURCES = ["dgswe_b200.cu"] + [f"deg_p{p}.cu" for p in range(7)]
HEADERS = ["dgswe_kernels.cuh", "dgswe_lo.cuh", "dgswe_adv.cuh", "dgswe_diag.cuh", "dgswe_degree.cuh", "dgswe_params.h",
           "dgswe_ctx.h"]
DEPS = SOURCES + HEADERS

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    header = os.path.join(os.path.dirname(HERE), "include", "dgswe_b200.h")
    return any(os.path.getmtime(os.path.join(SRC, f)) > t for f in DEPS) or \
        os.path.getmtime(header) > t


def _compile(src: str, extra: list, verbose: bool, objdir: str = OBJ) -> str:
    obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, *extra, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", obj,
           os.path.join(SRC, src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, out: str = OUT, extra: list | None = None) -> str:
    """Compile every unit (in parallel) and link ``out``; ``extra`` nvcc
    flags serve experiment builds (e.g. ``-DDG_TIMING``)."""
    if not force and out == OUT and not extra and not _stale():
        return out
    objdir = OBJ if out == OUT else out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, extra or [], verbose, objdir), SOURCES))
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", out + ".tmp", *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
