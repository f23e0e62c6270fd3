"""In-tree build of the CUDA library (sm_100a only).

    python -m paper_1503_08809_b200.build

Produces paper_1503_08809_b200/_native/libmodal_b200.so with
    nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -shared ...
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_native", "libmodal_b200.so")
SOURCES = ["mg_api.cu", "mg_gamma.cu", "mg_qtilde.cu", "mg_gamma2d.cu"]
HEADERS = ["mg_common.cuh", "mg_domain.cuh", "mg_dmma.cuh", "mg_gamma.cuh", "mg_bessel.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(SRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "modal_b200.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [NVCC, *FLAGS, "-o", tmp, *[os.path.join(SRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=SRC)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
