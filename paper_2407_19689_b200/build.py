"""Build libpdot.so in-tree for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# PDOT_BUILD_OUT: build elsewhere (e.g. the PDOT_DEVICE_CHECKS variant next to the product library)
OUT = Path(os.environ.get("PDOT_BUILD_OUT", PKG / "lib" / "libpdot.so"))
SOURCES = ["stream.cu", "screen.cu", "finalize.cu", "solver.cu", "sinkhorn.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    # no FMA contraction: element-wise updates must round like numpy;
    # reductions use explicit __fma_rn
    "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
]


def build_library(verbose: bool = False, force: bool = False) -> Path:
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + [CSRC / "pdot_internal.cuh", CSRC / "pass_ops.cuh", CSRC / "solver_internal.h", PKG.parent / "include" / "pdot.h"]
    if OUT.exists() and not force and all(OUT.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    extra = ["-DPDOT_DEVICE_CHECKS"] if os.environ.get("PDOT_DEVICE_CHECKS") == "1" else []
    extra += os.environ.get("PDOT_NVCC_EXTRA", "").split()  # A/B variants (measurement tooling)
    cmd = [NVCC, *FLAGS, *extra, *map(str, srcs), "-o", str(OUT)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libpdot.so")
    log = OUT.parent / "ptxas.log"
    log.write_text(r.stdout + r.stderr)
    if verbose:
        sys.stdout.write(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build_library(verbose=True, force="--force" in sys.argv))
