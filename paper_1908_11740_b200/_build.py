"""Build the in-tree CUDA library (and, for tests/bench, the CPU oracle).

``libpbsm.so`` is compiled with nvcc for sm_100a only and lives next to this
file in ``_lib/`` so it travels with the repo snapshot to the GPU box (it is
git-ignored, not gpurun-ignored).  No JIT cache is used.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_DIR = PKG / "_lib"
LIB_PATH = LIB_DIR / os.environ.get("PBSM_LIB_NAME", "libpbsm.so")
CSRC = PKG / "csrc"
SOURCES = [CSRC / "pbsm.cu"]
HEADERS = [ROOT / "include" / "pbsm.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    deps = SOURCES + sorted(CSRC.glob("*.cuh")) + HEADERS + [Path(__file__)]
    if not force and not _stale(LIB_PATH, deps):
        return LIB_PATH
    LIB_DIR.mkdir(exist_ok=True)
    tmp = LIB_PATH.with_suffix(".so.tmp")
    extra = os.environ.get("PBSM_DEFINES", "").split()  # experiments: -DPBSM_RPT=2 ...
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(tmp),
           *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
