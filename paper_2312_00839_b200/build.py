"""In-tree build of libpipeoptim.so (sm_100a) with nvcc.

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored). nvcc
cross-compiles without a GPU, so `build()` runs on the CPU container too.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_DIR = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO_DIR / "include"
LIB_NAME = "libpipeoptim.so"
LIB_PATH = PKG_DIR / LIB_NAME

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cutlass_include() -> list[str]:
    """CUTLASS/CuTe header trees vendored in the environment (used by
    csrc/pipeoptim_gemm.cu inside our own kernels)."""
    import site

    roots = [Path(p) for p in site.getsitepackages()]
    for root in roots:
        base = root / "flashinfer" / "data" / "cutlass"
        if (base / "include" / "cutlass" / "cutlass.h").exists():
            return [f"-I{base / 'include'}", f"-I{base / 'tools' / 'util' / 'include'}"]
    raise RuntimeError("CUTLASS headers not found (flashinfer/data/cutlass)")
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-shared",
    # no --use_fast_math: the kernels rely on IEEE div/sqrt for parity
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libpipeoptim.so")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    srcs = sources()
    deps = srcs + sorted(INCLUDE.glob("*.h")) + sorted(CSRC.glob("*.cuh"))
    if not force and not _stale(LIB_PATH, deps):
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc_path(), *ARCH_FLAGS, *NVCC_FLAGS, "--expt-relaxed-constexpr", "-diag-suppress", "20012",
           f"-I{INCLUDE}", *_cutlass_include(), "-o", str(tmp), *map(str, srcs), "-lcuda"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
