"""In-tree build of libpipeoptim.so (sm_100a) with nvcc.

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored). nvcc
cross-compiles without a GPU, so `build()` runs on the CPU container too.

Each translation unit compiles to its own object under `build/obj/` (in
parallel, each rebuilt only when it or a header changed), then one link. Only
`pipeoptim_gemm.cu` (the fp32 tensor-core stage GEMM) needs CUTLASS; when no
CUTLASS tree is found it is replaced by `pipeoptim_gemm_stub.cpp`, so the
optimizer kernels (K1/K2/K3), stage ops, LSTM cells and transports always
build.
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
OBJ_DIR = PKG_DIR / "build" / "obj"
LIB_NAME = "libpipeoptim.so"
LIB_PATH = PKG_DIR / LIB_NAME
GEMM_TU = "pipeoptim_gemm.cu"
GEMM_STUB = "pipeoptim_gemm_stub.cpp"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    "-diag-suppress",
    "20012",
    # no --use_fast_math: the kernels rely on IEEE div/sqrt for parity
]


def cutlass_root() -> Path | None:
    """A CUTLASS/CuTe header tree: $CUTLASS_DIR, /usr/local/cutlass, then the
    copies vendored in site-packages (flashinfer, tilelang). None if absent
    (or PO_NO_CUTLASS is set)."""
    import site

    if os.environ.get("PO_NO_CUTLASS"):
        return None
    cands: list[Path] = []
    if os.environ.get("CUTLASS_DIR"):
        cands.append(Path(os.environ["CUTLASS_DIR"]))
    cands.append(Path("/usr/local/cutlass"))
    for root in map(Path, site.getsitepackages()):
        cands += [root / "flashinfer" / "data" / "cutlass", root / "tilelang" / "3rdparty" / "cutlass"]
    for base in cands:
        if (base / "include" / "cutlass" / "cutlass.h").exists() and (base / "include" / "cute").is_dir():
            return base
    return None


def _cutlass_include(base: Path) -> list[str]:
    return [f"-I{base / 'include'}", f"-I{base / 'tools' / 'util' / 'include'}"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libpipeoptim.so")


def sources(cutlass: Path | None) -> list[Path]:
    srcs = sorted(p for p in CSRC.glob("*.cu") if p.name != GEMM_TU or cutlass is not None)
    if cutlass is None:
        srcs.append(CSRC / GEMM_STUB)
    return srcs


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    cutlass = cutlass_root()
    if cutlass is None:
        print("build: no CUTLASS tree found; po_gemm_f32x3 is a stub (stage GEMMs on cuBLAS)", file=sys.stderr)
    srcs = sources(cutlass)
    headers = sorted(INCLUDE.glob("*.h")) + sorted(CSRC.glob("*.cuh"))
    nvcc = nvcc_path()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    objs, jobs = [], []
    for src in srcs:
        obj = OBJ_DIR / (src.stem + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src, *headers]):
            continue
        extra = _cutlass_include(cutlass) if src.name == GEMM_TU else []
        cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, f"-I{INCLUDE}", *extra, "-c", "-o", str(obj) + ".tmp", str(src)]
        if src.suffix == ".cpp":
            cmd[1:1] = ["-x", "cu"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((obj, subprocess.Popen(cmd)))
    failed = [obj.name for obj, p in jobs if p.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    for obj, _ in jobs:
        os.replace(str(obj) + ".tmp", obj)
    if not force and not jobs and LIB_PATH.exists() and not _stale(LIB_PATH, objs):
        return LIB_PATH
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
