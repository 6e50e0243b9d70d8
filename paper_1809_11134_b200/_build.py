"""Builds libisq.so (the sm_100a kernels + C ABI) in-tree with nvcc.

The library has no torch dependency: it links the CUDA runtime statically and
exposes the plain C ABI declared in include/isq.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = Path(os.environ.get("ISQ_BUILD_DIR") or ROOT / "build" / "isq")
LIB = Path(os.environ.get("ISQ_LIBRARY") or PKG / "libisq.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xptxas",
    "-v",
    "--expt-relaxed-constexpr",
    f"-I{ROOT / 'include'}",
]


def _nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "isq.h", Path(__file__)]
    return any(p.stat().st_mtime > mtime for p in deps if p.exists())


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    BUILD.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()

    def compile_one(src: Path) -> tuple[Path, str]:
        obj = BUILD / (src.stem + ".o")
        extra = os.environ.get("ISQ_NVCC_EXTRA", "").split()
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{proc.stdout}\n{proc.stderr}")
        return obj, proc.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    log = "\n".join(r[1] for r in results)
    (BUILD / "ptxas.log").write_text(log)
    if verbose:
        print(log, file=sys.stderr)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *[str(r[0]) for r in results]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    try:
        build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    except RuntimeError as exc:
        print("BUILD FAILED\n" + str(exc)[-3000:], file=sys.stderr)
        print("BUILD FAILED")
        sys.exit(1)
    print("built", LIB)
