"""Build libbitrev_sm100a.so in-tree with nvcc (sm_100a only).

The library is a plain C-ABI shared object (include/bitrev_b200.h) loaded with
ctypes; no torch headers are involved, so one nvcc invocation builds it.
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
LIB_NAME = "libbitrev_sm100a.so"
LIB_PATH = PKG_DIR / LIB_NAME

SOURCES = [CSRC / "bitrev_capi.cu"]
DEPENDS = SOURCES + [CSRC / "bitrev_kernels.cuh", INCLUDE / "bitrev_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libbitrev_sm100a.so")


def needs_build() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    return any(p.stat().st_mtime > built for p in DEPENDS)


def build_library(force: bool = False, verbose: bool = False, out: Path | None = None,
                  defines: tuple[str, ...] = ()) -> Path:
    """Compile the CUDA sources into LIB_PATH (skipped when up to date).

    out/defines build a tuning variant elsewhere (e.g. -DBITREV_MINB_IP=6)."""
    target = Path(out) if out is not None else LIB_PATH
    if out is None and not force and not needs_build():
        return LIB_PATH
    tmp = target.with_suffix(".so.tmp")
    cmd = [_nvcc(), *NVCC_FLAGS, *(f"-D{d}" for d in defines), f"-I{INCLUDE}", f"-I{CSRC}",
           "-Xptxas", "-v", "-o", str(tmp), *map(str, SOURCES)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG_DIR / "csrc" / ("ptxas.log" if out is None else f"ptxas.{target.stem}.log")
    log.write_text(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode}): {' '.join(cmd)}")
    os.replace(tmp, target)
    if verbose:
        print(f"built {target}")
    return target


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    defines = tuple(a[2:] for a in args if a.startswith("-D"))
    if "--out" in args:
        out = Path(args[args.index("--out") + 1])
    build_library(force="--force" in args, verbose=True, out=out, defines=defines)
