"""Build libtfb200.so (the C-ABI CUDA library) in-tree for sm_100a.

    python -m paper_1511_07106_b200.build [--force]

Flags: ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false``.
``--fmad=false`` is belt and braces: the exact paths already use
round-to-nearest intrinsics that are never contracted.  No fast-math, so
IEEE division / square root everywhere.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libtfb200.so"
# the bounds-checked debug variant (-DTF_BOUNDS_CHECK, tf_common.cuh): loaded
# only by tests/test_gpu_bounds.py through TFB200_LIB
LIB_CHECKED = PKG / "libtfb200_checked.so"
SOURCES = ["api.cu", "integrate.cu", "raycast.cu", "icp.cu", "extract.cu", "comm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler",
              "-fPIC,-ffp-contract=off", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libtfb200.so")


def _stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> Path:
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    objs = []
    build_dir = PKG / ("_build_checked" if checked else "_build")
    build_dir.mkdir(exist_ok=True)
    log = []
    for s in SOURCES:
        obj = build_dir / (Path(s).stem + ".o")
        extra = os.environ.get("TFB200_NVCC_EXTRA", "").split()  # diagnostics builds only
        if checked:
            extra = extra + ["-DTF_BOUNDS_CHECK"]
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *extra, f"-I{INCLUDE}", "-c", str(CSRC / s), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{r.stdout}\n{r.stderr}")
        objs.append(str(obj))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    (build_dir / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    out = build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv)
    print(out)
