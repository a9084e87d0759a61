"""Build librtsdf.so (all CUDA kernels + the C ABI) in-tree for sm_100a.

Plain nvcc, no torch extension machinery: the library exports only the
`extern "C"` surface declared in include/rtsdf.h and is loaded with ctypes.
--fmad=false keeps every fp64 expression un-contracted (the reference's
numba kernels emit DMUL/DADD only).  Kernels that want
FMA for exact-integer arithmetic call fma intrinsics explicitly.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "librtsdf.so"
SOURCES = ["api.cu", "voxel.cu", "jfa.cu", "resample.cu", "bvh.cu", "raysample.cu", "raymarch.cu",
           "validate.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rtsdf.h"]
    return any(d.stat().st_mtime > mtime for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    extra = os.environ.get("RTSDF_NVCC_EXTRA", "").split()  # experiments, e.g. -DWF_MINB=6
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-o", str(tmp),
           *[str(CSRC / s) for s in SOURCES], "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = (res.stdout or "") + (res.stderr or "")
    (PKG / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed (exit {res.returncode}); see {PKG / 'build.log'}")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
