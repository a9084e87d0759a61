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
SOURCES = ["api.cu", "voxel.cu", "jfa.cu", "halo.cu", "resample.cu", "bvh.cu", "lbvh.cu",
           "raysample.cu", "raymarch.cu", "validate.cu"]

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


STAMP = LIB.with_suffix(".so.sha256")


def source_hash() -> str:
    """sha256 over every source, header and the compile command: the library is
    rebuilt whenever any of them differs from what the present .so was built
    from (content, not mtimes -- a pushed tree keeps no reliable mtimes)."""
    import hashlib

    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS + os.environ.get("RTSDF_NVCC_EXTRA", "").split()).encode())
    deps = [CSRC / s for s in SOURCES] + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.inc"))
    for d in deps + [ROOT / "include" / "rtsdf.h"]:
        h.update(d.name.encode())
        h.update(d.read_bytes())
    return h.hexdigest()


def needs_build() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit in parallel (nvcc -c per .cu), then link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    tmp = LIB.with_suffix(".so.tmp")
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    extra = os.environ.get("RTSDF_NVCC_EXTRA", "").split()  # experiments, e.g. -DWF_MINB=6
    comp = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc(), *comp, *extra, "-I", str(ROOT / "include"), "-c", "-o", str(obj),
               str(CSRC / src)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r, obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(" ".join(c) + "\n" + (r.stdout or "") + (r.stderr or "") for c, r, _ in results)
    failed = [c for c, r, _ in results if r.returncode != 0]
    if not failed:
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                "-fPIC", "-o", str(tmp), *[str(o) for _, _, o in results], "-lcudart"]
        r = subprocess.run(link, capture_output=True, text=True)
        log += " ".join(link) + "\n" + (r.stdout or "") + (r.stderr or "")
        if r.returncode != 0:
            failed = [link]
    (PKG / "build.log").write_text(log)
    if failed:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed; see {PKG / 'build.log'}")
    if verbose:
        sys.stderr.write(log)
    os.replace(tmp, LIB)
    STAMP.write_text(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
