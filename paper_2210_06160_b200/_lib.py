"""ctypes binding of librtsdf.so (the C ABI in include/rtsdf.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every op raises.  Buffers cross the ABI as raw device pointers
taken from torch tensors (torch is only the allocator/stream provider).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "librtsdf.so"
if os.environ.get("RTSDF_LIB"):  # experiments: an alternative build of the same ABI
    LIB_PATH = Path(os.environ["RTSDF_LIB"])

P = C.c_void_p
I = C.c_int
I64 = C.c_int64
U64 = C.c_uint64
D = C.c_double
F = C.c_float
SZ = C.c_size_t
DP = C.POINTER(C.c_double)


class ResampleDesc(C.Structure):
    """rtsdf_resample_desc (include/rtsdf.h)."""

    _fields_ = [("coarse", P), ("cnx", I), ("cny", I), ("cnz", I),
                ("clo", D * 3), ("ch", D * 3),
                ("fnx", I), ("fny", I), ("fnz", I), ("fh", D * 3)]


# name -> (restype, argtypes); mirrors include/rtsdf.h one to one
SIGNATURES = {
    "rtsdf_version": (C.c_char_p, []),
    "rtsdf_last_error": (C.c_char_p, []),
    "rtsdf_launch_count": (I64, []),
    "rtsdf_count_launches": (None, [I64]),
    "rtsdf_voxelize_ws_bytes": (SZ, [I64]),
    "rtsdf_voxelize": (I, [P, I64, P, I64, DP, DP, I, I, I, P, P, P, P, P, SZ, P]),
    "rtsdf_jfa_init": (I, [P, I, I, I, P, P, P]),
    "rtsdf_jfa_ws_bytes": (SZ, [I, I, I]),
    "rtsdf_jfa_step": (I, [P, P, I, I, I, I, D, D, D, I, I, I, P, SZ, P]),
    "rtsdf_jfa_step_slab": (I, [P, P, P, P, I, I, I, I, I, I, I, I, I, I, D, D, D, I, I, I, I, I, P,
                                SZ, P]),
    "rtsdf_halo_bitmap_words": (I64, [I64]),
    "rtsdf_halo_ws_bytes": (SZ, [I64]),
    "rtsdf_halo_compress": (I, [P, I64, P, P, P, P, SZ, P]),
    "rtsdf_halo_decompress": (I, [P, P, I64, P, P, SZ, P]),
    "rtsdf_jfa_run": (I, [P, P, I, I, I, D, D, D, I, I, I, C.POINTER(I), P, SZ, P]),
    "rtsdf_jfa_run_sdf": (I, [P, P, P, I, I, I, D, D, D, I, I, I, D, P, P, SZ, P]),
    "rtsdf_seeds_to_sdf": (I, [P, P, I, I, I, D, D, D, D, P, P]),
    "rtsdf_seeds_to_sdf_range": (I, [P, P, I, I, I, I, I, D, D, D, D, P, P]),
    "rtsdf_seeds_packed_to_linear": (I, [P, P, I, I, I, P]),
    "rtsdf_seeds_linear_to_packed": (I, [P, P, I, I, I, P]),
    "rtsdf_mask_blocks": (I64, [I64]),
    "rtsdf_resample_mask": (I, [P, I, I, I, DP, DP, I, I, I, DP, D, P, P, P, P, P, P, P, P, P]),
    "rtsdf_compact_ws_bytes": (SZ, [I64]),
    "rtsdf_compact_mask": (I, [P, I64, P, P, P, P, SZ, P]),
    "rtsdf_resample_mask_range": (I, [P, I, I, I, DP, DP, I, I, I, DP, D, I64, I64, P, P, P, P, P,
                                      P, P, P, P]),
    "rtsdf_compact_mask_range": (I, [P, I64, I64, P, P, P, P, SZ, P]),
    "rtsdf_exact_distance": (I, [P, I64, P, I64, P, P]),
    "rtsdf_reference_visibility": (I, [P, I64, P, P, P, I, I, DP, DP, DP, D, I, U64, P, P]),
    "rtsdf_unit_sphere_dirs": (I, [P, I64, I, P, P]),
    "rtsdf_glibc_sincos": (I, [P, I64, P, P, P]),
    "rtsdf_bvh_build_host": (I64, [P, P, I64, P, P, P, P, P]),
    "rtsdf_bvh_build_sah_host": (I64, [P, P, I64, I, P, P, P, P, P]),
    "rtsdf_bvh_packed_bytes": (SZ, [I64, I64]),
    "rtsdf_bvh_pack": (I, [P, P, P, P, P, P, P, P, P, I64, I64, P, P]),
    "rtsdf_ray_query": (I, [P, I64, I64, I, P, P, I64, D, P, P, P, P]),
    "rtsdf_sample_ws_bytes": (SZ, [I64, I]),
    "rtsdf_bvh4_collapse_host": (I64, [P, P, P, P, I64, P, I64]),
    "rtsdf_sample_update": (I, [P, I64, I64, I64, I, P, P, I64, C.POINTER(ResampleDesc), I, U64, I64, P, D, P,
                                P, P, P, P, P, P, P, P, D, P, P, SZ, P]),
    "rtsdf_occlusion": (I, [P, I, I, I, DP, DP, P, P, P, I, I, I, I, DP, D, I, D, D, D, D, D, I,
                            U64, F, P, P]),
    "rtsdf_sphere_trace": (I, [P, I, I, I, DP, DP, P, P, I64, D, I, D, D, P, D, P, P, P, P, P]),
    "rtsdf_trilinear_many": (I, [P, I, I, I, DP, DP, P, I64, P, P]),
    "rtsdf_gbuffer": (I, [P, I64, I64, I, P, P, DP, D, D, I, I, P, P, P, P, P]),
    "rtsdf_lbvh_ws_bytes": (SZ, [I64]),
    "rtsdf_lbvh_nodes": (I64, [I64]),
    "rtsdf_lbvh_build": (I, [P, P, P, I64, I, P, SZ, P, SZ, P, P]),
    "rtsdf_compose": (I, [P, P, P, P, I, I, DP, DP, P, P]),
    "rtsdf_apply_bias": (I, [P, I64, F, P, P]),
}

ERR_NAMES = {1: "invalid argument", 2: "CUDA error", 3: "unsupported dims", 4: "workspace too small"}

_lib = None


def lib():
    """Load librtsdf.so (raises loudly if it was never built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().rtsdf_last_error().decode(errors="replace")
        if rc in (1, 3):
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what} failed ({ERR_NAMES.get(rc, rc)}): {msg}")


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def dvec(values):
    arr = (C.c_double * len(values))(*[float(v) for v in values])
    return C.cast(arr, DP), arr


def stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch_count() -> int:
    return int(lib().rtsdf_launch_count())


def host_ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)
