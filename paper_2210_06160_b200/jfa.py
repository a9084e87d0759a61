"""3D jump flooding (K2/K3) -- mirrors sdfshadow.jfa (jfa.py:1-187).

SeedGrid keeps the reference's fields and semantics: `seed` is the int32
LINEAR index of each cell's best seed (EMPTY = -1).  Internally the device
works on packed coordinates (i<<20 | j<<10 | k; a dims-dependent i | j | k
layout beyond 1024 cells per axis); `seed` converts on demand so
a drop-in caller sees exactly the reference's array.

`jump_flood(voxels, beta)` is the north-star name for jfa_run + seeds_to_sdf.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from math import gcd

import numpy as np
import torch

from . import _lib
from ._device import device, to_device
from .field import DistanceField, make_field

EMPTY = np.int32(-1)
MAX_DIM = 1024


class NoSeedsError(ValueError):
    pass


@dataclass(frozen=True)
class SeedGrid:
    """Per-cell closest-seed record (jfa.py:27-44)."""

    packed: torch.Tensor  # (nx, ny, nz) int32 CUDA, packed coords, EMPTY = -1
    lo: np.ndarray
    hi: np.ndarray

    @property
    def dims(self):
        return tuple(int(n) for n in self.packed.shape)

    @property
    def cell_size(self):
        return (self.hi - self.lo) / np.array(self.dims, dtype=np.float64)

    @property
    def seed(self) -> torch.Tensor:
        """Reference layout: int32 linear seed index (jfa.py:31)."""
        out = torch.empty_like(self.packed)
        nx, ny, nz = self.dims
        _lib.check(_lib.lib().rtsdf_seeds_packed_to_linear(_lib.ptr(self.packed), _lib.ptr(out),
                                                           nx, ny, nz, _lib.stream()),
                   "seeds_packed_to_linear")
        return out

    def seed_count(self):
        return int((self.packed != EMPTY).sum().item())

    @classmethod
    def from_linear(cls, seed, lo, hi) -> "SeedGrid":
        lin = to_device(seed, torch.int32)
        nx, ny, nz = lin.shape
        _check_dims((nx, ny, nz))
        packed = torch.empty_like(lin)
        _lib.check(_lib.lib().rtsdf_seeds_linear_to_packed(_lib.ptr(lin), _lib.ptr(packed),
                                                           nx, ny, nz, _lib.stream()),
                   "seeds_linear_to_packed")
        return cls(packed, np.asarray(lo, np.float64), np.asarray(hi, np.float64))


def _bits(n: int) -> int:
    return max(1, int(n - 1).bit_length())


def _check_dims(dims):
    """Packed int32 seeds: i<<20 | j<<10 | k while every axis is <= MAX_DIM
    (the fast JFA kernels), else a dims-dependent i | j | k layout that needs
    bits(nx-1) + bits(ny-1) + bits(nz-1) <= 31 (the per-cell kernel)."""
    if max(dims) > MAX_DIM and sum(_bits(int(n)) for n in dims) > 31:
        raise ValueError(f"dims {dims}: packed int32 seeds need bits(nx-1) + bits(ny-1) + "
                         f"bits(nz-1) <= 31")


@lru_cache(maxsize=64)
def integer_weights(hx: float, hy: float, hz: float, dims: tuple) -> tuple:
    """Exact small-integer ratio wx:wy:wz = hx^2:hy^2:hz^2, or (0, 0, 0).

    Uses exact rational arithmetic on the fp64 cell sizes, so the fast
    integer ordering in the kernel is provably the reference's fp64 order
    whenever the integers differ (see csrc/jfa.cu header).
    """
    sq = [Fraction(h) ** 2 for h in (hx, hy, hz)]
    base = min(sq)
    ratios = [s / base for s in sq]
    den = 1
    for r in ratios:
        den = den * r.denominator // gcd(den, r.denominator)
    w = [int(r * den) for r in ratios]
    g = 0
    for v in w:
        g = gcd(g, v)
    w = [v // g for v in w]
    if max(w) > 16:  # csrc/jfa.cu weights_ok (EMPTY-key bound of the v2 pass)
        return (0, 0, 0)
    qmax = sum(wi * (n - 1) ** 2 for wi, n in zip(w, dims))
    if qmax >= 2**28:  # csrc/jfa.cu weights_ok: doubled relative keys need 3 spare bits
        return (0, 0, 0)
    return tuple(w)


def _weights(h, dims):
    return integer_weights(float(h[0]), float(h[1]), float(h[2]), tuple(int(n) for n in dims))


def jfa_init(voxels) -> SeedGrid:
    """Self-seed every occupied cell; NoSeedsError when the grid is empty."""
    if getattr(voxels, "seed_packed", None) is not None:
        if not voxels.any_occupied():
            raise NoSeedsError("voxel grid has no occupied cells")
        return SeedGrid(packed=voxels.seed_packed.clone(), lo=voxels.lo, hi=voxels.hi)
    occ = to_device(voxels.occupancy, torch.uint8)
    nx, ny, nz = occ.shape
    _check_dims((nx, ny, nz))
    seed = torch.empty(occ.shape, dtype=torch.int32, device=occ.device)
    count = torch.zeros(1, dtype=torch.int64, device=occ.device)
    _lib.check(_lib.lib().rtsdf_jfa_init(_lib.ptr(occ), nx, ny, nz, _lib.ptr(seed),
                                         _lib.ptr(count), _lib.stream()), "jfa_init")
    if int(count.item()) == 0:
        raise NoSeedsError("voxel grid has no occupied cells")
    return SeedGrid(packed=seed, lo=np.asarray(voxels.lo), hi=np.asarray(voxels.hi))


def jfa_offsets(dims):
    """Offset schedule n/2 ... 1 for n = smallest power of two >= max(dims)."""
    n = 1
    while n < max(dims):
        n *= 2
    offsets = []
    step = n // 2
    while step >= 1:
        offsets.append(step)
        step //= 2
    return offsets


_WS: dict = {}


def workspace(nx: int, ny: int, nz: int) -> torch.Tensor:
    """Per-device JFA workspace (the integer-tie fix-up list), grown on demand.
    Shared by every JFA launch of this process on that device's streams."""
    need = int(_lib.lib().rtsdf_jfa_ws_bytes(int(nx), int(ny), int(nz)))
    dev = device()
    ws = _WS.get(dev.index)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        _WS[dev.index] = ws
    return ws


def launch_step(src: torch.Tensor, dst: torch.Tensor, offset: int, h, w):
    nx, ny, nz = src.shape
    ws = workspace(nx, ny, nz)
    _lib.check(_lib.lib().rtsdf_jfa_step(_lib.ptr(src), _lib.ptr(dst), nx, ny, nz, int(offset),
                                         float(h[0]), float(h[1]), float(h[2]), *w,
                                         _lib.ptr(ws), ws.numel(), _lib.stream()), "jfa_step")


def jfa_step(seeds: SeedGrid, offset: int) -> SeedGrid:
    """One flooding pass at `offset`; pure function of its input (jfa.py:128-137)."""
    dims = seeds.dims
    if not 1 <= offset <= jfa_offsets(dims)[0]:
        raise ValueError(f"offset {offset} out of range for dims {dims}")
    h = seeds.cell_size
    dst = torch.empty_like(seeds.packed)
    launch_step(seeds.packed, dst, offset, h, _weights(h, dims))
    return SeedGrid(packed=dst, lo=seeds.lo, hi=seeds.hi)


def flood_inplace(a: torch.Tensor, b: torch.Tensor, h) -> torch.Tensor:
    """Full schedule ping-ponging a (init seeds) <-> b (one C call: sparse early
    passes, v2 pass kernel); returns the buffer holding the result."""
    nx, ny, nz = (int(n) for n in a.shape)
    w = _weights(h, (nx, ny, nz))
    ws = workspace(nx, ny, nz)
    which = ctypes.c_int(0)
    _lib.check(_lib.lib().rtsdf_jfa_run(_lib.ptr(a), _lib.ptr(b), nx, ny, nz, float(h[0]),
                                        float(h[1]), float(h[2]), *w, ctypes.byref(which),
                                        _lib.ptr(ws), ws.numel(), _lib.stream()), "jfa_run")
    return b if which.value else a


def flood_to_sdf(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, h, beta=0.0,
                 empty_count=None, ws=None):
    """Full schedule with seeds -> SDF fused into the last pass (a, b clobbered).
    ws: a private workspace (rtsdf_jfa_ws_bytes) for callers that flood on a
    stream of their own; None = the shared per-device one."""
    nx, ny, nz = a.shape
    w = _weights(h, (nx, ny, nz))
    if ws is None:
        ws = workspace(nx, ny, nz)
    _lib.check(_lib.lib().rtsdf_jfa_run_sdf(_lib.ptr(a), _lib.ptr(b), _lib.ptr(out), nx, ny, nz,
                                            float(h[0]), float(h[1]), float(h[2]), *w,
                                            float(beta), _lib.ptr(empty_count), _lib.ptr(ws),
                                            ws.numel(), _lib.stream()), "jfa_run_sdf")


def jfa_run(voxels) -> SeedGrid:
    """Full schedule over a voxel grid (jfa.py:140-145)."""
    seeds = jfa_init(voxels)
    out = flood_inplace(seeds.packed, torch.empty_like(seeds.packed), seeds.cell_size)
    return SeedGrid(packed=out, lo=seeds.lo, hi=seeds.hi)


def launch_seeds_to_sdf(packed: torch.Tensor, out: torch.Tensor, h, beta, empty_count=None):
    nx, ny, nz = packed.shape
    _lib.check(_lib.lib().rtsdf_seeds_to_sdf(_lib.ptr(packed), _lib.ptr(out), nx, ny, nz,
                                             float(h[0]), float(h[1]), float(h[2]), float(beta),
                                             _lib.ptr(empty_count), _lib.stream()),
               "seeds_to_sdf")


def seeds_to_sdf(seeds: SeedGrid, beta: float = 0.0, bounds=None) -> DistanceField:
    """World-unit distance to the recorded seed centre minus beta (jfa.py:163-181)."""
    if beta < 0:
        raise ValueError("beta must be >= 0")
    if bounds is not None:
        lo = np.asarray(bounds[0], dtype=np.float64)
        hi = np.asarray(bounds[1], dtype=np.float64)
        if not (np.allclose(lo, seeds.lo) and np.allclose(hi, seeds.hi)):
            raise ValueError("bounds differ from the seed grid's world box")
    out = torch.empty(seeds.dims, dtype=torch.float32, device=seeds.packed.device)
    empty = torch.zeros(1, dtype=torch.int64, device=seeds.packed.device)
    launch_seeds_to_sdf(seeds.packed, out, seeds.cell_size, beta, empty)
    if int(empty.item()) > 0:
        raise NoSeedsError("seed grid incomplete: flood before converting")
    return make_field(out, seeds.lo, seeds.hi, beta=beta)


def default_beta(voxels_or_seeds) -> float:
    h = voxels_or_seeds.cell_size
    return 0.5 * float(np.linalg.norm(h))


def jump_flood(voxels, beta: float = 0.0) -> DistanceField:
    """North-star name for jfa_run followed by seeds_to_sdf, fused on the device
    (the last pass writes the SDF)."""
    if beta < 0:
        raise ValueError("beta must be >= 0")
    seeds = jfa_init(voxels)
    out = torch.empty(seeds.dims, dtype=torch.float32, device=seeds.packed.device)
    empty = torch.zeros(1, dtype=torch.int64, device=out.device)
    flood_to_sdf(seeds.packed, torch.empty_like(seeds.packed), out, seeds.cell_size, beta, empty)
    if int(empty.item()) > 0:
        raise NoSeedsError("seed grid incomplete: flood before converting")
    return make_field(out, seeds.lo, seeds.hi, beta=beta)


__all__ = ["EMPTY", "NoSeedsError", "SeedGrid", "jfa_init", "jfa_offsets", "jfa_step",
           "jfa_run", "seeds_to_sdf", "default_beta", "jump_flood", "integer_weights",
           "flood_inplace", "device"]
