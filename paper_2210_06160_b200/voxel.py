"""Conservative surface voxelization (K1, rtsdf_voxelize) -- mirrors sdfshadow.voxel.

`voxelize` keeps voxel.py:150-181's signature, validation order and errors
(VoxelizeError on dims/bounds, OutOfBoundsError listing triangle ids); the
occupancy is a CUDA uint8 tensor (nx, ny, nz).  `voxelize_seeds` is the fused
hot-path form used by jump_flood/hybrid_sdf: it emits packed JFA seeds
directly (jfa.py:47-55 folded into the voxel kernel) with no occupancy pass.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, to_device, to_numpy


class VoxelizeError(ValueError):
    pass


class OutOfBoundsError(VoxelizeError):
    def __init__(self, triangle_ids):
        ids = list(triangle_ids)
        shown = ", ".join(str(i) for i in ids[:16])
        more = "" if len(ids) <= 16 else f" (+{len(ids) - 16} more)"
        super().__init__(f"triangles outside voxel bounds: {shown}{more}")
        self.triangle_ids = ids


@dataclass(frozen=True)
class VoxelGrid:
    occupancy: torch.Tensor  # (nx, ny, nz) uint8 CUDA, 1 = occupied
    lo: np.ndarray
    hi: np.ndarray
    # packed self-seeds emitted by the fused kernel (None when not requested)
    seed_packed: torch.Tensor | None = None
    _count: torch.Tensor | None = None  # device int64[2] counters from the kernel

    @property
    def dims(self):
        if self.occupancy is not None:
            return tuple(int(n) for n in self.occupancy.shape)
        return tuple(int(n) for n in self.seed_packed.shape)

    @property
    def cell_size(self):
        return (self.hi - self.lo) / np.array(self.dims, dtype=np.float64)

    @property
    def count(self):
        return int(self.occupancy.sum().item())

    def any_occupied(self) -> bool:
        if self._count is not None:
            return int(self._count[1].item()) > 0
        return bool(self.occupancy.any().item())


class _MeshBuffers:
    """Device copy of a mesh's vertices/triangles plus the voxelizer workspace."""

    def __init__(self, verts, tris):
        self.verts = to_device(np.ascontiguousarray(verts, dtype=np.float64))
        self.tris = to_device(np.ascontiguousarray(tris, dtype=np.int32))
        T = self.tris.shape[0]
        self.ws = torch.empty(int(_lib.lib().rtsdf_voxelize_ws_bytes(T)), dtype=torch.uint8,
                              device=self.verts.device)
        self.counters = torch.zeros(2, dtype=torch.int64, device=self.verts.device)
        self.bad = torch.empty(max(T, 1), dtype=torch.uint8, device=self.verts.device)


def _validate(dims, bounds):
    dims = tuple(int(n) for n in dims)
    if len(dims) != 3 or min(dims) < 2:
        raise VoxelizeError(f"dims must be >= 2 per axis, got {dims}")
    lo = np.asarray(bounds[0], dtype=np.float64)
    hi = np.asarray(bounds[1], dtype=np.float64)
    if np.any(hi <= lo):
        raise VoxelizeError("bounds must have positive extent")
    return dims, lo, hi


def launch_voxelize(buf: _MeshBuffers, dims, lo, hi, occ, seed):
    """Asynchronous K1 launch (no host sync); counters land in buf.counters."""
    T = buf.tris.shape[0]
    _lib.check(_lib.lib().rtsdf_voxelize(
        _lib.ptr(buf.verts), buf.verts.shape[0], _lib.ptr(buf.tris), T,
        (_lib.D * 3)(*lo), (_lib.D * 3)(*hi), dims[0], dims[1], dims[2],
        _lib.ptr(occ), _lib.ptr(seed), _lib.ptr(buf.counters), _lib.ptr(buf.bad),
        _lib.ptr(buf.ws), buf.ws.numel(), _lib.stream()), "voxelize")


def _raise_oob(buf: _MeshBuffers):
    if int(buf.counters[0].item()) > 0:
        bad = to_numpy(buf.bad[: buf.tris.shape[0]])
        raise OutOfBoundsError(np.nonzero(bad)[0].tolist())


def _mesh_arrays(mesh):
    if hasattr(mesh, "vertices"):
        return mesh.vertices, mesh.triangles
    return mesh


def voxelize(mesh, dims, bounds) -> VoxelGrid:
    """Conservative occupancy of `mesh` over a dims-cell grid covering `bounds`."""
    verts, tris = _mesh_arrays(mesh)
    dims, lo, hi = _validate(dims, bounds)
    buf = _MeshBuffers(verts, tris)
    occ = torch.empty(dims, dtype=torch.uint8, device=device())
    launch_voxelize(buf, dims, lo, hi, occ, None)
    _raise_oob(buf)
    return VoxelGrid(occupancy=occ, lo=lo, hi=hi, _count=buf.counters)


def voxelize_seeds(mesh, dims, bounds, check=True, buffers=None, out=None) -> VoxelGrid:
    """Fused K1: packed self-seeds straight from the triangles (no occupancy)."""
    verts, tris = _mesh_arrays(mesh)
    dims, lo, hi = _validate(dims, bounds)
    buf = buffers or _MeshBuffers(verts, tris)
    seed = out if out is not None else torch.empty(dims, dtype=torch.int32, device=device())
    launch_voxelize(buf, dims, lo, hi, None, seed)
    if check:
        _raise_oob(buf)
    return VoxelGrid(occupancy=None, lo=lo, hi=hi, seed_packed=seed, _count=buf.counters)


_DUMP_HEADER = struct.Struct("<3I6f")


def save_voxels(grid: VoxelGrid, path):
    header = _DUMP_HEADER.pack(*grid.dims, *[float(v) for v in grid.lo],
                               *[float(v) for v in grid.hi])
    bits = np.packbits(to_numpy(grid.occupancy).ravel(order="F"))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(bits.tobytes())


def load_voxels(path) -> VoxelGrid:
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _DUMP_HEADER.size:
        raise VoxelizeError("truncated voxel dump")
    nx, ny, nz, lox, loy, loz, hix, hiy, hiz = _DUMP_HEADER.unpack_from(blob)
    bits = np.frombuffer(blob[_DUMP_HEADER.size:], dtype=np.uint8)
    occ = np.unpackbits(bits, count=nx * ny * nz).reshape((nx, ny, nz), order="F")
    return VoxelGrid(occupancy=to_device(np.ascontiguousarray(occ)),
                     lo=np.array([lox, loy, loz]), hi=np.array([hix, hiy, hiz]))


__all__ = ["VoxelizeError", "OutOfBoundsError", "VoxelGrid", "voxelize", "voxelize_seeds",
           "save_voxels", "load_voxels"]
