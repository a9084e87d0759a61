"""Fine-field refinement (K4, K6, K7) -- mirrors sdfshadow.raysample.

    f_t = min(alpha * f_{t-1} + (1 - alpha) * c_t, r_t)   for c_t <= d
    f_t = c_t                                             for c_t >  d

`update_fine` keeps raysample.py:247-305's signature, validation and return
value (fine DistanceField, AccumulatorField), and runs three device stages:
resample + mask + band-exit reset (one full-grid pass), ordered compaction of
the masked texels, and the fused ray-sample + Eq. 1 kernel.  The accumulator
state lives on the device (CUDA tensors).  `ray_sample_sdf` is the north-star
name for update_fine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from ._device import device, to_device, to_numpy
from .field import DistanceField, make_field
from .geometry import BvhIndex, ray_query_many

INF = np.float32(np.inf)


@dataclass(frozen=True)
class SamplingParams:
    """Tunable constants (raysample.py:32-52): x, d, alpha, seed, t_max."""

    rays_per_frame: int = 5
    mask_distance: float = 0.1
    decay_alpha: float = 0.95
    seed: int = 0
    t_max: float | None = None

    def __post_init__(self):
        if self.rays_per_frame < 0:
            raise ValueError("rays_per_frame must be >= 0")
        if self.mask_distance <= 0:
            raise ValueError("mask_distance must be > 0")
        if not 0.0 <= self.decay_alpha < 1.0:
            raise ValueError("decay_alpha must be in [0, 1)")


@dataclass
class AccumulatorField:
    """Per-texel running state (raysample.py:55-79), resident on the device."""

    min_dist: torch.Tensor  # (fx, fy, fz) float32, +inf sentinel
    front: torch.Tensor     # int32
    back: torch.Tensor      # int32
    mask: torch.Tensor      # bool, current frame
    frames_seen: int = 0

    @classmethod
    def empty(cls, fine_dims):
        fine_dims = tuple(int(n) for n in fine_dims)
        dev = device()
        return cls(min_dist=torch.full(fine_dims, float("inf"), dtype=torch.float32, device=dev),
                   front=torch.zeros(fine_dims, dtype=torch.int32, device=dev),
                   back=torch.zeros(fine_dims, dtype=torch.int32, device=dev),
                   mask=torch.zeros(fine_dims, dtype=torch.bool, device=dev))


def _check_fine_dims(coarse: DistanceField, fine_dims):
    fine_dims = tuple(int(n) for n in fine_dims)
    for f, c in zip(fine_dims, coarse.dims):
        if f % c != 0:
            raise ValueError(
                f"fine dims {fine_dims} must be integer multiples of coarse dims {coarse.dims}")
    return fine_dims


class _RsGeom:
    """Host-side scalars of one coarse -> fine resample (raysample.py:108-119)."""

    def __init__(self, coarse: DistanceField, fine_dims):
        self.coarse = coarse
        self.fine_dims = fine_dims
        self.clo = (_lib.D * 3)(*coarse.lo)
        self.ch = (_lib.D * 3)(*coarse.cell_size)
        self.fh_np = (coarse.hi - coarse.lo) / np.array(fine_dims, dtype=np.float64)
        self.fh = (_lib.D * 3)(*self.fh_np)
        self.n = int(np.prod(fine_dims))
        self.nb = int(_lib.lib().rtsdf_mask_blocks(self.n))

    def desc(self) -> _lib.ResampleDesc:
        c = self.coarse
        return _lib.ResampleDesc(c.data.data_ptr(), *c.dims, (_lib.D * 3)(*c.lo),
                                 (_lib.D * 3)(*c.cell_size), *self.fine_dims,
                                 (_lib.D * 3)(*self.fh_np))


def launch_resample(g: _RsGeom, d, c_fine=None, out_unmasked=None, mask_new=None,
                    block_counts=None, accum: AccumulatorField | None = None):
    c = g.coarse
    _lib.check(_lib.lib().rtsdf_resample_mask(
        _lib.ptr(c.data), *c.dims, g.clo, g.ch, *g.fine_dims, g.fh, float(d),
        _lib.ptr(c_fine), _lib.ptr(out_unmasked), _lib.ptr(mask_new), _lib.ptr(block_counts),
        _lib.ptr(accum.mask if accum else None), _lib.ptr(accum.min_dist if accum else None),
        _lib.ptr(accum.front if accum else None), _lib.ptr(accum.back if accum else None),
        _lib.stream()), "resample_mask")


def _resample_and_mask(coarse: DistanceField, fine_dims, d: float):
    fine_dims = _check_fine_dims(coarse, fine_dims)
    g = _RsGeom(coarse, fine_dims)
    out = torch.empty(fine_dims, dtype=torch.float32, device=coarse.data.device)
    mask = torch.empty(fine_dims, dtype=torch.bool, device=coarse.data.device)
    launch_resample(g, d, c_fine=out, mask_new=mask)
    return out, mask


def coarse_at_fine(coarse: DistanceField, fine_dims) -> torch.Tensor:
    """Trilinear resample of the coarse field at every fine texel centre."""
    return _resample_and_mask(coarse, fine_dims, np.inf)[0]


def ray_mask(coarse: DistanceField, fine_dims, d: float) -> torch.Tensor:
    """Boolean mask of fine texels whose coarse sample is <= d."""
    return _resample_and_mask(coarse, fine_dims, d)[1]


class CompactBuffers:
    """Reusable buffers for mask compaction (idx capacity = all texels)."""

    def __init__(self, n_cells: int, dev=None):
        dev = dev or device()
        L = _lib.lib()
        self.n = n_cells
        self.idx = torch.empty(n_cells, dtype=torch.int64, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.ws = torch.empty(int(L.rtsdf_compact_ws_bytes(n_cells)), dtype=torch.uint8, device=dev)
        self.block_counts = torch.empty(int(L.rtsdf_mask_blocks(n_cells)), dtype=torch.int32,
                                        device=dev)


def launch_compact(mask: torch.Tensor, cb: CompactBuffers, block_counts=True):
    _lib.check(_lib.lib().rtsdf_compact_mask(
        _lib.ptr(mask), cb.n, _lib.ptr(cb.block_counts) if block_counts else None,
        _lib.ptr(cb.idx), _lib.ptr(cb.count), _lib.ptr(cb.ws), cb.ws.numel(), _lib.stream()),
        "compact_mask")


def masked_indices(mask: torch.Tensor) -> torch.Tensor:
    """np.flatnonzero(mask) on the device (ascending int64)."""
    cb = CompactBuffers(mask.numel(), mask.device)
    launch_compact(mask, cb, block_counts=False)
    return cb.idx[: int(cb.count.item())]


_SWS: dict = {}


def sample_workspace(m: int, x: int) -> torch.Tensor:
    """Wavefront-sampler workspace for m texels x x rays (grow-only, per device)."""
    need = int(_lib.lib().rtsdf_sample_ws_bytes(int(max(m, 1)), int(max(x, 1))))
    dev = device()
    ws = _SWS.get(dev.index)
    if ws is None or ws.numel() < need:
        ws = None
        _SWS.pop(dev.index, None)
        ws = torch.empty(int(need * 1.125) + 4096, dtype=torch.uint8, device=dev)
        _SWS[dev.index] = ws
    return ws


def launch_sample_update(bvh: BvhIndex, g: _RsGeom, cb: CompactBuffers, params: SamplingParams,
                         frame: int, t_max: float, dirs=None, samp=None, prev=None,
                         accum: AccumulatorField | None = None, out=None, m_cap=None,
                         frame_dev=None):
    """m_cap: texel capacity; when None the masked count is read back (one
    sync) so the wavefront workspace can be sized to the actual rays."""
    desc = g.desc()
    samp = samp or (None, None, None)
    if m_cap is None:
        m_cap = max(int(cb.count.item()), 1)
    ws = sample_workspace(m_cap, params.rays_per_frame) if params.rays_per_frame > 0 else None
    _lib.check(_lib.lib().rtsdf_sample_update(
        _lib.ptr(bvh.search), bvh.search_nodes, bvh.num_tris, bvh.search_nodes4,
        getattr(bvh, "search_stack4", 0), _lib.ptr(cb.idx),
        _lib.ptr(cb.count),
        int(m_cap), desc, int(params.rays_per_frame),
        int(params.seed) & 0xFFFFFFFFFFFFFFFF, int(frame), _lib.ptr(frame_dev), float(t_max),
        _lib.ptr(dirs),
        _lib.ptr(samp[0]), _lib.ptr(samp[1]), _lib.ptr(samp[2]),
        _lib.ptr(prev), _lib.ptr(accum.mask if accum else None),
        _lib.ptr(accum.min_dist if accum else None), _lib.ptr(accum.front if accum else None),
        _lib.ptr(accum.back if accum else None), float(params.decay_alpha), _lib.ptr(out),
        _lib.ptr(ws), 0 if ws is None else ws.numel(), _lib.stream()), "sample_update")


def sample_texel(bvh: BvhIndex, center, x: int, seed=0, stream=0, frame=0):
    """(min hit distance or None, front hits, back hits) for one texel."""
    if x < 0:
        raise ValueError("x must be >= 0")
    if x == 0:
        return None, 0, 0
    c = np.asarray(center, dtype=np.float64)
    key = _rng.stream_key(seed, np.int64(stream), frame)
    dx, dy, dz = _rng.unit_sphere_dir(key, np.arange(x, dtype=np.uint64))
    dirs = np.stack([dx, dy, dz], axis=-1)
    t, ids, fac = ray_query_many(bvh, np.broadcast_to(c, dirs.shape), dirs, np.inf)
    hit = ids >= 0
    best = float(t[hit].min()) if hit.any() else math.inf
    front = int((fac[hit] == 1).sum())
    return (None if math.isinf(best) else best), front, int(hit.sum()) - front


def resolve_sign(min_dist, front: int, back: int):
    """Negative iff back hits outnumber front hits (raysample.py:197-203)."""
    if min_dist is None:
        return None
    if math.isinf(min_dist):
        return min_dist
    return -min_dist if back > front else min_dist


def accumulate(f_prev: float, c_t: float, r_t, params: SamplingParams) -> float:
    """One Eq. 1 step; r_t None acts as +inf (raysample.py:206-212)."""
    r = math.inf if r_t is None else float(r_t)
    if c_t <= params.mask_distance:
        a = params.decay_alpha
        return min(a * float(f_prev) + (1.0 - a) * float(c_t), r)
    return float(c_t)


def update_fine(prev: DistanceField, coarse: DistanceField, bvh: BvhIndex,
                params: SamplingParams, frame: int, accum: AccumulatorField | None = None,
                directions=None, in_place: bool = False):
    """One frame of fine-field refinement (raysample.py:247-305).

    directions: optional host table (M, x, 3) in masked-texel order (parity
    mode, see rng.direction_table); default = on-device SplitMix64 stream.
    in_place: write the result into prev's buffer (the pipeline's mode).
    """
    fine_dims = _check_fine_dims(coarse, prev.dims)
    if accum is None:
        accum = AccumulatorField.empty(fine_dims)
    if not np.allclose(prev.lo, coarse.lo) or not np.allclose(prev.hi, coarse.hi):
        raise ValueError("prev and coarse fields must share world bounds")
    g = _RsGeom(coarse, fine_dims)
    dev = coarse.data.device
    out = prev.data if in_place else torch.empty(fine_dims, dtype=torch.float32, device=dev)
    mask_new = torch.empty(fine_dims, dtype=torch.bool, device=dev)
    cb = CompactBuffers(g.n, dev)
    launch_resample(g, params.mask_distance, out_unmasked=out, mask_new=mask_new,
                    block_counts=cb.block_counts, accum=accum)
    launch_compact(mask_new, cb)
    t_max = params.t_max
    if t_max is None:
        t_max = float(np.linalg.norm(coarse.hi - coarse.lo))
    dirs = None
    if directions is not None and params.rays_per_frame > 0:
        m = int(cb.count.item())
        dirs = to_device(np.ascontiguousarray(directions, dtype=np.float64))
        if tuple(dirs.shape) != (m, params.rays_per_frame, 3):
            raise ValueError(f"direction table must be ({m}, {params.rays_per_frame}, 3), "
                             f"got {tuple(dirs.shape)}")
    launch_sample_update(bvh, g, cb, params, frame, t_max, dirs=dirs, prev=prev.data,
                         accum=accum, out=out)
    accum.mask = mask_new
    accum.frames_seen += 1
    fine = make_field(out, coarse.lo, coarse.hi, beta=coarse.beta, bias=prev.bias, frame=int(frame))
    return fine, accum


def sample_masked(coarse: DistanceField, fine_dims, bvh: BvhIndex, params: SamplingParams,
                  frame: int, directions=None):
    """Per-masked-texel frame results (idx, min t, front, back) without the
    update -- the reference's _sample_masked_kernel outputs (raysample.py:272-286)."""
    fine_dims = _check_fine_dims(coarse, fine_dims)
    g = _RsGeom(coarse, fine_dims)
    dev = coarse.data.device
    mask = torch.empty(fine_dims, dtype=torch.bool, device=dev)
    cb = CompactBuffers(g.n, dev)
    launch_resample(g, params.mask_distance, mask_new=mask, block_counts=cb.block_counts)
    launch_compact(mask, cb)
    m = int(cb.count.item())
    t_max = params.t_max if params.t_max is not None else float(np.linalg.norm(coarse.hi - coarse.lo))
    smin = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    sf = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    sb = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    dirs = None
    if directions is not None and params.rays_per_frame > 0:
        dirs = to_device(np.ascontiguousarray(directions, dtype=np.float64))
    launch_sample_update(bvh, g, cb, params, frame, t_max, dirs=dirs, samp=(smin, sf, sb),
                         m_cap=max(m, 1))
    return cb.idx[:m], smin[:m], sf[:m], sb[:m]


def fine_from_coarse(coarse: DistanceField, fine_dims) -> DistanceField:
    """Frame-0 initialisation: the coarse field resampled at fine resolution."""
    return make_field(coarse_at_fine(coarse, fine_dims), coarse.lo, coarse.hi,
                      beta=coarse.beta, frame=0)


def masked_count(coarse: DistanceField, fine_dims, d: float) -> int:
    return int(ray_mask(coarse, fine_dims, d).sum().item())


ray_sample_sdf = update_fine

__all__ = ["INF", "SamplingParams", "AccumulatorField", "coarse_at_fine", "ray_mask",
           "sample_texel", "resolve_sign", "accumulate", "update_fine", "ray_sample_sdf",
           "fine_from_coarse", "masked_count", "masked_indices", "sample_masked", "to_numpy"]
