"""z-slab (outer-axis) sharding of the JFA across GPUs -- the north star's
multi-GPU path.

The grid is cut along its OUTERMOST memory axis (axis 0 of the reference's
C-order (nx, ny, nz) layout) into contiguous slabs, one per rank.  A pass at
offset k makes every cell of a slab read planes i - k and i + k; the planes
outside the slab are fetched from their owners before the pass:

    minus side  [x0 - k, min(x0, x0 + nxl - k)) n [0, nx)
    plus side   [max(x0 + nxl, x0 + k), x0 + nxl + k) n [0, nx)

i.e. k planes from each neighbour while k < slab thickness T, and T planes
from the rank(s) k / T away once k >= T.  The per-cell computation is the
single-GPU kernel's (rtsdf_jfa_step_slab), so sharded results are bit
identical to one GPU by construction.  The exchange is NCCL send/recv
(torch.distributed batch_isend_irecv) over NVLink; plan_pass() is pure host
logic and is unit-tested with gloo on the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import jfa as _jfa


def slab_bounds(nx: int, world: int):
    """[(x0, nxl)] per rank: contiguous, sizes differ by at most one plane."""
    base, extra = divmod(nx, world)
    out, x0 = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((x0, n))
        x0 += n
    return out


def owner_of(plane: int, bounds) -> int:
    for r, (x0, n) in enumerate(bounds):
        if x0 <= plane < x0 + n:
            return r
    raise ValueError(f"plane {plane} outside the grid")


def halo_ranges(nx: int, x0: int, nxl: int, k: int):
    """(lo_first, n_lo), (hi_first, n_hi): the foreign planes a slab reads at offset k."""
    lo_a, lo_b = max(x0 - k, 0), min(x0, x0 + nxl - k)
    hi_a, hi_b = max(x0 + nxl, x0 + k), min(x0 + nxl + k, nx)
    return (lo_a, max(lo_b - lo_a, 0)), (hi_a, max(hi_b - hi_a, 0))


@dataclass
class Transfer:
    src: int        # owner rank
    dst: int        # requesting rank
    first: int      # first global plane
    count: int      # number of planes
    side: str       # "lo" or "hi" halo buffer of dst
    offset: int     # plane offset inside dst's halo buffer


def plan_pass(nx: int, bounds, k: int):
    """Every (owner -> requester) plane range for one pass at offset k."""
    plan = []
    for dst, (x0, nxl) in enumerate(bounds):
        for side, (first, count) in zip(("lo", "hi"), halo_ranges(nx, x0, nxl, k)):
            p = first
            while p < first + count:
                src = owner_of(p, bounds)
                s0, sn = bounds[src]
                end = min(first + count, s0 + sn)
                plan.append(Transfer(src, dst, p, end - p, side, p - first))
                p = end
    return plan


def exchange(local: torch.Tensor, halo_lo: torch.Tensor, halo_hi: torch.Tensor, plan, rank: int,
             bounds, group=None):
    """Run this rank's sends/receives of one pass (torch.distributed P2P)."""
    import torch.distributed as dist

    x0 = bounds[rank][0]
    ops = []
    for t in plan:
        if t.src == rank and t.dst != rank:
            ops.append(dist.P2POp(dist.isend, local[t.first - x0: t.first - x0 + t.count].contiguous(),
                                  t.dst, group))
        elif t.dst == rank and t.src != rank:
            buf = halo_lo if t.side == "lo" else halo_hi
            ops.append(dist.P2POp(dist.irecv, buf[t.offset: t.offset + t.count], t.src, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def launch_step_slab(local, halo_lo, halo_hi, dst, nx, x0, k, h, w, lo, hi):
    nxl, ny, nz = local.shape
    ws = _jfa.workspace(nxl, ny, nz)
    _lib.check(_lib.lib().rtsdf_jfa_step_slab(
        _lib.ptr(local), _lib.ptr(halo_lo), _lib.ptr(halo_hi), _lib.ptr(dst), nx, x0, nxl,
        lo[0], lo[1], hi[0], hi[1], ny, nz, int(k), float(h[0]), float(h[1]), float(h[2]), *w,
        _lib.ptr(ws), ws.numel(), _lib.stream()), "jfa_step_slab")


_PLANS: dict = {}


def flood_slab(local: torch.Tensor, nx: int, rank: int, world: int, h, group=None) -> torch.Tensor:
    """Full JFA schedule on this rank's slab (init seeds in `local`, global
    packed coordinates); returns the flooded slab.  Collective: every rank of
    the group must call it with its own slab."""
    bounds = slab_bounds(nx, world)
    x0, nxl = bounds[rank]
    _, ny, nz = local.shape
    dims = (nx, ny, nz)
    w = _jfa.integer_weights(float(h[0]), float(h[1]), float(h[2]), dims)
    max_halo = max(1, max(min(nxl, k) for k in _jfa.jfa_offsets(dims)))
    halo_lo = torch.empty((max_halo, ny, nz), dtype=torch.int32, device=local.device)
    halo_hi = torch.empty_like(halo_lo)
    src, dst = local, torch.empty_like(local)
    for k in _jfa.jfa_offsets(dims):
        key = (nx, world, k)
        plan = _PLANS.get(key)
        if plan is None:  # pure host logic: once per (grid, world, offset)
            plan = _PLANS[key] = plan_pass(nx, bounds, k)
        exchange(src, halo_lo, halo_hi, plan, rank, bounds, group)
        lo, hi = halo_ranges(nx, x0, nxl, k)
        launch_step_slab(src, halo_lo, halo_hi, dst, nx, x0, k, h, w, lo, hi)
        src, dst = dst, src
    return src


def flood_loopback(seed: torch.Tensor, world: int, h) -> torch.Tensor:
    """Emulate `world` slabs on ONE device (sequentially, halos gathered by the
    same plan from the previous pass's full grid) -- covers the slab kernel
    and the plan on a single GPU; every pass is a separate launch per slab, no
    slab kernel waits on another."""
    nx, ny, nz = seed.shape
    bounds = slab_bounds(nx, world)
    dims = (nx, ny, nz)
    w = _jfa.integer_weights(float(h[0]), float(h[1]), float(h[2]), dims)
    cur = seed.clone()
    for k in _jfa.jfa_offsets(dims):
        nxt = torch.empty_like(cur)
        for r, (x0, nxl) in enumerate(bounds):
            lo, hi = halo_ranges(nx, x0, nxl, k)
            halo_lo = cur[lo[0]: lo[0] + lo[1]].contiguous() if lo[1] else cur[:1].clone()
            halo_hi = cur[hi[0]: hi[0] + hi[1]].contiguous() if hi[1] else cur[:1].clone()
            launch_step_slab(cur[x0: x0 + nxl], halo_lo, halo_hi, nxt[x0: x0 + nxl], nx, x0, k,
                             h, w, lo, hi)
        torch.cuda.current_stream().synchronize()
        cur = nxt
    return cur


def halo_volume(nx: int, ny: int, nz: int, world: int):
    """Inbound halo planes / bytes per rank over the whole schedule."""
    bounds = slab_bounds(nx, world)
    planes = np.zeros(world, dtype=np.int64)
    for k in _jfa.jfa_offsets((nx, ny, nz)):
        for r, (x0, nxl) in enumerate(bounds):
            lo, hi = halo_ranges(nx, x0, nxl, k)
            planes[r] += lo[1] + hi[1]
    return planes, planes * ny * nz * 4


__all__ = ["slab_bounds", "owner_of", "halo_ranges", "plan_pass", "exchange", "flood_slab",
           "flood_loopback", "halo_volume", "Transfer"]
