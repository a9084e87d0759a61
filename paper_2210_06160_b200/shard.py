"""z-slab sharded hybrid frame: every stage of a frame on one
rank's slab of planes [x0, x0 + nxl) of the outermost axis.

    V   voxelize the full grid (mesh replicated; the reference's cell ranges
        are relative to the global lo, so a slab-local voxelizer would change
        the fp64 arithmetic) and keep the slab's packed seeds;
    JF  the slab JFA (slab.flood_slab: per pass, +-k planes from the owners
        over NCCL P2P) + seeds -> SDF on the slab (rtsdf_seeds_to_sdf_range);
    --  one coarse plane from each neighbour (the trilinear resample reads
        coarse planes x0 - 1 .. x0 + nxl);
    RT  resample + mask + band reset, ordered compaction and the ray-sampled
        refine + Eq. 1 on the slab's texels only (mesh + BVH replicated;
        rtsdf_*_range and rtsdf_sample_update with global-indexed slab
        buffers, so texel indices, RNG streams and ray origins are the
        single-GPU ones);
    DL  the fine slabs are all-gathered (every rank holds the whole field),
        each rank shades its band of image rows (G-buffer + soft-shadow
        march; RNG streams stay the global pixel index) and rank 0 gathers
        the occlusion bands and composes the image.

Every per-cell computation is the single-GPU kernel's, so the sharded frame is
bit-identical to FramePipeline by construction (tests: LoopbackCluster runs W
slab ranks on one GPU with the exchanges done by copies).  Coarse and fine
grids must have the same dims (the hybrid config the north star names).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import jfa as _jfa
from . import raysample as _rs
from . import render as _render
from . import slab as _slab
from . import voxel as _voxel
from ._device import device
from .field import DistanceField
from .pipeline import PipelineConfig
from .raymarch import MarchParams
from .scenes import Scene


def _base(t: torch.Tensor, first_cell: int) -> int:
    """Global-indexed base address: base + c * itemsize is global cell c of a
    slab buffer whose element 0 is global cell `first_cell` (include/rtsdf.h,
    slab section)."""
    return t.data_ptr() - first_cell * t.element_size()


class ShardedFramePipeline:
    """One rank's share of FramePipeline (same config, same results)."""

    def __init__(self, scene: Scene, config: PipelineConfig, rank: int, world: int):
        if tuple(config.coarse_dims) != tuple(config.fine_dims):
            raise ValueError("the sharded frame needs coarse_dims == fine_dims")
        self.scene = scene
        self.cfg = config
        self.rank, self.world = rank, world
        self.dims = tuple(int(n) for n in config.coarse_dims)
        nx, ny, nz = self.dims
        self.bounds = _slab.slab_bounds(nx, world)
        self.x0, self.nxl = self.bounds[rank]
        self.plane = ny * nz
        self.c0 = self.x0 * self.plane
        self.n_local = self.nxl * self.plane
        self.frame = 0
        self.h = (scene.hi - scene.lo) / np.array(self.dims, dtype=np.float64)
        dev = device()
        sl = (self.nxl, ny, nz)
        self.seed_full = torch.empty(self.dims, dtype=torch.int32, device=dev)
        self.coarse_h = torch.zeros((self.nxl + 2, ny, nz), dtype=torch.float32, device=dev)
        self.fine = torch.empty(sl, dtype=torch.float32, device=dev)
        self.masks = [torch.zeros(sl, dtype=torch.bool, device=dev) for _ in range(2)]
        self.mask_cur = 0  # masks[mask_cur] = accumulator mask (mask_old)
        self.run_min = torch.full(sl, float("inf"), dtype=torch.float32, device=dev)
        self.front = torch.zeros(sl, dtype=torch.int32, device=dev)
        self.back = torch.zeros(sl, dtype=torch.int32, device=dev)
        self.empty = torch.zeros(1, dtype=torch.int64, device=dev)
        self.cb = _rs.CompactBuffers(max(self.n_local, 1), dev)
        self.started = False
        self.last_image = None
        self._dl = None
        self._gather_buf = None  # rank 0: persistent gather target of the fine slabs
        L = _lib.lib()
        self._clo = (_lib.D * 3)(*scene.lo)
        self._ch = (_lib.D * 3)(*self.h)
        self._nb = int(L.rtsdf_mask_blocks(self.n_local))

    # ------------------------------------------------------------- stages
    def stage_v(self):
        """V on the full grid (mesh replicated); returns this rank's seed slab (a view)."""
        view = self.scene.view(self.frame)
        vox = _voxel.voxelize_seeds(view.mesh, self.dims, (self.scene.lo, self.scene.hi),
                                    check=self.frame == 0, buffers=view.mesh_buffers(),
                                    out=self.seed_full)
        if self.frame == 0 and not vox.any_occupied():
            raise _jfa.NoSeedsError("voxel grid has no occupied cells")
        return self.seed_full[self.x0: self.x0 + self.nxl]

    def stage_sdf(self, seeds_local: torch.Tensor):
        """Seeds -> SDF of the owned planes (coarse_h[1 : nxl + 1])."""
        nx, ny, nz = self.dims
        _lib.check(_lib.lib().rtsdf_seeds_to_sdf_range(
            _lib.C.c_void_p(_base(seeds_local, self.c0)),
            _lib.C.c_void_p(_base(self.coarse_h, self.c0 - self.plane)), nx, ny, nz, self.x0,
            self.nxl, float(self.h[0]), float(self.h[1]), float(self.h[2]), float(self.cfg.beta),
            _lib.ptr(self.empty), _lib.stream()), "seeds_to_sdf_range")

    def coarse_owned(self) -> torch.Tensor:
        return self.coarse_h[1: self.nxl + 1]

    def _coarse_base(self) -> int:
        return _base(self.coarse_h, self.c0 - self.plane)

    def stage_rt(self):
        """Resample + mask + reset, compaction, ray-sampled refine + Eq. 1 on the slab."""
        cfg, s = self.cfg, self.cfg.sampling
        nx, ny, nz = self.dims
        L = _lib.lib()
        C = _lib.C
        fine_b = C.c_void_p(_base(self.fine, self.c0))
        coarse_b = C.c_void_p(self._coarse_base())
        if not self.started:  # frame 0: fine = coarse resampled (pipeline.py:126-131)
            _lib.check(L.rtsdf_resample_mask_range(
                coarse_b, nx, ny, nz, self._clo, self._ch, nx, ny, nz, self._ch, float("inf"),
                self.c0, self.n_local, fine_b, None, None, None, None, None, None, None,
                _lib.stream()), "resample_mask_range")
            self.started = True
        old, new = self.masks[self.mask_cur], self.masks[1 - self.mask_cur]
        acc = [C.c_void_p(_base(t, self.c0)) for t in (old, self.run_min, self.front, self.back)]
        new_b = C.c_void_p(_base(new, self.c0))
        _lib.check(L.rtsdf_resample_mask_range(
            coarse_b, nx, ny, nz, self._clo, self._ch, nx, ny, nz, self._ch,
            float(s.mask_distance), self.c0, self.n_local, None, fine_b, new_b,
            _lib.ptr(self.cb.block_counts), *acc, _lib.stream()), "resample_mask_range")
        cb = self.cb
        _lib.check(L.rtsdf_compact_mask_range(
            new_b, self.c0, self.n_local, _lib.ptr(cb.block_counts), _lib.ptr(cb.idx),
            _lib.ptr(cb.count), _lib.ptr(cb.ws), cb.ws.numel(), _lib.stream()), "compact_mask_range")
        view = self.scene.view(self.frame)
        bvh = view.bvh
        t_max = s.t_max if s.t_max is not None else float(np.linalg.norm(self.scene.hi - self.scene.lo))
        m_cap = max(int(cb.count.item()), 1)
        ws = _rs.sample_workspace(m_cap, s.rays_per_frame) if s.rays_per_frame > 0 else None
        desc = _lib.ResampleDesc(self._coarse_base(), nx, ny, nz, (_lib.D * 3)(*self.scene.lo),
                                 (_lib.D * 3)(*self.h), nx, ny, nz, (_lib.D * 3)(*self.h))
        _lib.check(L.rtsdf_sample_update(
            _lib.ptr(bvh.search), bvh.search_nodes, bvh.num_tris, bvh.search_nodes4,
            getattr(bvh, "search_stack4", 0), _lib.ptr(cb.idx), _lib.ptr(cb.count), m_cap, desc, int(s.rays_per_frame),
            int(s.seed) & 0xFFFFFFFFFFFFFFFF, int(self.frame), None, float(t_max), None, None, None,
            None,
            fine_b, *acc, float(s.decay_alpha), fine_b, _lib.ptr(ws), 0 if ws is None else ws.numel(),
            _lib.stream()), "sample_update")
        self.mask_cur = 1 - self.mask_cur
        return cb.count

    def _dl_state(self, cam):
        if self._dl is None or self._dl["cam"] is not cam:
            gb = _render.GBuffer.empty(cam.height, cam.width)
            dev = gb.position.device
            self._dl = dict(cam=cam, gb=gb, setup=_render.camera_setup(cam),
                            occ=torch.zeros((cam.height, cam.width), dtype=torch.float64, device=dev),
                            img=torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev))
        return self._dl

    def stage_dl_band(self, fine_full: torch.Tensor, rows, camera=None):
        """G-buffer + soft-shadow march of image rows [rows[0], rows[0] + rows[1])
        over the full fine field (pixel-sharded DL); returns the (H, W) occlusion
        buffer, valid on the band."""
        cfg = self.cfg
        cam = camera or self.scene.camera
        view = self.scene.view(self.frame)
        dl = self._dl_state(cam)
        fld = DistanceField(fine_full, np.asarray(self.scene.lo, np.float64),
                            np.asarray(self.scene.hi, np.float64), beta=cfg.beta, frame=self.frame)
        mp = MarchParams.for_field(fld, max_step=cfg.max_step, max_iterations=cfg.max_iterations,
                                   jitter=cfg.jitter, light_angle=self.scene.light.angular_radius)
        _render.launch_gbuffer(view, cam, dl["gb"], dl["setup"])
        _render.launch_occlusion(dl["gb"], fld, self.scene.light.unit(), mp, cfg.shade_draws,
                                 cfg.sampling.seed, dl["occ"], sample_bias=cfg.bias, rows=rows)
        return dl["occ"]

    def stage_compose(self, occ: torch.Tensor, camera=None):
        """Lambert compose of the G-buffer with the full occlusion image."""
        cam = camera or self.scene.camera
        dl = self._dl_state(cam)
        _render.launch_compose(dl["gb"], occ, self.scene.light.unit(), (0.05, 0.07, 0.10), dl["img"])
        self.last_image = dl["img"]
        return dl["img"]

    def stage_dl(self, fine_full: torch.Tensor, camera=None):
        """The whole image on one rank (G-buffer + march + compose)."""
        cam = camera or self.scene.camera
        occ = self.stage_dl_band(fine_full, (0, cam.height), cam)
        return self.stage_compose(occ, cam)

    # ---------------------------------------------------- distributed frame
    def advance(self, render=False, group=None):
        """One frame on this rank (collective over the process group)."""
        import torch.distributed as dist

        seeds = self.stage_v()
        seeds = _slab.flood_slab(seeds, self.dims[0], self.rank, self.world, self.h, group)
        self.stage_sdf(seeds)
        exchange_coarse_halo(self.coarse_h, self.rank, self.world, group)
        count = self.stage_rt()
        img = None
        if render:
            # every rank gets the whole fine field (all-gather over NVLink) and
            # shades its band of image rows; rank 0 gathers the bands and composes
            if self._gather_buf is None:
                nmax = max(n for _, n in self.bounds)
                self._gather_buf = torch.empty((nmax * self.world,) + self.dims[1:],
                                               dtype=self.fine.dtype, device=self.fine.device)
            full = allgather_slabs(self.fine, self.bounds, group, out=self._gather_buf)
            cam = self.scene.camera
            rows = row_bands(cam.height, self.world)[self.rank]
            occ = self.stage_dl_band(full, rows)
            occ_full = gather_rows(occ, row_bands(cam.height, self.world), self.rank, group)
            if self.rank == 0:
                img = self.stage_compose(occ_full)
            # no per-frame barrier: the next frame's collectives order the
            # ranks on the device, and the host may run ahead
        self.frame += 1
        return count, img


def exchange_coarse_halo(coarse_h: torch.Tensor, rank: int, world: int, group=None):
    """Plane x0 - 1 from rank - 1 and plane x0 + nxl from rank + 1 (P2P)."""
    import torch.distributed as dist

    nxl = coarse_h.shape[0] - 2
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, coarse_h[1].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, coarse_h[0], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, coarse_h[nxl].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, coarse_h[nxl + 1], rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def row_bands(height: int, world: int):
    """[(row0, nrows)] per rank: the pixel-sharded DL bands (slab_bounds of rows)."""
    return _slab.slab_bounds(height, world)


def allgather_slabs(local: torch.Tensor, bounds, group=None, out=None):
    """The concatenated slabs on EVERY rank (all-gather, slabs padded to the
    largest); `out`: a persistent (world * nmax, ...) buffer."""
    import torch.distributed as dist

    nmax = max(n for _, n in bounds)
    rest = tuple(local.shape[1:])
    send = local.contiguous()
    if local.shape[0] < nmax:
        send = torch.zeros((nmax,) + rest, dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    if out is None:
        out = torch.empty((nmax * len(bounds),) + rest, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, send, group=group)
    if all(n == nmax for _, n in bounds):
        return out
    return torch.cat([out[r * nmax: r * nmax + n] for r, (_, n) in enumerate(bounds)])


def gather_rows(img: torch.Tensor, bands, rank: int, group=None):
    """Rank 0 receives every rank's band of rows of an (H, W) image (None elsewhere)."""
    import torch.distributed as dist

    r0, n = bands[rank]
    band = img[r0: r0 + n]
    return gather_slabs(band, bands, rank, group)


def gather_slabs(local: torch.Tensor, bounds, rank: int, group=None, out=None):
    """Concatenated slabs on rank 0 (None elsewhere).  Slabs may differ by a
    plane; gather needs equal sizes, so each is padded to the largest.  `out`
    (rank 0, optional): a persistent (world * nmax, ...) buffer received into
    directly -- with equal slabs the result is a view of it, no copy."""
    import torch.distributed as dist

    nmax = max(n for _, n in bounds)
    rest = tuple(local.shape[1:])
    send = local.contiguous()
    if local.shape[0] < nmax:
        send = torch.zeros((nmax,) + rest, dtype=local.dtype, device=local.device)
        send[: local.shape[0]] = local
    if rank == 0:
        if out is None:
            out = torch.empty((nmax * len(bounds),) + rest, dtype=local.dtype, device=local.device)
        parts = [out[r * nmax: (r + 1) * nmax] for r in range(len(bounds))]
        dist.gather(send, parts, dst=0, group=group)
        if all(n == nmax for _, n in bounds):
            return out
        return torch.cat([p[:n] for p, (_, n) in zip(parts, bounds)])
    dist.gather(send, None, dst=0, group=group)
    return None


class LoopbackCluster:
    """W slab ranks in ONE process on one GPU, exchanges done by copies -- the
    single-GPU check that the sharded frame equals FramePipeline bit for bit
    (every slab launch is independent; no kernel waits on another)."""

    def __init__(self, scene: Scene, config: PipelineConfig, world: int):
        self.ranks = [ShardedFramePipeline(scene, config, r, world) for r in range(world)]
        self.world = world
        self.last_image = None

    @property
    def fine(self) -> torch.Tensor:
        return torch.cat([r.fine for r in self.ranks])

    def advance(self, render=False):
        r0 = self.ranks[0]
        for r in self.ranks:
            r.stage_v()
        flooded = _slab.flood_loopback(r0.seed_full, self.world, r0.h)
        for r in self.ranks:
            r.stage_sdf(flooded[r.x0: r.x0 + r.nxl])
        for i, r in enumerate(self.ranks):  # coarse halo planes by copy
            if i > 0:
                r.coarse_h[0].copy_(self.ranks[i - 1].coarse_h[self.ranks[i - 1].nxl])
            if i < self.world - 1:
                r.coarse_h[r.nxl + 1].copy_(self.ranks[i + 1].coarse_h[1])
        counts = [r.stage_rt() for r in self.ranks]
        if render:  # pixel-sharded DL: every rank shades its band, rank 0 composes
            full = self.fine
            cam = r0.scene.camera
            occ = torch.zeros((cam.height, cam.width), dtype=torch.float64, device=full.device)
            for r, (row0, n) in zip(self.ranks, row_bands(cam.height, self.world)):
                band = r.stage_dl_band(full, (row0, n))
                occ[row0: row0 + n] = band[row0: row0 + n]
            self.last_image = r0.stage_compose(occ)
        for r in self.ranks:
            r.frame += 1
        return int(sum(int(c.item()) for c in counts))


__all__ = ["ShardedFramePipeline", "LoopbackCluster", "exchange_coarse_halo", "gather_slabs",
           "allgather_slabs", "gather_rows", "row_bands"]
