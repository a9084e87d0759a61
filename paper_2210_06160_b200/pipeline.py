"""Per-frame hybrid SDF pipeline: voxelize -> jump flood -> ray refine -> deferred light.

Mirrors sdfshadow.pipeline (pipeline.py:1-165): FramePipeline owns the
temporal state (previous fine field + accumulator) and re-runs the coarse
passes every frame.  B200 form: every buffer is allocated once and stays in
HBM; a frame is a fixed sequence of ~35 kernel launches, with the JFA seeds
emitted directly by the voxelizer and the fine field updated in place.  V + JF
depend on the geometry only, so for a static scene frame f + 1's are launched
on a flood stream while frame f's RT / DL run on the caller's stream
(`PipelineConfig.overlap_frames`, auto = while the BVH is far below L2;
double-buffered seeds + coarse field).  Pass durations come from CUDA events,
not the host clock.

`hybrid_sdf(scene, config, frames)` is the north-star entry point.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from . import jfa as _jfa
from . import raysample as _rs
from . import render as _render
from . import voxel as _voxel
from ._device import device, to_device
from .field import DistanceField, apply_bias, make_field
from .raymarch import MarchParams
from .raysample import AccumulatorField, SamplingParams
from .scenes import Scene

PASSES = ("V", "JF", "RT", "DL")


@dataclass(frozen=True)
class PipelineConfig:
    coarse_dims: tuple = (128, 128, 128)
    fine_dims: tuple = (256, 256, 256)
    sampling: SamplingParams = dc_field(default_factory=SamplingParams)
    beta: float = 0.0
    bias: float = 0.01
    max_step: float = 0.05
    max_iterations: int = 256
    jitter: float = 1.0
    shade_draws: int = 1
    repeats: int = 1
    # static scenes: flood frame f+1 (V + JF, which depend on the geometry only)
    # on a second stream while frame f's RT / DL run (B200 form; no effect on
    # any result -- every frame still voxelizes and floods its own seeds).
    # None = auto: on while the tracer's BVH + triangles stay far below L2
    # (the flood's streaming grids would evict them: C4's 180 MB tree ran
    # 112-117 ms/frame overlapped vs 110 serial; C3's 0.2 MB tree 8.70 vs 9.00)
    overlap_frames: bool | None = None
    # static scenes, timing=False: from frame 2 on, replay each frame as one
    # CUDA graph (one per frame parity, render flag and camera); bit-identical
    cuda_graphs: bool = True

    def __post_init__(self):
        for f, c in zip(self.fine_dims, self.coarse_dims):
            if f % c != 0:
                raise ValueError(
                    f"fine dims {self.fine_dims} must be multiples of coarse dims {self.coarse_dims}")


class FrameRecord:
    """frame, durations_ns (pass -> int), masked_texels, rays_traced (pipeline.py:49-58).

    Device-side values are resolved lazily so advance() never has to sync.
    Durations come from CUDA event pairs, `repeats` pairs per pass; like the
    reference's _timed (pipeline.py:61-70) the reported value is
    sorted(times)[len // 2].
    """

    def __init__(self, frame, durations, masked_dev, rays_per_texel, events=None):
        self.frame = frame
        self._durations = durations
        self._events = events  # pass -> [(start, end), ...]
        self._masked_dev = masked_dev
        self._rays = rays_per_texel

    @property
    def durations_ns(self) -> dict:
        if self._events is not None:
            for name, pairs in self._events.items():
                pairs[-1][1].synchronize()
                times = sorted(int(round(a.elapsed_time(b) * 1e6)) for a, b in pairs)
                self._durations[name] = times[len(times) // 2]
            self._events = None
        return self._durations

    @property
    def masked_texels(self) -> int:
        if not isinstance(self._masked_dev, int):
            self._masked_dev = int(self._masked_dev.item())
        return self._masked_dev

    @property
    def rays_traced(self) -> int:
        return self.masked_texels * self._rays

    @property
    def total_ns(self):
        return sum(self.durations_ns.values())


class _Timer:
    """Per-pass CUDA event pairs on the current stream (no host sync)."""

    def __init__(self, on: bool, repeats: int):
        self.on = on
        self.repeats = max(1, int(repeats)) if on else 1
        self.events = {p: [] for p in PASSES} if on else None

    def run(self, name, fn):
        """fn(rep) for rep in range(repeats), each between its own event pair."""
        out = None
        for rep in range(self.repeats):
            if self.on:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
            out = fn(rep)
            if self.on:
                b.record()
                self.events[name].append((a, b))
        return out


class FramePipeline:
    def __init__(self, scene: Scene, config: PipelineConfig):
        self.scene = scene
        self.cfg = config
        self.frame = 0
        self.coarse: DistanceField | None = None
        self.fine: DistanceField | None = None
        self.accum: AccumulatorField | None = None
        self.records: list[FrameRecord] = []
        self.last_image = None
        self.last_occlusion = None
        self._bufs = None
        self._checked_view = None
        self._prefetch = None  # (frame, JF buffer set, event) flooded ahead
        self._jf_ws = None
        self._flood_marked = {}  # id -> tensor already recorded on the flood stream
        self._m_cap = None  # sampler workspace texel capacity (grow-only, _sample_capacity)
        self._frame_dev = None  # graph replays: the RNG frame number on the device
        self._count_host = None
        self._count_pending = None
        # cfg.overlap_frames (None = auto), switchable between frames: off when the caller
        # rewrites the mesh buffers every frame (frame f + 1's V is launched
        # during frame f and would read them one upload early)
        self.overlap_frames = config.overlap_frames
        # parity mode: callable(masked_idx ndarray, frame) -> (M, x, 3) host direction
        # table (the north star's host-supplied table); None = device SplitMix64
        self.direction_fn = None

    # ------------------------------------------------------------- buffers
    def _buffers(self):
        if self._bufs is None:
            cfg = self.cfg
            dev = device()
            cd = tuple(int(n) for n in cfg.coarse_dims)
            fd = tuple(int(n) for n in cfg.fine_dims)
            nf = int(np.prod(fd))
            self._bufs = dict(
                seed_a=torch.empty(cd, dtype=torch.int32, device=dev),
                seed_b=torch.empty(cd, dtype=torch.int32, device=dev),
                coarse=torch.empty(cd, dtype=torch.float32, device=dev),
                mask_a=torch.zeros(fd, dtype=torch.bool, device=dev),
                mask_b=torch.zeros(fd, dtype=torch.bool, device=dev),
                compact=_rs.CompactBuffers(nf, dev),
                masked=torch.zeros(1, dtype=torch.int64, device=dev),
            )
            self._bufs["jf"] = [dict(seed_a=self._bufs["seed_a"], seed_b=self._bufs["seed_b"],
                                     coarse=self._bufs["coarse"]), None]
            # private JFA workspace: the flood stream must not share _jfa's
            n = int(_lib.lib().rtsdf_jfa_ws_bytes(*cd))
            self._jf_ws = torch.empty(n, dtype=torch.uint8, device=dev)
        return self._bufs

    def _jf_set(self, s):
        b = self._buffers()
        if b["jf"][s] is None:
            ref = b["jf"][0]
            b["jf"][s] = {k: torch.empty_like(v) for k, v in ref.items()}
        return b["jf"][s]

    def _dl_buffers(self, cam):
        key = (cam, id(self.scene.view(self.frame)))
        dl = getattr(self, "_dl", None)
        if dl is None or dl["key"] != key:
            gb = _render.GBuffer.empty(cam.height, cam.width)
            dev = gb.position.device
            dl = dict(key=key, gb=gb, cam=_render.camera_setup(cam),
                      occ=torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev),
                      img=torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev))
            self._dl = dl
        return dl

    def march_params(self, **kw) -> MarchParams:
        fine = self.fine if self.fine is not None else self._fine_placeholder()
        kw.setdefault("max_step", self.cfg.max_step)
        kw.setdefault("max_iterations", self.cfg.max_iterations)
        kw.setdefault("jitter", self.cfg.jitter)
        kw.setdefault("light_angle", self.scene.light.angular_radius)
        return MarchParams.for_field(fine, **kw)

    def _fine_placeholder(self):
        return make_field(np.zeros((2, 2, 2), np.float32) + 1.0, self.scene.lo, self.scene.hi)

    @property
    def fine_for_shading(self) -> DistanceField:
        if self.fine is None:
            raise RuntimeError("advance() at least one frame first")
        return apply_bias(self.fine, self.cfg.bias)

    @property
    def coarse_for_shading(self) -> DistanceField:
        if self.coarse is None:
            raise RuntimeError("advance() at least one frame first")
        return apply_bias(self.coarse, self.cfg.bias)

    # --------------------------------------------------------------- frame
    def upload_mesh(self, frame: int, vertices, triangles):
        """Stage frame `frame`'s device mesh (static-topology scenes): copies the
        host arrays (pinned tensors copy asynchronously) into one of two staged
        buffer sets (frame parity) that that frame's V reads instead of the view's
        mesh buffers -- so a caller streaming a new mesh every frame can upload
        frame f + 1 while frame f traces and keep the cross-frame flood overlap.
        Must be called before the call to advance() that floods `frame` (i.e.
        before advance(frame - 1) when the overlap is on)."""
        view = self.scene.view(frame)
        ref = view.mesh_buffers()
        st = self.__dict__.setdefault("_staged", [None, None])
        sf = self.__dict__.setdefault("_staged_frame", [None, None])
        p = frame % 2
        if st[p] is None:
            from .voxel import _MeshBuffers

            st[p] = _MeshBuffers(view.mesh.vertices, view.mesh.triangles)
        v = vertices if isinstance(vertices, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(vertices, dtype=np.float64))
        t = triangles if isinstance(triangles, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(triangles, dtype=np.int32))
        if v.shape != ref.verts.shape or t.shape != ref.tris.shape:
            raise ValueError("upload_mesh: the staged mesh must match the scene's topology")
        st[p].verts.copy_(v, non_blocking=True)
        st[p].tris.copy_(t, non_blocking=True)
        sf[p] = frame

    def _mesh_for(self, view, frame):
        sf = self.__dict__.get("_staged_frame")
        if frame is not None and sf is not None and sf[frame % 2] == frame:
            return self._staged[frame % 2]
        return view.mesh_buffers()

    def _coarse_pass(self, view, s, timer=None, frame=None):
        """V (K1) + JF (K2, K3 fused) of `view` (the staged mesh of `frame` when
        one was uploaded) into JF buffer set s, on the current stream; returns
        the coarse SDF buffer."""
        cfg = self.cfg
        timer = timer or _Timer(False, 1)
        js = self._jf_set(s)
        mb_in = self._mesh_for(view, frame)
        first = self._checked_view is not view

        def vox(rep):
            return _voxel.voxelize_seeds(view.mesh, cfg.coarse_dims, (self.scene.lo, self.scene.hi),
                                         check=first and rep == 0, buffers=mb_in,
                                         out=js["seed_a"])

        vox_res = timer.run("V", vox)
        if first:
            if not vox_res.any_occupied():
                raise _jfa.NoSeedsError("voxel grid has no occupied cells")
            self._checked_view = view

        def flood(rep):
            if rep:  # the flood consumed seed_a: re-voxelize outside the JF timing
                _voxel.voxelize_seeds(view.mesh, cfg.coarse_dims, (self.scene.lo, self.scene.hi),
                                      check=False, buffers=mb_in, out=js["seed_a"])
            return None

        def jf(rep):
            _jfa.flood_to_sdf(js["seed_a"], js["seed_b"], js["coarse"], vox_res.cell_size, cfg.beta,
                              ws=self._jf_ws)

        if timer.repeats > 1:
            for rep in range(timer.repeats):
                flood(rep)
                sub = _Timer(True, 1)
                sub.run("JF", jf)
                timer.events["JF"] += sub.events["JF"]
        else:
            timer.run("JF", jf)
        cur = torch.cuda.current_stream()
        if cur == getattr(self, "_flood", None):
            # buffers allocated on the caller's stream and written here: the
            # allocator must not hand them out again before this work is done
            for t in (*js.values(), self._jf_ws, *vars(mb_in).values()):
                if isinstance(t, torch.Tensor) and id(t) not in self._flood_marked:
                    t.record_stream(cur)
                    self._flood_marked[id(t)] = t
        return js["coarse"]

    def join(self):
        """Make the caller's stream wait for the frame flooded ahead (if any):
        after it, every kernel this pipeline launched precedes what the caller
        queues next -- timing loops end with it so the timed region holds
        exactly one V + JF per frame."""
        if self._prefetch is not None:
            torch.cuda.current_stream().wait_event(self._prefetch[2])

    OVERLAP_MAX_BVH_BYTES = 16 << 20  # << the 126 MB L2

    def _overlap_for(self, view) -> bool:
        if self.overlap_frames is not None:
            return bool(self.overlap_frames)
        bvh = view.bvh
        return bvh.search.numel() * bvh.search.element_size() <= self.OVERLAP_MAX_BVH_BYTES

    def _flood_ahead(self, frame):
        """Launch V + JF of `frame` on the flood stream.  It waits for
        everything already queued on the main stream -- frame - 2's RT read the
        buffer set it overwrites -- but not for this frame's RT, which is
        queued after it and overlaps it."""
        flood = self._flood_stream()
        flood.wait_stream(torch.cuda.current_stream())
        view = self.scene.view(frame)
        view.mesh_buffers()  # allocated on the caller's stream (see _coarse_pass)
        self._jf_set(frame % 2)
        with torch.cuda.stream(flood):
            self._coarse_pass(view, frame % 2, frame=frame)
            ev = torch.cuda.Event()
            ev.record(flood)
        self._prefetch = (frame, frame % 2, ev)

    def _flood_stream(self):
        st = getattr(self, "_flood", None)
        if st is None or st.device != torch.cuda.current_stream().device:
            st = self._flood = torch.cuda.Stream()  # default priority (measured: a high-priority
            # flood stream 8.81 vs 8.62 ms/frame, a high-priority RT stream 8.63; unjoined timing)
        return st

    def _side_stream(self):
        st = getattr(self, "_side", None)
        if st is None or st.device != torch.cuda.current_stream().device:
            st = self._side = torch.cuda.Stream()
        return st

    def _sample_capacity(self, cb) -> int:
        """Texel capacity of the sampler workspace, grow-only and sync-free after
        the first frame: the masked count of earlier frames is copied to pinned
        host memory asynchronously and read only once its event has completed
        (never waited on).  Texels beyond the capacity are still sampled, by the
        workspace-free tail kernel (rtsdf_sample_update), so the capacity only
        steers speed, never the result."""
        if self._m_cap is None:  # frame 0: one sync; 25 % headroom (<= every cell)
            self._m_cap = min(int(max(int(cb.count.item()), 1) * 1.25) + 1, cb.n)
            return self._m_cap
        pend = self._count_pending
        if pend is not None and pend[1].query():
            seen = int(pend[0][0])
            if seen > self._m_cap:  # that frame ran texels through the tail kernel
                self._m_cap = min(int(seen * 1.25) + 1, cb.n)
            self._count_pending = None
        return self._m_cap

    def _note_count(self, cb):
        if self._count_pending is None:
            if self._count_host is None:
                self._count_host = torch.empty(1, dtype=torch.int64).pin_memory()
            self._count_host.copy_(cb.count, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._count_pending = (self._count_host, ev)

    def _rt_pass(self, view, frame, b, frame_dev=None):
        """RT: resample + mask + band reset (K4), compaction, fused sample + Eq. 1
        (K6/K7); returns the new mask buffer.  frame_dev: the frame number as a
        device scalar (graph replays)."""
        cfg = self.cfg
        g = _rs._RsGeom(self.coarse, tuple(cfg.fine_dims))
        mask_new = b["mask_b"] if self.accum.mask is b["mask_a"] else b["mask_a"]
        cb = b["compact"]
        _rs.launch_resample(g, cfg.sampling.mask_distance, out_unmasked=self.fine.data,
                            mask_new=mask_new, block_counts=cb.block_counts, accum=self.accum)
        _rs.launch_compact(mask_new, cb)
        t_max = cfg.sampling.t_max
        if t_max is None:
            t_max = float(np.linalg.norm(self.coarse.hi - self.coarse.lo))
        dirs = None
        m_cap = None
        if self.direction_fn is not None and cfg.sampling.rays_per_frame > 0:
            m = int(cb.count.item())  # parity mode: the host table needs the texel list
            idx = cb.idx[:m].cpu().numpy()
            dirs = to_device(np.ascontiguousarray(self.direction_fn(idx, frame), dtype=np.float64))
            m_cap = max(m, 1)
        elif cfg.sampling.rays_per_frame > 0:
            m_cap = self._m_cap if frame_dev is not None else self._sample_capacity(cb)
        _rs.launch_sample_update(view.bvh, g, cb, cfg.sampling, frame, t_max, dirs=dirs,
                                 prev=self.fine.data, accum=self.accum, out=self.fine.data,
                                 m_cap=m_cap if m_cap is not None else 1, frame_dev=frame_dev)
        if frame_dev is None:
            self._note_count(cb)
        return mask_new

    def advance(self, render=False, camera=None, timing=True) -> FrameRecord:
        """Run one frame of V -> JF -> RT (-> DL when render=True).

        No host synchronisation after the first frame (parity mode's host
        direction table aside).  timing=True records per-pass CUDA events,
        `cfg.repeats` times per pass (median, as pipeline.py:61-70); RT repeats
        run on a restored copy of the temporal state, so the result is that of
        one frame."""
        cfg = self.cfg
        frame = self.frame
        view = self.scene.view(frame)
        b = self._buffers()
        lo, hi = self.scene.lo, self.scene.hi
        if self._graph_ok(view, timing):
            return self._advance_graphed(view, render, camera)
        self._graph_flooded = False
        timer = _Timer(timing, cfg.repeats)

        # DL's G-buffer depends only on mesh + camera: it runs on a side stream
        # while V / JF / RT occupy the main one (joined before the march)
        gb_done = None
        if render:
            cam = camera or self.scene.camera
            dl = self._dl_buffers(cam)
            main = torch.cuda.current_stream()
            side = self._side_stream()
            side.wait_stream(main)  # the previous frame's march has read dl["gb"]
            with torch.cuda.stream(side):
                _render.launch_gbuffer(view, cam, dl["gb"], dl["cam"])
                gb_done = torch.cuda.Event()
                gb_done.record(side)

        # V + JF: packed self-seeds straight from the triangles (K1), full
        # schedule (K2) + seeds -> SDF (K3).  Static scenes with overlap_frames
        # run them on the flood stream one frame ahead (see _flood_ahead).
        overlap = not timing and not self.scene.animated and self._overlap_for(view)
        pre = self._prefetch
        self._prefetch = None
        main = torch.cuda.current_stream()
        if pre is not None:
            main.wait_event(pre[2])  # its buffers are written on the flood stream
        if overlap and pre is not None and pre[0] == frame:
            coarse_buf = self._jf_set(pre[1])["coarse"]
        elif overlap:
            # buffers of the first overlapped frame are allocated on the caller's
            # stream before the flood stream touches them (see _coarse_pass)
            view.mesh_buffers()
            flood = self._flood_stream()
            flood.wait_stream(main)
            self._jf_set(frame % 2)
            with torch.cuda.stream(flood):
                self._coarse_pass(view, frame % 2, frame=frame)
                ev = torch.cuda.Event()
                ev.record(flood)
            main.wait_event(ev)
            coarse_buf = self._jf_set(frame % 2)["coarse"]
        else:
            coarse_buf = self._coarse_pass(view, 0, timer, frame=frame)
        self.coarse = DistanceField(coarse_buf, np.asarray(lo, np.float64), np.asarray(hi, np.float64),
                                    beta=cfg.beta)
        if overlap:
            self._flood_ahead(frame + 1)
        if self.fine is None:
            self.fine = _rs.fine_from_coarse(self.coarse, cfg.fine_dims)
            self.accum = AccumulatorField.empty(cfg.fine_dims)
            self.accum.mask = b["mask_a"]

        state = None
        if timer.repeats > 1:  # pipeline.py:131: every repeat starts from the same state
            acc = self.accum
            state = [t.clone() for t in (self.fine.data, acc.min_dist, acc.front, acc.back)]

        def rt(rep):
            if rep:
                for dst, src in zip((self.fine.data, self.accum.min_dist, self.accum.front,
                                     self.accum.back), state):
                    dst.copy_(src)
            return self._rt_pass(view, frame, b)

        mask_new = timer.run("RT", rt)
        self.accum.mask = mask_new
        self.accum.frames_seen += 1
        self.fine = DistanceField(self.fine.data, self.coarse.lo, self.coarse.hi,
                                  beta=self.coarse.beta, bias=self.fine.bias, frame=frame)
        masked = b["compact"].count.clone()

        self.last_image = None
        if render:
            # DL: G-buffer (K6 traversal) -> soft-shadow march (K8, fine_for_shading's
            # bias fused into the samples) -> compose; buffers persist per camera
            torch.cuda.current_stream().wait_event(gb_done)
            light = self.scene.light.unit()

            def dlp(rep):
                _render.launch_occlusion(dl["gb"], self.fine, light, self.march_params(),
                                         cfg.shade_draws, cfg.sampling.seed, dl["occ"],
                                         sample_bias=cfg.bias)
                _render.launch_compose(dl["gb"], dl["occ"], light, (0.05, 0.07, 0.10), dl["img"])

            timer.run("DL", dlp)
            self.last_occlusion = dl["occ"]
            self.last_image = dl["img"]

        rec = FrameRecord(frame, {p: 0 for p in PASSES}, masked, cfg.sampling.rays_per_frame,
                          {k: v for k, v in timer.events.items() if v} if timing else None)
        self.records.append(rec)
        self.frame += 1
        return rec

    # ------------------------------------------------------------ CUDA graphs
    def _graph_ok(self, view, timing) -> bool:
        cfg = self.cfg
        # a view not validated yet (first frame of a new SceneView) runs eagerly:
        # its voxelization checks read back
        return (cfg.cuda_graphs and not timing and not self.scene.animated and self.frame >= 2
                and self.direction_fn is None and cfg.sampling.rays_per_frame > 0
                and self._m_cap is not None and self._checked_view is view)

    def _advance_graphed(self, view, render, camera) -> FrameRecord:
        """One frame as a CUDA-graph replay.  Graph (parity p = frame % 2, render,
        camera, overlap): [G-buffer on the side stream] || [with overlap: V + JF of
        frame + 1 into JF set 1 - p on the flood stream] || [RT of the frame from
        JF set p (without overlap: V + JF first), DL], all joined at the end.  The
        RNG frame number is a device scalar written before each replay; every
        buffer is the one the eager frame of the same parity would use, so the
        replay is the eager frame bit for bit."""
        cfg = self.cfg
        frame = self.frame
        p = frame % 2
        b = self._buffers()
        cam = (camera or self.scene.camera) if render else None
        overlap = self._overlap_for(view)
        main = torch.cuda.current_stream()
        if self._prefetch is not None:  # the eager frame before flooded this one
            main.wait_event(self._prefetch[2])
            pre_set = self._prefetch[1]
            self._prefetch = None
        else:
            pre_set = None
        if overlap and pre_set is None and not getattr(self, "_graph_flooded", False):
            # the previous frame did not flood this one (e.g. it was serial):
            # flood set p eagerly once
            self._jf_set(p)
            self._coarse_pass(view, p, frame=frame)
        if self._frame_dev is None:
            self._frame_dev = torch.zeros(1, dtype=torch.int64, device=b["masked"].device)
        if render:
            dl = self._dl_buffers(cam)
        for s_ in (0, 1):
            self._jf_set(s_)
        view.mesh_buffers()  # every buffer the graph touches exists before the capture
        m_cap = self._m_cap
        _rs.sample_workspace(m_cap, cfg.sampling.rays_per_frame)  # no growth inside a capture
        # the view is part of the key: a graph references its mesh / BVH buffers
        staged = self._mesh_for(view, frame + 1) is not view.mesh_buffers() if overlap else \
            self._mesh_for(view, frame) is not view.mesh_buffers()
        key = (p, bool(render), cam, overlap, m_cap, id(view), staged)
        graphs = self.__dict__.setdefault("_graphs", {})
        self._frame_dev.fill_(frame)
        mask_old = b["mask_a"] if p == 0 else b["mask_b"]  # eager: frame f reads mask (f - 1) % 2
        mask_new = b["mask_b"] if p == 0 else b["mask_a"]
        if self.accum.mask is not mask_old:
            raise RuntimeError("graph replay out of step with the temporal state")
        coarse_buf = self._jf_set(p)["coarse"] if overlap else b["jf"][0]["coarse"]
        self.coarse = DistanceField(coarse_buf, np.asarray(self.scene.lo, np.float64),
                                    np.asarray(self.scene.hi, np.float64), beta=cfg.beta)
        entry = graphs.get(key)
        if entry is None:
            g = torch.cuda.CUDAGraph()
            cap_stream = self.__dict__.setdefault("_cap_stream", torch.cuda.Stream())
            n0 = _lib.launch_count()
            with torch.cuda.graph(g, stream=cap_stream):
                self._graph_body(view, frame, p, render, cam, overlap, b, staged)
            while len(graphs) >= 8:  # drop the oldest graph (and its view's buffers)
                graphs.pop(next(iter(graphs)))
            entry = graphs[key] = (g, _lib.launch_count() - n0, view)
        else:
            _lib.lib().rtsdf_count_launches(entry[1])
        entry[0].replay()
        self._graph_flooded = overlap
        self.accum.mask = mask_new
        self.accum.frames_seen += 1
        self.fine = DistanceField(self.fine.data, self.coarse.lo, self.coarse.hi,
                                  beta=self.coarse.beta, bias=self.fine.bias, frame=frame)
        self.last_image = None
        if render:
            self.last_occlusion = dl["occ"]
            self.last_image = dl["img"]
        rec = FrameRecord(frame, {q: 0 for q in PASSES}, b["compact"].count.clone(),
                          cfg.sampling.rays_per_frame, None)
        self.records.append(rec)
        self.frame += 1
        return rec

    def _graph_body(self, view, frame, p, render, cam, overlap, b, staged=False):
        """The launches of one graph-mode frame (captured once per key)."""
        cfg = self.cfg
        main = torch.cuda.current_stream()
        gb_done = None
        if render:
            dl = self._dl_buffers(cam)
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                _render.launch_gbuffer(view, cam, dl["gb"], dl["cam"])
                gb_done = torch.cuda.Event()
                gb_done.record(side)
        flood_done = None
        if overlap:
            flood = self._flood_stream()
            flood.wait_stream(main)
            with torch.cuda.stream(flood):
                # V + JF of frame + 1 (static scene; its staged upload when `staged`)
                self._coarse_pass(view, 1 - p, frame=frame + 1 if staged else None)
                flood_done = torch.cuda.Event()
                flood_done.record(flood)
        else:
            self._coarse_pass(view, 0, frame=frame if staged else None)
        self._rt_pass(view, frame, b, frame_dev=self._frame_dev)
        if render:
            main.wait_event(gb_done)
            light = self.scene.light.unit()
            _render.launch_occlusion(dl["gb"], self.fine, light, self.march_params(),
                                     cfg.shade_draws, cfg.sampling.seed, dl["occ"],
                                     sample_bias=cfg.bias)
            _render.launch_compose(dl["gb"], dl["occ"], light, (0.05, 0.07, 0.10), dl["img"])
        if flood_done is not None:
            main.wait_event(flood_done)

    def run(self, frames: int, render_last=False, camera=None):
        for i in range(frames):
            self.advance(render=render_last and i == frames - 1, camera=camera)
        return self.records


def hybrid_sdf(scene: Scene, config: PipelineConfig, frames: int = 1, render_last=False):
    """North-star entry point: run `frames` hybrid-SDF frames, return the pipeline."""
    pipe = FramePipeline(scene, config)
    pipe.run(frames, render_last=render_last)
    return pipe


__all__ = ["PASSES", "PipelineConfig", "FrameRecord", "FramePipeline", "hybrid_sdf"]
