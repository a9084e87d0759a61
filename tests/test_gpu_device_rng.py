"""The benchmarked device-RNG path IS the parity path.

The sampler generates its ray directions on the device (SplitMix64 +
the restatement of the host glibc's cos/sin in csrc/glibc_sincos.cuh).  These
tests pin that path to the reference bit for bit:

  * the device cos/sin == the host libm (the reference's rng.py:53 calls) on
    2^22 direction arguments plus every branch boundary;
  * device directions == the reference's own golden direction table
    (tests/golden/golden.json "rng.dirs", made by sdfshadow.rng);
  * per-texel (min t, front, back) with device directions == the oracle with
    glibc directions (C1 x = 5 / 32, C3 x = 32: 76.7 M rays);
  * whole hybrid_sdf frames with NO host table == the reference's digests
    (C1 x 3 frames; C3 frame 0 + the shaded image), which is exactly the
    workload bench.py times.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from common import C1, C3, digest, golden, golden_arrays, scene_mesh

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    import paper_2210_06160_b200 as rt

    torch.cuda.set_device(0)
    return rt


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _device_sincos(rt, x):
    from paper_2210_06160_b200 import _lib

    xd = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    s, c = torch.empty_like(xd), torch.empty_like(xd)
    _lib.check(_lib.lib().rtsdf_glibc_sincos(_lib.ptr(xd), xd.numel(), _lib.ptr(s), _lib.ptr(c),
                                             _lib.stream()), "glibc_sincos")
    return _np(s), _np(c)


def test_device_sincos_equals_host_libm(rt):
    rng = np.random.default_rng(5)
    k = rng.integers(0, 2**53, size=1 << 22, dtype=np.uint64)
    phi = 6.283185307179586 * (k.astype(np.float64) * (1.0 / 9007199254740992.0))
    m = rng.random(1 << 20)
    e = rng.integers(-40, 27, size=m.size)
    wide = np.ldexp(1.0 + m, e) * np.where(rng.random(m.size) < 0.5, -1.0, 1.0)
    wide = wide[np.abs(wide) < 105414350.0]
    knots = []
    for t in [2.0**-26, 2.0**-27, 0.126, 0.855469, 2.426265, np.pi / 2, np.pi, 2 * np.pi] + \
            [(q + 0.5) / 128 for q in range(110)]:
        v = (np.float64(t).view(np.int64) + np.arange(-512, 512, dtype=np.int64)).view(np.float64)
        knots += [v, -v]
    x = np.concatenate([phi, wide] + knots)
    s, c = _device_sincos(rt, x)
    ws, wc = O.libm_sincos(x)
    np.testing.assert_array_equal(s.view(np.uint64), ws.view(np.uint64))
    np.testing.assert_array_equal(c.view(np.uint64), wc.view(np.uint64))


def test_device_directions_equal_reference_table(rt):
    from paper_2210_06160_b200 import _lib, rng

    g = golden()["rng.dirs"]
    idx = np.asarray(g["idx"], np.int64)
    keys = torch.from_numpy(rng.stream_key(0, idx, g["frame"]).astype(np.uint64).view(np.int64)).cuda()
    out = torch.empty((len(idx), g["x"], 3), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().rtsdf_unit_sphere_dirs(_lib.ptr(keys), len(idx), g["x"], _lib.ptr(out),
                                                 _lib.stream()), "unit_sphere_dirs")
    got = _np(out)
    assert digest(got) == g["digest"]
    np.testing.assert_array_equal(got, golden_arrays()["rng.dirs"])
    # and through the product's public helper
    np.testing.assert_array_equal(rt.rng.device_direction_table(0, idx, g["frame"], g["x"]), got)


@pytest.mark.parametrize("name,dims,x", [("sphere", (64, 64, 64), 5), ("sphere", (64, 64, 64), 32),
                                         ("sphere_plane", (400, 200, 400), 32)])
def test_device_rng_sampling_bit_exact(rt, name, dims, x):
    """sample_masked with on-device directions == the oracle with glibc ones."""
    scene, mesh = scene_mesh(name)
    view = scene.view(0)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    coarse_np = O.seeds_to_sdf(O.jfa_run(occ, h), h)
    coarse = rt.make_field(coarse_np, scene.lo, scene.hi)
    gidx, gmin, gf, gb = rt.sample_masked(coarse, dims, view.bvh, rt.SamplingParams(rays_per_frame=x),
                                          2)
    idx = _np(gidx)
    b = O.bvh_build(mesh.vertices, mesh.triangles, mesh.normals)
    wmin, wf, wb = O.sample_masked(b, idx, scene.lo, h, dims, x, 0, 2,
                                   float(np.linalg.norm(scene.hi - scene.lo)))
    np.testing.assert_array_equal(_np(gf), wf)
    np.testing.assert_array_equal(_np(gb), wb)
    np.testing.assert_array_equal(_np(gmin), wmin)


@pytest.mark.parametrize("case", ["c1", "c3"])
@pytest.mark.parametrize("timing", [True, False])
def test_pipeline_device_rng_frames_golden(rt, case, timing):
    """hybrid_sdf frames exactly as bench.py runs them (device RNG, no host
    table; timing=False also takes the cross-frame flood overlap) == the
    reference's frame digests."""
    G = golden()
    cfg = C1 if case == "c1" else C3
    pc = rt.PipelineConfig(coarse_dims=cfg["dims"], fine_dims=cfg["dims"],
                           sampling=rt.SamplingParams(rays_per_frame=cfg["x"]))
    pipe = rt.FramePipeline(rt.get_scene(cfg["scene"]), pc)
    frames = 3 if case == "c1" else 1
    for f in range(frames):
        rec = pipe.advance(render=(case == "c3"), timing=timing)
        g = G[f"{case}.frame{f}"]
        assert rec.masked_texels == g["masked"]
        assert digest(_np(pipe.coarse.data)) == g["coarse"]
        assert digest(_np(pipe.fine.data)) == g["fine"]
        assert digest(_np(pipe.accum.min_dist)) == g["min_dist"]
        assert digest(_np(pipe.accum.front)) == g["front"]
        assert digest(_np(pipe.accum.back)) == g["back"]
    if case == "c3":
        assert digest(_np(pipe.last_occlusion)) == G["c3.dl"]["occlusion"]
        np.testing.assert_allclose(_np(pipe.last_image), golden_arrays()["c3.image"], rtol=1e-6,
                                   atol=1e-7)


def test_sampler_capacity_tail_exact(rt):
    """Frames whose masked count exceeds the sampler workspace capacity (sized
    without a sync from earlier frames) still equal the reference: the texels
    beyond it go through the workspace-free tail kernel."""
    G = golden()
    pc = rt.PipelineConfig(coarse_dims=C1["dims"], fine_dims=C1["dims"],
                           sampling=rt.SamplingParams(rays_per_frame=C1["x"]))
    pipe = rt.FramePipeline(rt.get_scene(C1["scene"]), pc)
    pipe._sample_capacity = lambda cb: 1000  # far below the 13,012 masked texels
    for f in range(3):
        rec = pipe.advance(render=False, timing=False)
        g = G[f"c1.frame{f}"]
        assert rec.masked_texels == g["masked"] > 1000
        assert digest(_np(pipe.fine.data)) == g["fine"]
        assert digest(_np(pipe.accum.min_dist)) == g["min_dist"]
        assert digest(_np(pipe.accum.front)) == g["front"]
        assert digest(_np(pipe.accum.back)) == g["back"]


@pytest.mark.parametrize("graphs", [False, True])
def test_frame_is_sync_free_after_the_first(rt, monkeypatch, graphs):
    """advance() after the first frames (capacity, graph captures) never blocks
    the host on the device (no .item(), no synchronize): every device->host
    read is replaced by a failing stub."""
    pc = rt.PipelineConfig(coarse_dims=C1["dims"], fine_dims=C1["dims"], cuda_graphs=graphs,
                           sampling=rt.SamplingParams(rays_per_frame=C1["x"]))
    pipe = rt.FramePipeline(rt.get_scene(C1["scene"]), pc)
    for _ in range(4):  # frame 0 (capacity), frames 2 / 3 capture their CUDA graphs
        pipe.advance(render=True, timing=False)
    torch.cuda.synchronize()

    def boom(*a, **k):
        raise AssertionError("host sync inside advance()")

    monkeypatch.setattr(torch.Tensor, "item", boom)
    monkeypatch.setattr(torch.Tensor, "cpu", boom)
    monkeypatch.setattr(torch.cuda, "synchronize", boom)
    monkeypatch.setattr(torch.cuda.Event, "synchronize", boom)
    for _ in range(3):
        pipe.advance(render=True, timing=False)
    monkeypatch.undo()
    assert pipe.records[-1].masked_texels == golden()["c1.frame0"]["masked"]


@pytest.mark.parametrize("case,frames", [("c1", 6), ("c3", 4)])
def test_cuda_graph_frames_bit_identical(rt, case, frames):
    """Frames replayed as CUDA graphs (frame >= 2, static scene) == the eager
    frames: coarse, fine, accumulator, masked count and the shaded image."""
    cfg = C1 if case == "c1" else C3
    outs = []
    for graphs in (False, True):
        pc = rt.PipelineConfig(coarse_dims=cfg["dims"], fine_dims=cfg["dims"], cuda_graphs=graphs,
                               sampling=rt.SamplingParams(rays_per_frame=cfg["x"]))
        pipe = rt.FramePipeline(rt.get_scene(cfg["scene"]), pc)
        seq = []
        for f in range(frames):
            rec = pipe.advance(render=(f % 2 == 1), timing=False)
            pipe.join()
            seq.append((rec.masked_texels, _np(pipe.coarse.data), _np(pipe.fine.data),
                        _np(pipe.accum.min_dist), _np(pipe.accum.front), _np(pipe.accum.back),
                        None if pipe.last_image is None else _np(pipe.last_image)))
        if graphs:
            assert len(pipe._graphs) == 2  # (parity, render) pairs captured once each
        outs.append(seq)
        del pipe
    for a, b in zip(*outs):
        assert a[0] == b[0]
        for x, y in zip(a[1:], b[1:]):
            if x is None:
                assert y is None
            else:
                np.testing.assert_array_equal(x, y)


def test_staged_mesh_uploads_pipelined_frames(rt):
    """upload_mesh(f + 1, ...) before advance(f) (the pipelined e2e input):
    every frame voxelizes its own uploaded mesh, in eager and graph frames,
    with the flood overlap on -- and equals the reference digests (C1)."""
    G = golden()
    scene = rt.get_scene(C1["scene"])
    pc = rt.PipelineConfig(coarse_dims=C1["dims"], fine_dims=C1["dims"],
                           sampling=rt.SamplingParams(rays_per_frame=C1["x"]))
    pipe = rt.FramePipeline(scene, pc)
    mesh = scene.view(0).mesh
    hv = torch.from_numpy(mesh.vertices.copy()).pin_memory()
    ht = torch.from_numpy(mesh.triangles.copy()).pin_memory()
    pipe.upload_mesh(0, hv, ht)
    for f in range(6):
        pipe.upload_mesh(f + 1, hv, ht)
        rec = pipe.advance(render=f % 2 == 1, timing=False)
        if f < 3:
            g = G[f"c1.frame{f}"]
            assert rec.masked_texels == g["masked"]
            assert digest(_np(pipe.fine.data)) == g["fine"], f
    # a staged mesh is really what V reads: a shifted upload changes the field
    bad = hv.clone() * 1.1  # a larger sphere (a whole-cell shift would keep the count)
    pipe.upload_mesh(pipe.frame + 1, bad, ht)
    pipe.advance(timing=False)
    pipe.join()
    rec = pipe.advance(timing=False)
    pipe.join()
    assert rec.masked_texels != G["c1.frame0"]["masked"]


def test_sampler_capacity_headroom_after_a_larger_call(rt):
    """The wavefront workspace is sized for a texel CAPACITY; records beyond the
    actual rays hold whatever an earlier, larger call left there.  A call with
    headroom (m_cap > count) after a larger one must ignore them (the octant
    queue reads only the chunks this call's pass 1 wrote) and still equal the
    oracle bit for bit."""
    from paper_2210_06160_b200 import raysample as RS

    # a larger call first: fills the shared workspace with its chunk records
    big, _ = scene_mesh("sphere_plane")
    dims_big = (128, 128, 128)
    view = big.view(0)
    occ = O.voxelize(view.mesh.vertices, view.mesh.triangles, dims_big, big.bounds)
    hb = (big.hi - big.lo) / np.array(dims_big, dtype=np.float64)
    coarse_b = rt.make_field(O.seeds_to_sdf(O.jfa_run(occ, hb), hb), big.lo, big.hi)
    rt.sample_masked(coarse_b, dims_big, view.bvh, rt.SamplingParams(rays_per_frame=32), 1)
    # then a small one with 3x headroom on the same workspace
    scene, mesh = scene_mesh("sphere")
    dims = (64, 64, 64)
    view = scene.view(0)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    coarse = rt.make_field(O.seeds_to_sdf(O.jfa_run(occ, h), h), scene.lo, scene.hi)
    params = rt.SamplingParams(rays_per_frame=32)
    g = RS._RsGeom(coarse, dims)
    dev = coarse.data.device
    mask = torch.empty(dims, dtype=torch.bool, device=dev)
    cb = RS.CompactBuffers(g.n, dev)
    RS.launch_resample(g, params.mask_distance, mask_new=mask, block_counts=cb.block_counts)
    RS.launch_compact(mask, cb)
    m = int(cb.count.item())
    smin = torch.empty(m, dtype=torch.float64, device=dev)
    sf = torch.empty(m, dtype=torch.int32, device=dev)
    sb = torch.empty(m, dtype=torch.int32, device=dev)
    t_max = float(np.linalg.norm(scene.hi - scene.lo))
    RS.launch_sample_update(view.bvh, g, cb, params, 2, t_max, samp=(smin, sf, sb), m_cap=3 * m)
    idx = cb.idx[:m].cpu().numpy()
    b = O.bvh_build(mesh.vertices, mesh.triangles, mesh.normals)
    wmin, wf, wb = O.sample_masked(b, idx, scene.lo, h, dims, 32, 0, 2, t_max)
    np.testing.assert_array_equal(sf.cpu().numpy(), wf)
    np.testing.assert_array_equal(sb.cpu().numpy(), wb)
    np.testing.assert_array_equal(smin.cpu().numpy(), wmin)
