"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle and the
reference's golden digests.  Integer/index/mask outputs must be bit-exact;
fp32 fields are compared bit-exact too (same fp64 arithmetic, no FMA) and the
north-star tolerance (1e-5 relative) is asserted on top as the floor."""

import math
import sys
from pathlib import Path

import numpy as np
import pytest

from common import C1, C3, digest, golden, golden_arrays, scene_mesh

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # north star: distances within 1e-5 relative


def _np(t):
    return t.detach().cpu().numpy()


def _assert_close_f32(a, b):
    """Bit-exact expected; the 1e-5 relative tolerance is the contract floor."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    fin = np.isfinite(b)
    assert np.array_equal(np.isfinite(a), fin)
    np.testing.assert_allclose(a[fin], b[fin], rtol=REL_TOL, atol=1e-6)


@pytest.fixture(scope="module")
def rt():
    import paper_2210_06160_b200 as rt

    return rt


# ---------------------------------------------------------------- voxelize
def test_voxelize_closed_box_square(rt):
    verts = np.array([[0, 0.5, 0], [4, 0.5, 0], [4, 0.5, 4], [0, 0.5, 4]], np.float64)
    tris = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    vg = rt.voxelize((verts, tris), (8, 8, 8), (np.zeros(3), np.full(3, 8.0)))
    assert vg.count == 25
    np.testing.assert_array_equal(_np(vg.occupancy), golden_arrays()["voxel_square.occ"])


def test_voxelize_errors(rt):
    verts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [5, 5, 5]], np.float64)
    tris = np.array([[0, 1, 2], [1, 2, 3]], np.int32)
    with pytest.raises(rt.OutOfBoundsError) as ei:
        rt.voxelize((verts, tris), (4, 4, 4), (np.zeros(3), np.full(3, 2.0)))
    assert ei.value.triangle_ids == [1]
    with pytest.raises(rt.VoxelizeError):
        rt.voxelize((verts, tris), (1, 4, 4), (np.zeros(3), np.full(3, 8.0)))
    with pytest.raises(rt.VoxelizeError):
        rt.voxelize((verts, tris), (4, 4, 4), (np.zeros(3), np.zeros(3)))


@pytest.mark.parametrize("name,dims", [("sphere", (64, 64, 64)), ("sphere_plane", (64, 64, 64)),
                                       ("sphere_plane", (128, 128, 128)),
                                       ("sphere_plane", (256, 256, 256)),
                                       ("sphere_plane", (400, 200, 400)),
                                       ("thin_plate", (96, 80, 112))])
def test_voxelize_matches_oracle(rt, name, dims):
    """Includes the 1-ulp boundary-plane cases (Appendix A.2: 0 ground cells at 256^3)."""
    scene, mesh = scene_mesh(name)
    want = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    vg = rt.voxelize(mesh, dims, scene.bounds)
    np.testing.assert_array_equal(_np(vg.occupancy), want)
    # fused seed form == jfa_init(occupancy)
    vs = rt.voxelize_seeds(mesh, dims, scene.bounds)
    lin = _np(rt.jfa.SeedGrid(vs.seed_packed, vs.lo, vs.hi).seed)
    np.testing.assert_array_equal(lin, O.jfa_init(want))


def test_voxelize_golden_counts(rt):
    G = golden()
    scene, mesh = scene_mesh("sphere_plane")
    assert rt.voxelize(mesh, (400, 200, 400), scene.bounds).count == G["c3.voxel"]["count"]
    assert rt.voxelize(mesh, (128,) * 3, scene.bounds).count == G["sp128"]["count"]


# --------------------------------------------------------------------- JFA
def test_jfa_tie_rule_fp64(rt):
    occ = np.zeros((16, 16, 16), np.uint8)
    occ[0, 3, 4] = 1
    occ[5, 0, 0] = 1
    vg = rt.VoxelGrid(rt._device.to_device(occ) if hasattr(rt, "_device") else occ,
                      np.zeros(3), np.full(3, 1.6))
    seeds = rt.jfa_run(vg)
    got = _np(seeds.seed)
    assert got[0, 0, 0] == 5 * 256
    np.testing.assert_array_equal(got, golden_arrays()["jfa_tie.seed"])
    np.testing.assert_array_equal(_np(rt.seeds_to_sdf(seeds).data), golden_arrays()["jfa_tie.sdf"])


def test_jfa_fp64_general_path(rt):
    """Non-rational spacing ratios take the fp64 comparison path."""
    G, A = golden(), golden_arrays()
    mesh = rt.make_mesh(A["soup.vertices"], A["soup.triangles"])
    vg = rt.voxelize(mesh, (40, 33, 27), (np.zeros(3), np.ones(3)))
    assert rt.jfa.integer_weights(*map(float, vg.cell_size), (40, 33, 27)) == (0, 0, 0)
    seeds = rt.jfa_run(vg)
    assert digest(_np(seeds.seed)) == G["soup.jfa"]["seed"]
    assert digest(_np(rt.seeds_to_sdf(seeds, beta=0.01).data)) == G["soup.sdf"]["data"]


@pytest.mark.parametrize("name,dims", [("sphere", (64, 64, 64)), ("sphere_plane", (128, 128, 128)),
                                       ("sphere_plane", (400, 200, 400))])
def test_jfa_every_pass_matches_oracle(rt, name, dims):
    scene, mesh = scene_mesh(name)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    ref = O.jfa_init(occ)
    vg = rt.voxelize(mesh, dims, scene.bounds)
    cur = rt.jfa_init(vg)
    for off in rt.jfa_offsets(dims):
        ref = O.jfa_step(ref, off, h)
        cur = rt.jfa_step(cur, off)
        np.testing.assert_array_equal(_np(cur.seed), ref, err_msg=f"offset {off}")
    np.testing.assert_array_equal(_np(rt.seeds_to_sdf(cur).data), O.seeds_to_sdf(ref, h))


@pytest.mark.parametrize("dims,hi,frac,weights", [
    # weights 1:9:16 over 1000-cell axes: the packed EMPTY's virtual seed is
    # NOT provably the farthest (jfa.cu natural_empty_ok false -> select path)
    ((8, 1000, 1000), (0.064, 24.0, 32.0), 2e-4, (1, 9, 16)),
    # C3's 1:4:1 weights on a random dense-ish soup: many integer ties
    ((64, 48, 80), (0.512, 0.768, 0.64), 0.01, (1, 4, 1)),
    # dyadic spacing 1/128: fp64 d2 exact -> EXACT mode (64-bit lexicographic test)
    ((64, 48, 80), (0.5, 0.375, 0.625), 0.01, (1, 1, 1)),
    # ragged grids for v5's 2 x 2 register tiles (jfa5.cuh): chains shorter than a
    # tile, odd extents, offsets beyond an axis -- every clamped tap and masked output
    ((37, 23, 51), (0.37, 0.46, 0.51), 0.02, (1, 4, 1)),
    ((5, 70, 3), (0.05, 1.4, 0.03), 0.05, (1, 4, 1)),
    ((3, 41, 66), (0.096, 1.312, 2.112), 0.03, (1, 1, 1)),
    # axes beyond 1024 cells: dims-dependent packed seeds, per-cell kernel
    ((2100, 6, 10), (2.1, 0.012, 0.01), 0.002, (1, 4, 1)),
    ((20, 1500, 12), (0.02, 3.0, 0.012), 0.002, (1, 4, 1)),
    ((3, 40, 1100), (0.375, 5.0, 137.5), 0.003, (1, 1, 1)),
    ((1030, 9, 5), (1.03, 0.0045, 0.0155), 0.004, (0, 0, 0)),
])
def test_jfa_random_occupancy_every_pass_and_schedule(rt, dims, hi, frac, weights):
    """Random seeds, non-dyadic spacings (INT mode with tie marks + fix-ups):
    every pass and the whole schedule (sparse early passes) == the oracle."""
    rng = np.random.default_rng(7)
    occ = (rng.random(dims) < frac).astype(np.uint8)
    lo, hi = np.zeros(3), np.array(hi, dtype=np.float64)
    h = (hi - lo) / np.array(dims, dtype=np.float64)
    assert rt.jfa.integer_weights(*map(float, h), dims) == weights
    vg = rt.VoxelGrid(rt._device.to_device(occ), lo, hi)
    ref = O.jfa_init(occ)
    cur = rt.jfa_init(vg)
    for off in rt.jfa_offsets(dims):
        ref = O.jfa_step(ref, off, h)
        cur = rt.jfa_step(cur, off)
        np.testing.assert_array_equal(_np(cur.seed), ref, err_msg=f"offset {off}")
    np.testing.assert_array_equal(_np(rt.jfa_run(vg).seed), ref)
    np.testing.assert_array_equal(_np(rt.jump_flood(vg).data), O.seeds_to_sdf(ref, h))


def test_jfa_golden_c3_and_sp128(rt):
    G = golden()
    scene, mesh = scene_mesh("sphere_plane")
    for dims, key, ck in (((400, 200, 400), "c3.jfa", "c3.frame0"), ((128,) * 3, "sp128", "sp128")):
        seeds = rt.jfa_run(rt.voxelize(mesh, dims, scene.bounds))
        assert digest(_np(seeds.seed)) == G[key]["seed"]
        assert digest(_np(rt.seeds_to_sdf(seeds).data)) == G[ck]["coarse"]


@pytest.mark.parametrize("name,dims,beta", [("sphere", (64, 64, 64), 0.0),
                                            ("sphere_plane", (400, 200, 400), 0.0),
                                            ("sphere_plane", (128, 96, 80), 0.02),
                                            ("thin_plate", (96, 80, 112), 0.0)])
def test_jump_flood_fused_sdf(rt, name, dims, beta):
    """jump_flood (last pass writes the SDF) == jfa_run + seeds_to_sdf on the oracle."""
    scene, mesh = scene_mesh(name)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    want = O.seeds_to_sdf(O.jfa_run(occ, h), h, beta)
    got = rt.jump_flood(rt.voxelize(mesh, dims, scene.bounds), beta=beta)
    np.testing.assert_array_equal(_np(got.data), want)


def test_jfa_errors(rt):
    occ = np.zeros((8, 8, 8), np.uint8)
    vg = rt.VoxelGrid(rt._device.to_device(occ), np.zeros(3), np.ones(3))
    with pytest.raises(rt.NoSeedsError):
        rt.jfa_init(vg)
    occ[1, 2, 3] = 1
    seeds = rt.jfa_init(rt.VoxelGrid(rt._device.to_device(occ), np.zeros(3), np.ones(3)))
    with pytest.raises(ValueError):
        rt.jfa_step(seeds, 5)
    with pytest.raises(rt.NoSeedsError):
        rt.seeds_to_sdf(seeds)  # incomplete: not flooded
    with pytest.raises(ValueError):
        rt.seeds_to_sdf(seeds, beta=-1)


def test_jfa_single_seed_exact_and_upper_bound(rt):
    """SPEC invariants: single seed -> exact everywhere; JFA never underestimates."""
    occ = np.zeros((48, 40, 36), np.uint8)
    occ[7, 30, 11] = 1
    vg = rt.VoxelGrid(rt._device.to_device(occ), np.zeros(3), np.array([1.2, 1.0, 0.9]))
    seeds = rt.jfa_run(vg)
    assert (_np(seeds.seed) == 7 * 40 * 36 + 30 * 36 + 11).all()
    rng = np.random.default_rng(5)
    occ = (rng.random((32, 32, 32)) < 0.0015).astype(np.uint8)
    vg = rt.VoxelGrid(rt._device.to_device(occ), np.zeros(3), np.ones(3))
    sdf = _np(rt.seeds_to_sdf(rt.jfa_run(vg)).data).astype(np.float64)
    pts = np.argwhere(occ > 0)
    grid = np.stack(np.meshgrid(*[np.arange(32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    exact = np.sqrt(((grid[:, None, :] - pts[None]) ** 2).sum(-1).min(1)) / 32.0
    assert (sdf.reshape(-1) >= exact - 1e-6).all()
    assert (np.abs(sdf.reshape(-1) - exact) < 1e-6).mean() >= 0.99


# ---------------------------------------------------- resample / mask / BVH
@pytest.mark.parametrize("coarse_dims,fine_dims", [((128,) * 3, (128,) * 3), ((64,) * 3, (128,) * 3),
                                                   ((200, 100, 200), (400, 200, 400))])
def test_resample_mask_compaction(rt, coarse_dims, fine_dims):
    scene, mesh = scene_mesh("sphere_plane")
    occ = O.voxelize(mesh.vertices, mesh.triangles, coarse_dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(coarse_dims, dtype=np.float64)
    coarse_np = O.seeds_to_sdf(O.jfa_run(occ, h), h)
    want_f, want_m = O.resample_mask(coarse_np, scene.lo, scene.hi, fine_dims, 0.1)
    coarse = rt.make_field(coarse_np, scene.lo, scene.hi)
    np.testing.assert_array_equal(_np(rt.coarse_at_fine(coarse, fine_dims)), want_f)
    m = rt.ray_mask(coarse, fine_dims, 0.1)
    np.testing.assert_array_equal(_np(m), want_m)
    idx = rt.raysample.masked_indices(m)
    np.testing.assert_array_equal(_np(idx), np.flatnonzero(want_m.ravel()))


def test_compaction_random_odd_sizes_and_ranges(rt):
    """Ordered compaction == np.flatnonzero on random masks of odd sizes, and
    the range form (global cell addressing, unaligned c0) == the slice."""
    import torch
    from paper_2210_06160_b200 import _lib

    rng = np.random.default_rng(5)
    for n in (1, 15, 17, 4095, 4097, 100003):
        m = rng.random(n) < 0.3
        got = _np(rt.raysample.masked_indices(torch.from_numpy(m).cuda()))
        np.testing.assert_array_equal(got, np.flatnonzero(m))
    m = rng.random(200_000) < 0.1
    md = torch.from_numpy(m).cuda()
    for c0, cnt in ((0, 200_000), (7, 123_457), (4096 * 3 + 5, 50_001)):
        cb = rt.raysample.CompactBuffers(cnt)
        _lib.check(_lib.lib().rtsdf_compact_mask_range(
            _lib.ptr(md), c0, cnt, None, _lib.ptr(cb.idx), _lib.ptr(cb.count), _lib.ptr(cb.ws),
            cb.ws.numel(), _lib.stream()), "compact_mask_range")
        k = int(cb.count.item())
        np.testing.assert_array_equal(_np(cb.idx[:k]), c0 + np.flatnonzero(m[c0:c0 + cnt]))


def test_bvh_closest_hits_match_reference(rt):
    G, A = golden(), golden_arrays()
    mesh = rt.make_mesh(A["soup.vertices"], A["soup.triangles"])
    bvh = rt.build_bvh(mesh)
    for k in ("node_lo", "node_hi", "node_left", "node_right", "order"):
        assert digest(getattr(bvh, k)) == G["soup.bvh"][k]
    t, ids, fac = rt.ray_query_many(bvh, A["soup.ray_o"], A["soup.ray_d"])
    np.testing.assert_array_equal(ids, A["soup.ray_id"])
    np.testing.assert_array_equal(fac, A["soup.ray_facing"])
    np.testing.assert_array_equal(t, A["soup.ray_t"])
    hit = rt.ray_query(bvh, A["soup.ray_o"][0], A["soup.ray_d"][0])
    assert hit.hit == (A["soup.ray_id"][0] >= 0)
    # the K6 search (fp32 conservative boxes + pre-test, fp64 confirm) == reference
    t2, ids2, fac2 = rt.ray_query_many(bvh, A["soup.ray_o"], A["soup.ray_d"], fast=True)
    np.testing.assert_array_equal(ids2, A["soup.ray_id"])
    np.testing.assert_array_equal(fac2, A["soup.ray_facing"])
    np.testing.assert_array_equal(t2, A["soup.ray_t"])


@pytest.mark.parametrize("name", ["sphere_plane", "thin_plate", "soup"])
def test_fast_traversal_equals_brute_force(rt, name):
    """geometry.py:3-6 contract: traversal == brute-force closest (t, min id)."""
    rng = np.random.default_rng(11)
    if name == "soup":
        A = golden_arrays()
        mesh = rt.make_mesh(A["soup.vertices"], A["soup.triangles"])
        lo, hi = np.zeros(3), np.ones(3)
    else:
        scene, mesh = scene_mesh(name)
        lo, hi = scene.lo, scene.hi
    bvh = rt.build_bvh(mesh)
    n = 20000
    o = rng.uniform(lo, hi, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    # a slice of axis-aligned and grazing directions (degenerate slabs)
    d[:500] = np.eye(3)[rng.integers(0, 3, 500)] * rng.choice([-1.0, 1.0], (500, 1))
    t_max = float(np.linalg.norm(hi - lo))
    assert bvh.search_nodes4 > 0
    tf, idf, ff = rt.ray_query_many(bvh, o, d, t_max, fast=True)  # BVH4 search
    tb2, idb2, fb2 = rt.ray_query_many(bvh, o, d, t_max, fast="binary")
    np.testing.assert_array_equal(idf, idb2)
    np.testing.assert_array_equal(tf, tb2)
    te, ide, fe = rt.ray_query_many(bvh, o, d, t_max, fast=False)
    np.testing.assert_array_equal(idf, ide)
    np.testing.assert_array_equal(tf, te)
    np.testing.assert_array_equal(ff, fe)
    # brute force over every triangle with the oracle's exact fp64 test
    b1 = O.bvh_build(mesh.vertices, mesh.triangles, mesh.normals)
    tb, ib, fb = O.ray_brute(b1, o, d, t_max)
    np.testing.assert_array_equal(idf, ib)
    np.testing.assert_array_equal(tf, tb)
    np.testing.assert_array_equal(ff, fb)


# ------------------------------------------------------------ ray sampling
def _c_setup(rt, name, dims):
    scene, mesh = scene_mesh(name)
    view = scene.view(0)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    coarse_np = O.seeds_to_sdf(O.jfa_run(occ, h), h)
    return scene, mesh, view, coarse_np, h


@pytest.mark.parametrize("name,dims,x", [("sphere", (64, 64, 64), 32), ("sphere", (64, 64, 64), 5),
                                         ("sphere", (64, 64, 64), 8), ("sphere", (64, 64, 64), 64),
                                         ("sphere_plane", (400, 200, 400), 32),
                                         ("thin_plate", (96, 80, 112), 40)])
def test_sample_hit_counts_bit_exact_host_table(rt, name, dims, x):
    """Same host direction table -> min t, front and back counts bit-exact."""
    scene, mesh, view, coarse_np, h = _c_setup(rt, name, dims)
    _, mask = O.resample_mask(coarse_np, scene.lo, scene.hi, dims, 0.1)
    idx = np.flatnonzero(mask.ravel())
    dirs = O.dir_table(0, idx, 1, x)
    b = O.bvh_build(mesh.vertices, mesh.triangles, mesh.normals)
    t_max = float(np.linalg.norm(scene.hi - scene.lo))
    wmin, wf, wb = O.sample_masked(b, idx, scene.lo, h, dims, x, 0, 1, t_max, dirs)
    coarse = rt.make_field(coarse_np, scene.lo, scene.hi)
    params = rt.SamplingParams(rays_per_frame=x)
    gidx, gmin, gf, gb = rt.sample_masked(coarse, dims, view.bvh, params, 1, directions=dirs)
    np.testing.assert_array_equal(_np(gidx), idx)
    np.testing.assert_array_equal(_np(gf), wf)
    np.testing.assert_array_equal(_np(gb), wb)
    np.testing.assert_array_equal(_np(gmin), wmin)


def test_update_fine_three_frames_golden(rt):
    """C1: three frames of update_fine with the host table == reference digests."""
    G = golden()
    scene, mesh = scene_mesh("sphere")
    view = scene.view(0)
    dims = (64, 64, 64)
    h = (scene.hi - scene.lo) / 64
    coarse_np = O.seeds_to_sdf(O.jfa_run(O.voxelize(mesh.vertices, mesh.triangles, dims,
                                                     scene.bounds), h), h)
    coarse = rt.make_field(coarse_np, scene.lo, scene.hi)
    params = rt.SamplingParams(rays_per_frame=32, mask_distance=0.1, decay_alpha=0.95, seed=0)
    fine = rt.fine_from_coarse(coarse, dims)
    acc = None
    for f in range(3):
        idx = _np(rt.raysample.masked_indices(rt.ray_mask(coarse, dims, 0.1)))
        fine, acc = rt.update_fine(fine, coarse, view.bvh, params, f, acc,
                                   directions=O.dir_table(0, idx, f, 32))
        g = G[f"c1.frame{f}"]
        assert digest(_np(fine.data)) == g["fine"], f
        assert digest(_np(acc.front)) == g["front"] and digest(_np(acc.back)) == g["back"]
        assert digest(_np(acc.min_dist)) == g["min_dist"]
        assert digest(_np(acc.mask)) == g["mask"]


@pytest.mark.parametrize("case", ["c1", "c3"])
def test_pipeline_frames_golden(rt, case):
    """hybrid_sdf / FramePipeline with the host table == reference frames."""
    G = golden()
    cfg = C1 if case == "c1" else C3
    scene = rt.get_scene(cfg["scene"])
    pc = rt.PipelineConfig(coarse_dims=cfg["dims"], fine_dims=cfg["dims"],
                           sampling=rt.SamplingParams(rays_per_frame=cfg["x"]))
    pipe = rt.FramePipeline(scene, pc)
    pipe.direction_fn = lambda idx, frame: O.dir_table(0, idx, frame, cfg["x"])
    frames = 3 if case == "c1" else 1
    for f in range(frames):
        rec = pipe.advance(render=(case == "c3"))
        g = G[f"{case}.frame{f}"]
        assert rec.masked_texels == g["masked"]
        assert digest(_np(pipe.coarse.data)) == g["coarse"]
        assert digest(_np(pipe.fine.data)) == g["fine"]
        assert digest(_np(pipe.accum.front)) == g["front"]
        assert digest(_np(pipe.accum.back)) == g["back"]
        assert set(rec.durations_ns) == {"V", "JF", "RT", "DL"}
    if case == "c3":
        gd = G["c3.dl"]
        occ = _np(pipe.last_occlusion)
        assert digest(occ) == gd["occlusion"]
        img = _np(pipe.last_image)
        np.testing.assert_allclose(img, golden_arrays()["c3.image"], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("timings", [(False, False, False), (False, True, False)])
def test_pipeline_overlapped_frames_golden(rt, timings):
    """Cross-frame flood overlap (static scene, timing=False: frame f + 1's V + JF
    run on the flood stream during frame f's RT) == the reference frames; the
    mixed case switches to the serial, event-timed path and back mid-run."""
    G = golden()
    scene = rt.get_scene(C1["scene"])
    pc = rt.PipelineConfig(coarse_dims=C1["dims"], fine_dims=C1["dims"],
                           sampling=rt.SamplingParams(rays_per_frame=C1["x"]))
    assert pc.overlap_frames is None  # auto
    pipe = rt.FramePipeline(scene, pc)
    assert pipe._overlap_for(scene.view(0))  # a 5,120-triangle tree: far below L2
    pipe.direction_fn = lambda idx, frame: O.dir_table(0, idx, frame, C1["x"])
    for f, timing in enumerate(timings):
        rec = pipe.advance(render=False, timing=timing)
        assert (pipe._prefetch is not None) == (not timing)  # frame f + 1 in flight
        g = G[f"c1.frame{f}"]
        assert rec.masked_texels == g["masked"]
        assert digest(_np(pipe.coarse.data)) == g["coarse"]
        assert digest(_np(pipe.fine.data)) == g["fine"]
        assert digest(_np(pipe.accum.front)) == g["front"]
        assert digest(_np(pipe.accum.back)) == g["back"]


def test_pipeline_overlap_c3_device_rng_identical(rt):
    """C3, device RNG, rendered: 3 overlapped frames == 3 serial frames, bit for bit."""
    out = []
    for overlap in (False, True):
        pc = rt.PipelineConfig(coarse_dims=C3["dims"], fine_dims=C3["dims"], overlap_frames=overlap,
                               sampling=rt.SamplingParams(rays_per_frame=C3["x"]))
        pipe = rt.FramePipeline(rt.get_scene(C3["scene"]), pc)
        for _ in range(3):
            rec = pipe.advance(render=True, timing=False)
        out.append((rec.masked_texels, _np(pipe.coarse.data), _np(pipe.fine.data),
                    _np(pipe.last_occlusion)))
        del pipe
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1:], out[1][1:]):
        np.testing.assert_array_equal(a, b)


def test_animated_scene_frames_match_oracle(rt):
    """Dynamic scene: the orbit scene's occluder moves every
    frame -> per-frame merged mesh + BVH; 3 frames of the pipeline with the host
    direction table == the oracle run on each frame's mesh (fine field, votes,
    masked count bit-exact)."""
    scene = rt.get_scene("orbit")
    dims = (64, 32, 64)
    x = 8
    pc = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims,
                           sampling=rt.SamplingParams(rays_per_frame=x))
    pipe = rt.FramePipeline(scene, pc)
    pipe.direction_fn = lambda idx, frame: O.dir_table(0, idx, frame, x)

    def mesh_at(f):
        m = scene.view(f).mesh
        return m.vertices, m.triangles, m.normals

    m0 = scene.view(0).mesh
    ho = O.HybridOracle(m0.vertices, m0.triangles, m0.normals, scene.bounds, dims, dims, x=x,
                        mesh_fn=mesh_at)
    prev_verts = None
    for f in range(3):
        rec = pipe.advance(render=False)
        want = ho.advance(dirs_fn=lambda idx, frame: O.dir_table(0, idx, frame, x))
        verts = scene.view(f).mesh.vertices
        if prev_verts is not None:
            assert not np.array_equal(verts, prev_verts)  # the occluder really moved
        prev_verts = verts
        assert rec.masked_texels == len(want["idx"]), f
        np.testing.assert_array_equal(_np(pipe.coarse.data), want["coarse"])
        np.testing.assert_array_equal(_np(pipe.fine.data), want["fine"])
        np.testing.assert_array_equal(_np(pipe.accum.front), ho.accum["front"])
        np.testing.assert_array_equal(_np(pipe.accum.back), ho.accum["back"])


# ---------------------------------------------------------- soft shadow (K8)
def test_gbuffer_and_occlusion_c3(rt):
    G, A = golden(), golden_arrays()
    scene, mesh = scene_mesh("sphere_plane")
    view = scene.view(0)
    gb = rt.rasterize_gbuffer(view, scene.camera)
    gd = G["c3.dl"]
    assert digest(_np(gb.coverage)) == gd["coverage"]
    assert digest(_np(gb.position)) == gd["position"]
    assert digest(_np(gb.normal)) == gd["normal"]
    assert digest(_np(gb.albedo)) == gd["albedo"]
    # occlusion over the oracle's frame-0 fine field
    dims = (400, 200, 400)
    H = O.HybridOracle(mesh.vertices, mesh.triangles, mesh.normals, scene.bounds, dims, dims, x=32)
    H.advance()
    fine = rt.make_field(H.fine, scene.lo, scene.hi)
    fld = rt.apply_bias(fine, 0.01)
    mp = rt.MarchParams.for_field(fine, max_step=0.05, max_iterations=256, jitter=1.0,
                                  light_angle=scene.light.angular_radius)
    occ = _np(rt.occlusion_image(gb, fld, scene.light, mp, draws=1, seed=0))
    np.testing.assert_array_equal(occ, A["c3.occlusion"])


def test_sphere_trace_kats_c1(rt):
    G, A = golden(), golden_arrays()
    mp = G["c1.march"]
    fld = rt.make_field(A["c1.fine2"], np.full(3, -2.0), np.full(3, 2.0), bias=0.0)
    fld = rt.apply_bias(fld, mp["bias"])
    params = rt.MarchParams(epsilon=mp["epsilon"], max_iterations=mp["max_iterations"],
                            max_step=mp["max_step"], t_max=mp["t_max"], jitter=1.0,
                            light_angle=mp["light_angle"])
    for o, d, want in zip(A["c1.trace_o"], A["c1.trace_d"], A["c1.trace_res"]):
        r = rt.sphere_trace(fld, o, d, params)
        st = {"hit": 0, "miss-exited": 1, "miss-max-iter": 2}[r.status]
        assert (r.t, r.iterations, r.occlusion, st) == tuple(want)


def test_soft_shadow_matches_oracle(rt):
    A = golden_arrays()
    fld = rt.make_field(A["c1.fine2"], np.full(3, -2.0), np.full(3, 2.0))
    params = rt.MarchParams.for_field(fld, light_angle=0.08)
    p = np.array([0.0, 1.2, 0.1])
    l = np.array([0.3, 1.0, 0.25])
    got = rt.soft_shadow(fld, p, l, params, seed=3, stream=7, draws=4)
    key = O.stream_key(3, 7, 0)
    lu = l / np.linalg.norm(l)
    total = 0.0
    for j in range(4):
        t0 = params.jitter * params.max_step * O.uniform(key, j)
        st, t, it, mt = O.march(A["c1.fine2"], np.full(3, -2.0), np.full(3, 4.0 / 64), p, lu,
                                params.epsilon, params.max_iterations, params.max_step,
                                params.t_max, t0, params.cone_k)
        total += 1.0 if st == 0 else 1.0 - mt
    assert got == total / 4


# ------------------------------------------------------------ field formats
def test_rsdf_roundtrip_and_errors(rt, tmp_path):
    A = golden_arrays()
    fld = rt.make_field(A["c1.fine2"], np.full(3, -2.0), np.full(3, 2.0), beta=0.1, bias=0.01,
                        frame=2)
    p = tmp_path / "f.rsdf"
    rt.save_field(fld, p)
    back = rt.load_field(p)
    np.testing.assert_array_equal(_np(back.data), A["c1.fine2"])
    assert back.frame == 2 and back.dims == fld.dims
    raw = bytearray(p.read_bytes())
    raw[0:4] = b"XXXX"
    p.write_bytes(bytes(raw))
    with pytest.raises(rt.FieldFormatError):
        rt.load_field(p)
    # (byte-for-byte compatibility with the reference's writer: test_host.py /
    # test_gpu_large.py against a reference-written file)


# ------------------------------------------------- validation oracles (f)-4
def _validation_golden():
    with np.load(Path(__file__).resolve().parent / "golden" / "golden_validation.npz") as z:
        return {k: z[k] for k in z.files}


def test_exact_distance_matches_reference(rt):
    """geometry.exact_distance_many on the GPU == the reference's, bit for bit
    (soup + C1 sphere, 3000 points each; reference traversal order)."""
    V, A = _validation_golden(), golden_arrays()
    soup = rt.make_mesh(A["soup.vertices"], A["soup.triangles"])
    np.testing.assert_array_equal(rt.exact_distance_many(rt.build_bvh(soup), V["soup.points"]),
                                  V["soup.exact_distance"])
    scene = rt.get_scene("sphere")
    view = scene.view(0)
    np.testing.assert_array_equal(rt.exact_distance_many(view.bvh, V["sphere.points"]),
                                  V["sphere.exact_distance"])
    assert rt.exact_distance(view.bvh, V["sphere.points"][7]) == V["sphere.exact_distance"][7]


def test_reference_visibility_matches_reference(rt):
    """render.reference_visibility on the GPU vs the reference (C1 camera, 16
    cone samples): coverage and per-pixel visibility bit-exact (the cone
    directions use the restated glibc cos/sin)."""
    V = _validation_golden()
    scene = rt.get_scene("sphere")
    view = scene.view(0)
    gb = rt.rasterize_gbuffer(view, scene.camera)
    np.testing.assert_array_equal(_np(gb.coverage), V["sphere.coverage"])
    vis = _np(rt.reference_visibility(view, gb, scene.light, spp=16, seed=3))
    want = V["sphere.visibility16"]
    np.testing.assert_array_equal(vis, want)
    img = _np(rt.reference_render(view, scene.camera, scene.light, spp=4, seed=0))
    assert img.shape == (scene.camera.height, scene.camera.width, 3) and np.isfinite(img).all()


@pytest.mark.parametrize("dims", [(1040, 14, 12), (12, 10, 1100)])
def test_frame_on_an_axis_beyond_1024(rt, dims):
    """A hybrid frame on a grid with one axis past the packed 10:10:10 seed
    layout (dims-dependent packed seeds, per-cell JFA kernel; resample weight
    tables sized from the dims) == the oracle."""
    scene = rt.get_scene("sphere")
    cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims,
                            sampling=rt.SamplingParams(rays_per_frame=4, mask_distance=0.3))
    pipe = rt.FramePipeline(scene, cfg)
    pipe.direction_fn = lambda idx, frame: O.dir_table(0, idx, frame, 4)
    rec = pipe.advance(render=False)
    mesh = scene.view(0).mesh
    h = O.HybridOracle(mesh.vertices, mesh.triangles, mesh.normals, scene.bounds, dims, dims, x=4, d=0.3)
    want = h.advance(dirs_fn=lambda idx, frame: O.dir_table(0, idx, frame, 4))
    assert rec.masked_texels == len(want["idx"])
    np.testing.assert_array_equal(_np(pipe.coarse.data), want["coarse"])
    np.testing.assert_array_equal(_np(pipe.fine.data), want["fine"])
