"""Bit-exact parity at every BASELINE config and on the §8(f) rows, against the
reference's own outputs (tests/golden/make_golden.py, make_golden_large.py).

  * C2: 256^3 box_spheres JFA (seeds, SDF);
  * C4: the 512^3 hybrid frame of the 1,310,720-triangle icosphere (seeds,
    coarse, fine, mask, min t, votes) -- device RNG, exactly as timed;
  * C5: the 1024^3 box_spheres JFA (10 passes; seeds and SDF);
  * coarse != fine: sphere_plane coarse 200x100x200 -> fine 400x200x400, three
    frames + the shaded image (the reference's default 2x ratio);
  * the reference's orbit scene (bundled blob.obj) over three frames + image;
  * the ghosting experiment (bench.py:310-364) on the orbit scene;
  * RSDF: the reference-written file read back.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from common import digest, golden, golden_large, golden_large_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    import paper_2210_06160_b200 as rt

    torch.cuda.set_device(0)
    return rt


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _check_frame(pipe, rec, g):
    assert rec.masked_texels == g["masked"]
    assert digest(_np(pipe.coarse.data)) == g["coarse"]
    assert digest(_np(pipe.accum.mask)) == g["mask"]
    assert digest(_np(pipe.fine.data)) == g["fine"]
    assert digest(_np(pipe.accum.min_dist)) == g["min_dist"]
    assert digest(_np(pipe.accum.front)) == g["front"]
    assert digest(_np(pipe.accum.back)) == g["back"]


def _box_spheres(rt):
    scene = rt.get_scene("box_spheres")
    return scene, scene.view(0).mesh


def test_c2_jfa_golden(rt):
    g = golden()["c2"]
    scene, mesh = _box_spheres(rt)
    vg = rt.voxelize(mesh, (256,) * 3, scene.bounds)
    assert vg.count == g["count"] and digest(_np(vg.occupancy)) == g["occ"]
    seeds = rt.jfa_run(vg)
    assert digest(_np(seeds.seed)) == g["seed"]
    assert digest(_np(rt.seeds_to_sdf(seeds).data)) == g["coarse"]


def test_c5_jfa_golden(rt):
    g = golden_large()["c5"]
    scene, mesh = _box_spheres(rt)
    dims = (1024,) * 3
    vg = rt.voxelize(mesh, dims, scene.bounds)
    assert vg.count == g["count"] and digest(_np(vg.occupancy)) == g["occ"]
    del vg
    sdf = rt.jump_flood(rt.voxelize(mesh, dims, scene.bounds))
    assert digest(_np(sdf.data)) == g["coarse"]
    del sdf
    torch.cuda.empty_cache()
    seeds = rt.jfa_run(rt.voxelize(mesh, dims, scene.bounds))
    assert digest(_np(seeds.seed)) == g["seed"]


def test_c4_frame_golden(rt):
    G = golden_large()
    scene = rt.get_scene("big_sphere")
    dims = (512,) * 3
    mesh = scene.view(0).mesh
    vg = rt.voxelize(mesh, dims, scene.bounds)
    assert vg.count == G["c4.jfa"]["count"] and digest(_np(vg.occupancy)) == G["c4.jfa"]["occ"]
    assert digest(_np(rt.jfa_run(vg).seed)) == G["c4.jfa"]["seed"]
    del vg
    cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims,
                            sampling=rt.SamplingParams(rays_per_frame=32))
    pipe = rt.FramePipeline(scene, cfg)
    rec = pipe.advance(render=False, timing=False)
    _check_frame(pipe, rec, G["c4.frame0"])


@pytest.mark.parametrize("timing", [True, False])
def test_coarse_ne_fine_frames_golden(rt, timing):
    G, A = golden_large(), golden_large_arrays()
    cfg = rt.PipelineConfig(coarse_dims=(200, 100, 200), fine_dims=(400, 200, 400),
                            sampling=rt.SamplingParams(rays_per_frame=32))
    pipe = rt.FramePipeline(rt.get_scene("sphere_plane"), cfg)
    for f in range(3):
        rec = pipe.advance(render=f == 2, timing=timing)
        _check_frame(pipe, rec, G[f"cf.frame{f}"])
    np.testing.assert_allclose(_np(pipe.last_image), A["cf.image"], rtol=1e-6, atol=1e-7)


def test_orbit_frames_golden(rt):
    """The reference's animated orbit scene (blob.obj): per-frame merged mesh +
    BVH, three frames == the reference's digests."""
    G, A = golden_large(), golden_large_arrays()
    scene = rt.get_scene("orbit")
    dims = (128, 64, 128)
    cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims,
                            sampling=rt.SamplingParams(rays_per_frame=8))
    pipe = rt.FramePipeline(scene, cfg)
    for f in range(3):
        rec = pipe.advance(render=f == 2)
        _check_frame(pipe, rec, G[f"orbit.frame{f}"])
    np.testing.assert_allclose(_np(pipe.last_image), A["orbit.image"], rtol=1e-6, atol=1e-7)


def test_ghosting_experiment_matches_reference(rt):
    from paper_2210_06160_b200.temporal import Scenario, ghosting_experiment

    g = golden_large()["ghost"]
    s = g["scenario"]
    r = ghosting_experiment(Scenario("ghost", scene=s["scene"], size=s["size"], x=s["x"]),
                            warmup=s["warmup"], window=s["window"], band_lo=s["band_lo"])
    assert r.tracked == g["tracked"]
    assert r.outside_exact == g["outside_exact"]
    assert r.frames == g["frames"]
    assert r.envelope == g["envelope"]
    assert r.residual_in_band == g["residual_in_band"]
    assert r.max_ratio == g["max_ratio"]
    assert r.decays_within() == g["decays_within"]


def test_rsdf_reads_reference_file(rt, tmp_path):
    G, A = golden_large(), golden_large_arrays()
    p = tmp_path / "ref.rsdf"
    p.write_bytes(A["rsdf.bytes"].tobytes())
    fld = rt.load_field(p)
    np.testing.assert_array_equal(_np(fld.data), A["rsdf.data"])
    assert fld.frame == 5 and fld.dims == A["rsdf.data"].shape
    assert np.float32(fld.beta) == np.float32(0.125) and np.float32(fld.bias) == np.float32(0.01)
    np.testing.assert_array_equal(fld.lo, [-1.0, -0.5, -2.0])
    q = tmp_path / "again.rsdf"
    rt.save_field(fld, q)
    assert q.read_bytes() == A["rsdf.bytes"].tobytes()
