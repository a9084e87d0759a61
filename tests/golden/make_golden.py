"""Generate the golden fixtures by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.json (sha256 digests + scalar facts) and
tests/golden/golden.npz (small arrays).  The reference (`sdfshadow`) is only
imported here; nothing at test/bench time reads /root/reference.  Every
value is the reference's own output on the survey's configs (SURVEY §8(d),
Appendix A).  tests/test_oracle_golden.py pins the CPU oracle to these
fixtures; the GPU parity tests compare the CUDA path to the oracle and to
the same digests.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.path.insert(0, "/root/reference/pkg/src")
import sdfshadow as ref  # noqa: E402
from sdfshadow import geometry as rgeo  # noqa: E402
from sdfshadow import jfa as rjfa  # noqa: E402
from sdfshadow import raysample as rrs  # noqa: E402
from sdfshadow import render as rrender  # noqa: E402
from sdfshadow import rng as rrng  # noqa: E402
from sdfshadow import scenes as rscenes  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


G: dict = {}
ARR: dict = {}


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def mesh_facts(name, mesh):
    G[f"{name}.mesh"] = dict(vertices=digest(mesh.vertices), triangles=digest(mesh.triangles),
                             normals=digest(mesh.normals), n_tris=int(mesh.num_triangles))


def bvh_facts(name, bvh):
    G[f"{name}.bvh"] = {k: digest(getattr(bvh, k)) for k in
                        ("node_lo", "node_hi", "node_left", "node_right", "order")}
    G[f"{name}.bvh"]["n_nodes"] = int(bvh.num_nodes)


def case_jfa_tie():
    """Appendix A.1: 16^3, h = 0.1, seeds (0,3,4) and (5,0,0)."""
    occ = np.zeros((16, 16, 16), np.uint8)
    occ[0, 3, 4] = 1
    occ[5, 0, 0] = 1
    vg = ref.VoxelGrid(occ, np.zeros(3), np.full(3, 1.6))
    seeds = rjfa.jfa_run(vg)
    ARR["jfa_tie.seed"] = seeds.seed
    G["jfa_tie"] = dict(seed_000=int(seeds.seed[0, 0, 0]), expected_linear_500=5 * 256,
                        digest=digest(seeds.seed))
    sdf = rjfa.seeds_to_sdf(seeds, beta=0.0)
    ARR["jfa_tie.sdf"] = sdf.data


def case_voxel_square():
    """Closed-box SAT: square [0,4] x {0.5} x [0,4] on a unit 8^3 grid."""
    verts = np.array([[0, 0.5, 0], [4, 0.5, 0], [4, 0.5, 4], [0, 0.5, 4]], np.float64)
    tris = np.array([[0, 1, 2], [0, 2, 3]], np.int32)
    vg = ref.voxelize((verts, tris), (8, 8, 8), (np.zeros(3), np.full(3, 8.0)))
    ARR["voxel_square.occ"] = vg.occupancy
    G["voxel_square"] = dict(count=int(vg.count))


def case_random_soup():
    rng = np.random.default_rng(7)
    verts = rng.uniform(0.05, 0.95, size=(300, 3))
    tris = rng.integers(0, 300, size=(200, 3)).astype(np.int32)
    mesh = rgeo.make_mesh(verts, tris)
    ARR["soup.vertices"] = mesh.vertices
    ARR["soup.triangles"] = mesh.triangles
    vg = ref.voxelize(mesh, (40, 33, 27), (np.zeros(3), np.ones(3)))
    G["soup.voxel"] = dict(count=int(vg.count), occ=digest(vg.occupancy))
    seeds = rjfa.jfa_run(vg)
    G["soup.jfa"] = dict(seed=digest(seeds.seed))
    sdf = rjfa.seeds_to_sdf(seeds, beta=0.01)
    G["soup.sdf"] = dict(data=digest(sdf.data))
    bvh = rgeo.build_bvh(mesh)
    bvh_facts("soup", bvh)
    # closest-hit queries vs the reference BVH
    o = rng.uniform(-0.2, 1.2, size=(4096, 3))
    d = rng.normal(size=(4096, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    t = np.empty(4096); ids = np.empty(4096, np.int32); fac = np.empty(4096, np.int32)
    for q in range(4096):
        hit = rgeo.ray_query(bvh, o[q], d[q], t_max=np.inf)
        t[q], ids[q], fac[q] = (hit.t, hit.triangle, hit.facing) if hit.hit else (-1.0, -1, 0)
    ARR["soup.ray_o"], ARR["soup.ray_d"] = o, d
    ARR["soup.ray_t"], ARR["soup.ray_id"], ARR["soup.ray_facing"] = t, ids, fac


def case_rng():
    keys = [rrng.stream_key(0, s, f) for s in (0, 1, 12345, 31999999) for f in (0, 1, 2)]
    G["rng.keys"] = [int(k) for k in keys]
    idx = np.arange(0, 64000, 641, dtype=np.int64)
    dirs = np.empty((len(idx), 32, 3))
    for n, lin in enumerate(idx):
        key = np.uint64(rrng.stream_key(0, lin, 2))
        for r in range(32):
            dirs[n, r] = rrng.unit_sphere_dir(key, np.uint64(r))
    G["rng.dirs"] = dict(idx=idx.tolist(), frame=2, x=32, digest=digest(dirs))
    ARR["rng.dirs"] = dirs


def run_pipeline(name, scene, coarse_dims, fine_dims, x, frames, render_last=False):
    cfg = ref.PipelineConfig(coarse_dims=coarse_dims, fine_dims=fine_dims,
                             sampling=ref.SamplingParams(rays_per_frame=x, mask_distance=0.1,
                                                         decay_alpha=0.95, seed=0))
    pipe = ref.FramePipeline(scene, cfg)
    view = scene.view(0)
    mesh_facts(name, view.mesh)
    bvh_facts(name, view.bvh)
    vg = ref.voxelize(view.mesh, coarse_dims, scene.bounds)
    seeds = rjfa.jfa_run(vg)
    G[f"{name}.voxel"] = dict(count=int(vg.count), occ=digest(vg.occupancy))
    G[f"{name}.jfa"] = dict(seed=digest(seeds.seed), offsets=rjfa.jfa_offsets(seeds.dims))
    for f in range(frames):
        t0 = time.time()
        pipe.advance(render=render_last and f == frames - 1)
        log(f"{name} frame {f}: {time.time() - t0:.1f}s masked={int(pipe.accum.mask.sum())}")
        acc = pipe.accum
        G[f"{name}.frame{f}"] = dict(
            coarse=digest(pipe.coarse.data), fine=digest(pipe.fine.data),
            mask=digest(acc.mask), masked=int(acc.mask.sum()), min_dist=digest(acc.min_dist),
            front=digest(acc.front), back=digest(acc.back),
            front_sum=int(acc.front.sum()), back_sum=int(acc.back.sum()))
    return pipe, view


def case_c1():
    pipe, view = run_pipeline("c1", rscenes.get_scene("sphere"), (64, 64, 64), (64, 64, 64), 32, 3)
    ARR["c1.fine2"] = pipe.fine.data
    # sphere traces over the fine field
    fld = pipe.fine_for_shading
    mp = pipe.march_params()
    rng = np.random.default_rng(3)
    res = []
    for q in range(64):
        o = rng.uniform(-1.9, 1.9, size=3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        r = ref.sphere_trace(fld, o, d, mp)
        res.append([float(r.t), float(r.iterations), float(r.occlusion),
                    {"hit": 0, "miss-exited": 1, "miss-max-iter": 2}[r.status]])
        ARR.setdefault("c1.trace_o", []).append(o)
        ARR.setdefault("c1.trace_d", []).append(d)
    ARR["c1.trace_o"] = np.array(ARR["c1.trace_o"])
    ARR["c1.trace_d"] = np.array(ARR["c1.trace_d"])
    ARR["c1.trace_res"] = np.array(res)
    G["c1.march"] = dict(epsilon=mp.epsilon, t_max=mp.t_max, max_step=mp.max_step,
                         max_iterations=mp.max_iterations, light_angle=mp.light_angle,
                         bias=float(fld.bias))


def case_sphere_plane_128():
    scene = rscenes.get_scene("sphere_plane")
    view = scene.view(0)
    vg = ref.voxelize(view.mesh, (128, 128, 128), scene.bounds)
    seeds = rjfa.jfa_run(vg)
    coarse = rjfa.seeds_to_sdf(seeds)
    fine, mask = rrs._resample_and_mask(coarse, (128, 128, 128), 0.1)
    G["sp128"] = dict(count=int(vg.count), occ=digest(vg.occupancy), seed=digest(seeds.seed),
                      coarse=digest(coarse.data), fine=digest(fine), mask=digest(mask),
                      masked=int(mask.sum()),
                      resample_max_diff=float(np.abs(fine.astype(np.float64) - coarse.data).max()))
    fine2, _ = rrs._resample_and_mask(coarse, (256, 256, 256), 0.1)
    G["sp128.fine256"] = dict(fine=digest(fine2))


def case_c2():
    mesh = rscenes.merge_meshes([
        rscenes.make_box((0, -.8, 0), (.9, .05, .9)), rscenes.make_box((-.4, -.4, .3), (.15, .3, .15)),
        rscenes.make_box((.45, -.5, -.35), (.2, .2, .2)), rscenes.make_icosphere(.25, (.3, .2, .4), 3),
        rscenes.make_icosphere(.18, (-.5, .4, -.4), 3), rscenes.make_icosphere(.35, (0, .45, -.1), 4)])
    mesh_facts("c2", mesh)
    vg = ref.voxelize(mesh, (256, 256, 256), (np.full(3, -1.0), np.full(3, 1.0)))
    t0 = time.time()
    seeds = rjfa.jfa_run(vg)
    log(f"c2 jfa {time.time() - t0:.1f}s")
    coarse = rjfa.seeds_to_sdf(seeds)
    G["c2"] = dict(count=int(vg.count), occ=digest(vg.occupancy), seed=digest(seeds.seed),
                   coarse=digest(coarse.data))


def case_c3():
    scene = rscenes.get_scene("sphere_plane")
    dims = (400, 200, 400)
    pipe, view = run_pipeline("c3", scene, dims, dims, 32, 1, render_last=True)
    # DL pass pieces at the scene camera
    gb = rrender.rasterize_gbuffer(view, scene.camera)
    occ = rrender.occlusion_image(gb, pipe.fine_for_shading, scene.light, pipe.march_params(),
                                  draws=1, seed=0)
    G["c3.dl"] = dict(coverage=digest(gb.coverage), covered=int(gb.coverage.sum()),
                      position=digest(gb.position), normal=digest(gb.normal),
                      albedo=digest(gb.albedo), occlusion=digest(occ),
                      occlusion_sum=float(occ.sum()))
    ARR["c3.occlusion"] = occ.astype(np.float64)
    ARR["c3.image"] = pipe.last_image


def main():
    t0 = time.time()
    for fn in (case_jfa_tie, case_voxel_square, case_random_soup, case_rng, case_c1,
               case_sphere_plane_128, case_c2, case_c3):
        log(fn.__name__)
        fn()
    G["_meta"] = dict(generator="tests/golden/make_golden.py", reference="sdfshadow "
                      + ref.__version__, numba=__import__("numba").__version__,
                      numpy=np.__version__, seconds=round(time.time() - t0, 1))
    (OUT / "golden.json").write_text(json.dumps(G, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "golden.npz", **{k: np.asarray(v) for k, v in ARR.items()})
    log("done")


if __name__ == "__main__":
    main()
