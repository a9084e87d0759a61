"""Golden fixtures for the large BASELINE configs, the coarse != fine frame, the
reference's orbit scene, the ghosting experiment and the RSDF writer -- all
produced by running the REFERENCE implementation itself.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \
        python tests/golden/make_golden_large.py [case ...]

Cases (SURVEY §8(d) names): c4 (512^3 hybrid frame of the 1,310,720-triangle
icosphere, ~4 min), c5 (1024^3 JFA of box_spheres, ~7 min), cf (sphere_plane
coarse 200x100x200 -> fine 400x200x400, 3 frames + DL), orbit (bundled
blob.obj orbiting, 3 frames + DL), ghost (bench.ghosting_experiment on the
orbit scene), rsdf (field.save_field bytes).  Writes / updates
tests/golden/golden_large.json (digests + scalars) and golden_large.npz (small
arrays).  Only this script imports the reference; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.path.insert(0, "/root/reference/pkg/src")
import sdfshadow as ref  # noqa: E402
from sdfshadow import bench as rbench  # noqa: E402
from sdfshadow import field as rfield  # noqa: E402
from sdfshadow import jfa as rjfa  # noqa: E402
from sdfshadow import render as rrender  # noqa: E402
from sdfshadow import scenes as rscenes  # noqa: E402

OUT = Path(__file__).resolve().parent
JSON = OUT / "golden_large.json"
NPZ = OUT / "golden_large.npz"


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def frame_facts(pipe):
    acc = pipe.accum
    return dict(coarse=digest(pipe.coarse.data), fine=digest(pipe.fine.data), mask=digest(acc.mask),
                masked=int(acc.mask.sum()), min_dist=digest(acc.min_dist), front=digest(acc.front),
                back=digest(acc.back), front_sum=int(acc.front.sum()), back_sum=int(acc.back.sum()))


def run_frames(G, ARR, name, scene, coarse_dims, fine_dims, x, frames, render_last=False):
    cfg = ref.PipelineConfig(coarse_dims=coarse_dims, fine_dims=fine_dims,
                             sampling=ref.SamplingParams(rays_per_frame=x, mask_distance=0.1,
                                                         decay_alpha=0.95, seed=0))
    pipe = ref.FramePipeline(scene, cfg)
    for f in range(frames):
        t0 = time.time()
        view = scene.view(f)
        G[f"{name}.mesh{f}"] = dict(vertices=digest(view.mesh.vertices),
                                    triangles=digest(view.mesh.triangles),
                                    normals=digest(view.mesh.normals))
        pipe.advance(render=render_last and f == frames - 1)
        G[f"{name}.frame{f}"] = frame_facts(pipe)
        log(f"{name} frame {f}: {time.time() - t0:.1f}s masked={G[f'{name}.frame{f}']['masked']}")
    if render_last:
        G[f"{name}.dl"] = dict(image=digest(pipe.last_image))
        ARR[f"{name}.image"] = pipe.last_image
    return pipe


def case_c4(G, ARR):
    mesh = rscenes.make_icosphere(1.0, subdivisions=8)
    scene = rscenes.Scene(name="big_sphere_8", instances=(rscenes.Instance(mesh),),
                          lo=np.full(3, -2.0), hi=np.full(3, 2.0),
                          light=rscenes.DirectionalLight((0.3, 1.0, 0.25), angular_radius=0.08),
                          camera=rscenes.Camera((0.0, 0.6, -3.2), (0.0, 0.0, 0.0), width=240,
                                                height=180))
    dims = (512, 512, 512)
    t0 = time.time()
    view = scene.view(0)
    log(f"c4 view (BVH build) {time.time() - t0:.1f}s")
    vg = ref.voxelize(view.mesh, dims, scene.bounds)
    t0 = time.time()
    seeds = rjfa.jfa_run(vg)
    log(f"c4 jfa {time.time() - t0:.1f}s")
    G["c4.jfa"] = dict(count=int(vg.count), occ=digest(vg.occupancy), seed=digest(seeds.seed))
    del seeds
    run_frames(G, ARR, "c4", scene, dims, dims, 32, 1)


def case_c5(G, ARR):
    mesh = rscenes.merge_meshes([
        rscenes.make_box((0, -.8, 0), (.9, .05, .9)), rscenes.make_box((-.4, -.4, .3), (.15, .3, .15)),
        rscenes.make_box((.45, -.5, -.35), (.2, .2, .2)), rscenes.make_icosphere(.25, (.3, .2, .4), 3),
        rscenes.make_icosphere(.18, (-.5, .4, -.4), 3), rscenes.make_icosphere(.35, (0, .45, -.1), 4)])
    dims = (1024, 1024, 1024)
    vg = ref.voxelize(mesh, dims, (np.full(3, -1.0), np.full(3, 1.0)))
    t0 = time.time()
    seeds = rjfa.jfa_run(vg)
    log(f"c5 jfa {time.time() - t0:.1f}s")
    sdf = rjfa.seeds_to_sdf(seeds)
    G["c5"] = dict(count=int(vg.count), occ=digest(vg.occupancy), seed=digest(seeds.seed),
                   coarse=digest(sdf.data), offsets=rjfa.jfa_offsets(dims))


def case_cf(G, ARR):
    scene = rscenes.get_scene("sphere_plane")
    run_frames(G, ARR, "cf", scene, (200, 100, 200), (400, 200, 400), 32, 3, render_last=True)


def case_orbit(G, ARR):
    scene = rscenes.get_scene("orbit")
    blob = rscenes.load_blob_mesh()
    G["orbit.blob"] = dict(vertices=digest(blob.vertices), triangles=digest(blob.triangles),
                           n_tris=int(blob.num_triangles))
    run_frames(G, ARR, "orbit", scene, (128, 64, 128), (128, 64, 128), 8, 3, render_last=True)


def case_ghost(G, ARR):
    scn = rbench.Scenario("ghost", scene="orbit", size="S", x=5)
    t0 = time.time()
    r = rbench.ghosting_experiment(scn)
    log(f"ghost {time.time() - t0:.1f}s tracked={r.tracked} max_ratio={r.max_ratio}")
    G["ghost"] = dict(scenario=dict(scene="orbit", size="S", x=5, warmup=10, window=14,
                                    band_lo=0.035),
                      frames=list(map(int, r.frames)), envelope=list(map(float, r.envelope)),
                      residual_in_band=list(map(float, r.residual_in_band)),
                      max_ratio=float(r.max_ratio), outside_exact=bool(r.outside_exact),
                      tracked=int(r.tracked), decays_within=bool(r.decays_within()))


def case_rsdf(G, ARR):
    rng = np.random.default_rng(11)
    data = rng.normal(size=(12, 10, 8)).astype(np.float32)
    fld = rfield.make_field(data, np.array([-1.0, -0.5, -2.0]), np.array([1.0, 0.75, 0.5]),
                            beta=0.125, bias=0.01, frame=5)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "f.rsdf"
        rfield.save_field(fld, p)
        raw = p.read_bytes()
    G["rsdf"] = dict(digest=hashlib.sha256(raw).hexdigest(), size=len(raw))
    ARR["rsdf.data"] = data
    ARR["rsdf.bytes"] = np.frombuffer(raw, np.uint8)


CASES = dict(rsdf=case_rsdf, cf=case_cf, orbit=case_orbit, ghost=case_ghost, c4=case_c4,
             c5=case_c5)


def main(names):
    G = json.loads(JSON.read_text()) if JSON.exists() else {}
    ARR = {}
    if NPZ.exists():
        with np.load(NPZ) as z:
            ARR = {k: z[k] for k in z.files}
    for n in names or list(CASES):
        log(n)
        t0 = time.time()
        CASES[n](G, ARR)
        G.setdefault("_meta", {})[n] = dict(seconds=round(time.time() - t0, 1))
        G["_meta"]["generator"] = "tests/golden/make_golden_large.py"
        G["_meta"]["reference"] = "sdfshadow " + ref.__version__
        JSON.write_text(json.dumps(G, indent=1, sort_keys=True))
        buf = io.BytesIO()
        np.savez_compressed(buf, **ARR)
        NPZ.write_bytes(buf.getvalue())
    log("done")


if __name__ == "__main__":
    main(sys.argv[1:])
