"""Golden vectors for the validation oracles: the REFERENCE's
exact_distance_many (geometry.py:588-594) and reference_visibility
(render.py:231-254), run in the build container (the only place
/root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nbcache \\
        python tests/golden/make_golden_validation.py

Writes tests/golden/golden_validation.npz.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.path.insert(0, "/root/reference/pkg/src")
from sdfshadow import geometry as rgeo  # noqa: E402
from sdfshadow import render as rrender  # noqa: E402
from sdfshadow import scenes as rscenes  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    arr = {}
    # exact distance: the golden random soup (golden.npz) + the C1 sphere
    with np.load(OUT / "golden.npz") as z:
        sv, st = z["soup.vertices"], z["soup.triangles"]
    soup = rgeo.make_mesh(sv, st)
    rng = np.random.default_rng(21)
    pts = rng.uniform(-0.2, 1.2, size=(3000, 3))
    pts[:200] = sv[rng.integers(0, len(sv), 200)]  # on vertices: distance 0
    arr["soup.points"] = pts
    arr["soup.exact_distance"] = rgeo.exact_distance_many(rgeo.build_bvh(soup), pts)
    sphere = rscenes.get_scene("sphere")
    view = sphere.view(0)
    p2 = rng.uniform(-2.0, 2.0, size=(3000, 3))
    arr["sphere.points"] = p2
    arr["sphere.exact_distance"] = rgeo.exact_distance_many(view.bvh, p2)
    # reference visibility: C1 scene camera, 16 cone samples per pixel
    gb = rrender.rasterize_gbuffer(view, sphere.camera)
    vis = rrender.reference_visibility(view, gb, sphere.light, spp=16, seed=3)
    arr["sphere.visibility16"] = vis
    arr["sphere.coverage"] = gb.coverage
    np.savez_compressed(OUT / "golden_validation.npz", **arr)
    print({k: v.shape for k, v in arr.items()})


if __name__ == "__main__":
    main()
