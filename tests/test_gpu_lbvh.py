"""K5 on the device (csrc/lbvh.cu): the dynamic-scene search tree.

Any tree must give the reference's closest hit -- the brute-force (t, min id,
facing) over all triangles (geometry.py:3-6) -- so the device LBVH, its refit
after the vertices move, and the G-buffer traced through it are checked
against the oracle's brute force and the reference-order traversal.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from common import golden_arrays, scene_mesh

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rt():
    import paper_2210_06160_b200 as rt

    torch.cuda.set_device(0)
    return rt


def _device_bvh(rt, mesh, state=None, rebuild_every=8):
    from paper_2210_06160_b200.geometry import DeviceBvh
    from paper_2210_06160_b200.voxel import _MeshBuffers

    mb = _MeshBuffers(mesh.vertices, mesh.triangles)
    return DeviceBvh(mesh, mb.verts, mb.tris, state=state, rebuild_every=rebuild_every), mb


def _rays(rng, n, lo, hi):
    o = rng.uniform(lo, hi, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    return o, d


def _check_brute(rt, bvh, mesh, o, d, t_max=np.inf):
    tf, idf, ff = rt.ray_query_many(bvh, o, d, t_max, fast="binary")
    b = O.bvh_build(mesh.vertices, mesh.triangles, mesh.normals)
    tb, ib, fb = O.ray_brute(b, o, d, t_max)
    np.testing.assert_array_equal(idf, ib)
    np.testing.assert_array_equal(tf, tb)
    np.testing.assert_array_equal(ff, fb)
    return (ib >= 0).mean()


@pytest.mark.parametrize("name", ["sphere", "sphere_plane", "orbit", "soup"])
def test_lbvh_equals_brute_force(rt, name):
    rng = np.random.default_rng(11)
    if name == "soup":
        A = golden_arrays()
        mesh = rt.make_mesh(A["soup.vertices"], A["soup.triangles"])
        lo, hi = -0.2, 1.2
    else:
        scene, mesh = scene_mesh(name)
        lo, hi = scene.lo, scene.hi
    bvh, _ = _device_bvh(rt, mesh)
    assert bvh.search_nodes == 2 * mesh.num_triangles - 1 and not bvh.refit
    o, d = _rays(rng, 20000, lo, hi)
    assert _check_brute(rt, bvh, mesh, o, d) > 0.05


def test_lbvh_refit_after_motion(rt):
    """Same triangle list, moved vertices: the refit tree (old topology, new
    boxes) still returns the brute-force closest hits; so does a rebuild."""
    rng = np.random.default_rng(12)
    scene = rt.get_scene("orbit")
    state = {}
    meshes = [scene_mesh("orbit", f)[1] for f in range(4)]
    for f, mesh in enumerate(meshes):
        bvh, _ = _device_bvh(rt, mesh, state=state, rebuild_every=3)
        assert bvh.refit == (f % 3 != 0), f
        o, d = _rays(rng, 8000, scene.lo, scene.hi)
        _check_brute(rt, bvh, mesh, o, d)


def test_orbit_gbuffer_through_device_tree(rt):
    """The G-buffer of an animated frame (traced through the device tree) ==
    the one traced through the reference-order tree."""
    scene = rt.get_scene("orbit")
    view = scene.view(1)
    assert getattr(view.bvh, "device_built", False)
    gb_fast = rt.rasterize_gbuffer(view, scene.camera)
    ref = view.bvh.reference_tree()

    class _V:  # the same view, reference-order tree
        bvh = ref
        albedo_dev = view.albedo_dev

    gb_ref = rt.rasterize_gbuffer(_V, scene.camera)
    for a, b in ((gb_fast.coverage, gb_ref.coverage), (gb_fast.position, gb_ref.position),
                 (gb_fast.normal, gb_ref.normal), (gb_fast.albedo, gb_ref.albedo)):
        np.testing.assert_array_equal(a.cpu().numpy(), b.cpu().numpy())
    assert gb_fast.coverage.sum() > 1000
