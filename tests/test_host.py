"""CPU tests of the product's host side: the C ABI surface, host BVH build,
scene inputs, validation and scalar API functions (no GPU compute)."""

import ctypes
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from common import digest, golden, golden_arrays, golden_large, golden_large_arrays, scene_mesh

ROOT = Path(__file__).resolve().parent.parent


def _header_symbols():
    text = (ROOT / "include" / "rtsdf.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rtsdf_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2210_06160_b200 import _lib

    lib = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.rtsdf_version().decode().startswith("rtsdf-b200")


def test_bvh4_nodes_are_128_byte_aligned_in_the_packed_layout():
    """The BVH4 collapse is appended at rtsdf_bvh_packed_bytes: a multiple of
    128 B, so its nodes (fetched with 256-bit loads) are aligned for any mesh."""
    from paper_2210_06160_b200 import _lib

    lib = _lib.lib()
    for n_nodes, n_tris in ((1, 1), (3, 2), (1023, 1282), (2047, 7716), (1048575, 1310720), (7, 5)):
        nb = int(lib.rtsdf_bvh_packed_bytes(n_nodes, n_tris))
        assert nb % 128 == 0, (n_nodes, n_tris, nb)
        assert nb >= n_nodes * 64 + n_tris * (128 + 48)


def test_library_is_sm100a():
    import subprocess

    from paper_2210_06160_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("case", ["c1", "soup"])
def test_host_bvh_build_is_the_reference_tree(case):
    """rtsdf_bvh_build_host (C++) == geometry.build_bvh's median-split tree."""
    from paper_2210_06160_b200 import _lib

    G = golden()
    if case == "c1":
        _, mesh = scene_mesh("sphere")
        v, t = mesh.vertices, mesh.triangles
    else:
        A = golden_arrays()
        v, t = A["soup.vertices"], A["soup.triangles"]
    p0, p1, p2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    lo = np.ascontiguousarray(np.minimum(np.minimum(p0, p1), p2))
    hi = np.ascontiguousarray(np.maximum(np.maximum(p0, p1), p2))
    T = len(t)
    nlo, nhi = np.empty((2 * T, 3)), np.empty((2 * T, 3))
    left, right = np.empty(2 * T, np.int32), np.empty(2 * T, np.int32)
    order = np.empty(T, np.int32)
    L = _lib.lib()
    n = L.rtsdf_bvh_build_host(*[_lib.host_ptr(a) for a in (lo, hi)], T,
                               *[_lib.host_ptr(a) for a in (nlo, nhi, left, right, order)])
    g = G[f"{case}.bvh"]
    assert n == g["n_nodes"]
    assert digest(nlo[:n]) == g["node_lo"] and digest(nhi[:n]) == g["node_hi"]
    assert digest(left[:n]) == g["node_left"] and digest(right[:n]) == g["node_right"]
    assert digest(order) == g["order"]


def test_bvh4_collapse_writes_eight_octant_copies_per_node():
    """rtsdf_bvh4_collapse_host: record 8 i + o is node i with the x / y / z lo
    and hi planes swapped where bit 0 / 1 / 2 of o is set, inner child refs are
    copy-0 records (multiples of 8), and every child box contains its
    subtree's triangles (the traversal reads a ray's near planes from the lo
    slots of its octant copy)."""
    from paper_2210_06160_b200 import _lib

    _, mesh = scene_mesh("sphere_plane")
    v, t = mesh.vertices, mesh.triangles
    p0, p1, p2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    lo = np.ascontiguousarray(np.minimum(np.minimum(p0, p1), p2))
    hi = np.ascontiguousarray(np.maximum(np.maximum(p0, p1), p2))
    T = len(t)
    L = _lib.lib()
    slo, shi = np.empty((2 * T, 3)), np.empty((2 * T, 3))
    sl, sr = np.empty(2 * T, np.int32), np.empty(2 * T, np.int32)
    so = np.empty(T, np.int32)
    ns = L.rtsdf_bvh_build_sah_host(_lib.host_ptr(lo), _lib.host_ptr(hi), T, 4,
                                    *[_lib.host_ptr(a) for a in (slo, shi, sl, sr, so)])
    assert ns > 0
    recs = np.zeros((8 * ns, 128), np.uint8)
    n4 = L.rtsdf_bvh4_collapse_host(*[_lib.host_ptr(np.ascontiguousarray(a[:ns])) for a in (slo, shi, sl, sr)],
                                    int(ns), _lib.host_ptr(recs), recs.shape[0])
    assert n4 > 0 and n4 % 8 == 0
    assert L.rtsdf_bvh4_collapse_host(*[_lib.host_ptr(np.ascontiguousarray(a[:ns])) for a in (slo, shi, sl, sr)],
                                      int(ns), _lib.host_ptr(recs), n4 - 1) < 0  # capacity counts records
    f = recs[:n4].view(np.float32).reshape(-1, 8, 32)
    c = recs[:n4].view(np.int32).reshape(-1, 8, 32)[:, :, 24:28]
    base = f[:, 0, :24].reshape(-1, 6, 4)  # lox, loy, loz, hix, hiy, hiz
    for o in range(8):
        want = base.copy()
        for a in range(3):
            if o >> a & 1:
                want[:, [a, a + 3]] = want[:, [a + 3, a]]
        assert np.array_equal(f[:, o, :24].reshape(-1, 6, 4), want), o
        assert np.array_equal(c[:, o], c[:, 0]), o
    inner = c[:, 0][(c[:, 0] >= 0) & (c[:, 0] != 0x7FFFFFFF)]
    assert len(inner) and np.all(inner % 8 == 0) and np.all(inner < n4)
    # every triangle sits inside the padded box of each BVH4 child on its path
    order = so[:T]
    tri_lo, tri_hi = lo[order], hi[order]

    def check(rec, blo, bhi):
        for q in range(4):
            ref = int(c[rec // 8, 0, q])
            if ref == 0x7FFFFFFF:
                continue
            qlo = np.array([base[rec // 8, a, q] for a in range(3)], np.float64)
            qhi = np.array([base[rec // 8, 3 + a, q] for a in range(3)], np.float64)
            if ref < 0:
                code = -ref - 1
                s0, cnt = code >> 3, code & 7
                assert np.all(tri_lo[s0:s0 + cnt] >= qlo) and np.all(tri_hi[s0:s0 + cnt] <= qhi)
            else:
                check(ref, qlo, qhi)

    check(0, None, None)


@pytest.mark.parametrize("name,key", [("sphere", "c1"), ("sphere_plane", "c3")])
def test_scene_meshes_match_reference(name, key):
    _, mesh = scene_mesh(name)
    g = golden()[f"{key}.mesh"]
    assert mesh.num_triangles == g["n_tris"]
    for k in ("vertices", "triangles", "normals"):
        assert digest(getattr(mesh, k)) == g[k], k


def test_orbit_scene_is_the_references_blob_orbit():
    """the orbit scene's occluder is the vendored blob.obj and its
    per-frame merged meshes equal the reference's (tests/golden/make_golden_large.py)."""
    from paper_2210_06160_b200 import scenes

    G = golden_large()
    blob = scenes.load_blob_mesh()
    assert blob.num_triangles == G["orbit.blob"]["n_tris"] == 1024
    assert digest(blob.vertices) == G["orbit.blob"]["vertices"]
    assert digest(blob.triangles) == G["orbit.blob"]["triangles"]
    for f in range(3):
        _, mesh = scene_mesh("orbit", f)
        for k in ("vertices", "triangles", "normals"):
            assert digest(getattr(mesh, k)) == G[f"orbit.mesh{f}"][k], (f, k)


def test_rsdf_writer_bytes_match_reference(tmp_path):
    """field.save_field writes the reference's RSDF v1 bytes exactly (header
    <4sI3I6fffQ + x-fastest f32 payload, field.py:190-201); the reader side of
    the reference-written file is a GPU test (load_field returns a device field)."""
    import torch

    from paper_2210_06160_b200 import field as F

    G, A = golden_large(), golden_large_arrays()
    data = A["rsdf.data"]
    fld = F.DistanceField(torch.from_numpy(data.copy()), np.array([-1.0, -0.5, -2.0]),
                          np.array([1.0, 0.75, 0.5]), beta=0.125, bias=0.01, frame=5)
    p = tmp_path / "ours.rsdf"
    F.save_field(fld, p)
    raw = p.read_bytes()
    assert len(raw) == G["rsdf"]["size"]
    assert raw == A["rsdf.bytes"].tobytes()
    # x-fastest payload: the first nx floats are data[:, 0, 0]
    hdr = len(raw) - data.size * 4
    np.testing.assert_array_equal(np.frombuffer(raw[hdr:hdr + 4 * data.shape[0]], np.float32),
                                  data[:, 0, 0])


def test_integer_weights_exact():
    from paper_2210_06160_b200.jfa import integer_weights

    # C3: hx = hz = 3.2/400, hy = 3.2/200 = 2 hx exactly -> (1, 4, 1)
    lo, hi = np.array([-1.6, -0.1, -1.6]), np.array([1.6, 3.1, 1.6])
    h = (hi - lo) / np.array([400, 200, 400], dtype=np.float64)
    assert integer_weights(*map(float, h), (400, 200, 400)) == (1, 4, 1)
    assert integer_weights(0.1, 0.1, 0.1, (16, 16, 16)) == (1, 1, 1)
    # fp64 0.1/0.3/0.7 are not in small-integer ratio -> general fp64 path
    assert integer_weights(0.1, 0.3, 0.7, (16, 16, 16)) == (0, 0, 0)
    # any returned weights must be exact ratios of the squared fp64 spacings
    for hs in [(0.008, 0.016, 0.008), (1 / 3, 2 / 3, 1 / 3), (0.25, 0.5, 1.0)]:
        w = integer_weights(*hs, (64, 64, 64))
        if w != (0, 0, 0):
            sq = [Fraction(x) ** 2 for x in hs]
            assert sq[0] * w[1] == sq[1] * w[0] and sq[0] * w[2] == sq[2] * w[0]


def test_jfa_offsets_schedule():
    from paper_2210_06160_b200.jfa import jfa_offsets

    assert jfa_offsets((128, 128, 128)) == [64, 32, 16, 8, 4, 2, 1]
    assert jfa_offsets((400, 200, 400)) == [256, 128, 64, 32, 16, 8, 4, 2, 1]
    assert jfa_offsets((64, 64, 64)) == [32, 16, 8, 4, 2, 1]


def test_sampling_params_validation_and_scalar_kats():
    from paper_2210_06160_b200.raysample import SamplingParams, accumulate, resolve_sign

    with pytest.raises(ValueError):
        SamplingParams(rays_per_frame=-1)
    with pytest.raises(ValueError):
        SamplingParams(mask_distance=0)
    with pytest.raises(ValueError):
        SamplingParams(decay_alpha=1.0)
    p = SamplingParams()
    # SPEC.md raysample KATs
    assert accumulate(0.5, 0.05, 0.2, p) == pytest.approx(0.2)
    assert accumulate(0.5, 0.4, 0.01, p) == 0.4
    assert accumulate(0.02, 0.05, None, p) == pytest.approx(0.0215)
    assert resolve_sign(0.3, 10, 2) == 0.3
    assert resolve_sign(0.3, 2, 10) == -0.3
    assert resolve_sign(0.3, 5, 5) == 0.3
    assert resolve_sign(None, 1, 2) is None


def test_march_params_validation():
    from paper_2210_06160_b200.raymarch import MarchParams

    for bad in (dict(epsilon=0), dict(max_iterations=0), dict(max_step=0), dict(jitter=1.5),
                dict(light_angle=0.0)):
        with pytest.raises(ValueError):
            MarchParams(**bad)
    assert MarchParams(light_angle=0.08).cone_k == pytest.approx(12.473, rel=1e-4)


def test_pipeline_config_validation():
    from paper_2210_06160_b200.pipeline import PipelineConfig

    with pytest.raises(ValueError):
        PipelineConfig(coarse_dims=(3, 3, 3), fine_dims=(4, 4, 4))
    PipelineConfig(coarse_dims=(200, 100, 200), fine_dims=(400, 200, 400))


def test_load_mesh_obj_subset():
    from paper_2210_06160_b200.geometry import EmptyMeshError, MeshParseError, load_mesh

    m = load_mesh(b"v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n")
    assert m.num_triangles == 2
    np.testing.assert_allclose(m.normals, [[0, 0, 1], [0, 0, 1]])
    with pytest.raises(MeshParseError):
        load_mesh(b"v 0 0\nf 1 2 3\n")
    with pytest.raises(EmptyMeshError):
        load_mesh(b"v 0 0 0\n")


def test_product_does_not_import_oracle():
    """Only tests/, smoke() and bench.py may touch oracle/ (the checker)."""
    pkg = ROOT / "paper_2210_06160_b200"
    pat = re.compile(r"(import\s+oracle|from\s+oracle|rtsdf_oracle|oracle\.py|sys\.path.*oracle)")
    for f in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*.c*")):
        assert not pat.search(f.read_text()), f


def test_pipeline_overlap_config_host_side():
    """Flood-ahead overlap knobs (no GPU): auto by default, switchable per
    pipeline, join() a no-op with nothing flooded ahead, animated scenes never
    overlap (their next frame needs a new mesh + BVH)."""
    import paper_2210_06160_b200 as rt

    pc = rt.PipelineConfig(coarse_dims=(8, 8, 8), fine_dims=(8, 8, 8))
    assert pc.overlap_frames is None
    pipe = rt.FramePipeline(rt.get_scene("sphere"), pc)
    assert pipe.overlap_frames is None and pipe._prefetch is None
    pipe.join()
    pipe.overlap_frames = False
    assert pipe._overlap_for(None) is False  # explicit setting wins before any BVH lookup
    assert rt.get_scene("orbit").animated and not rt.get_scene("sphere").animated
    assert rt.FramePipeline.OVERLAP_MAX_BVH_BYTES < 126 << 20
