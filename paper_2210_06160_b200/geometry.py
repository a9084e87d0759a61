"""Triangle meshes, the BVH, and batched closest-hit ray queries.

Mirrors sdfshadow.geometry (geometry.py:1-410).  Mesh construction stays on
the host in numpy (it is the input format, geometry.py:76-163); the BVH is
built by the library's C++ median-split builder (rtsdf_bvh_build_host, the
reference's own tree, geometry.py:202-267), uploaded once and packed into the
device traversal layout; queries run on the GPU (rtsdf_ray_query).
"""

from __future__ import annotations

import logging
import os
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from ._device import to_device, to_numpy

log = logging.getLogger(__name__)

DEGENERATE_AREA = 1e-12
# leaf size of the K6 search tree (binned SAH; csrc/bvh.cu)
SAH_MAX_LEAF = int(os.environ.get("RTSDF_SAH_LEAF", "4"))
USE_BVH4 = os.environ.get("RTSDF_BVH4", "1") != "0"
FACING_NONE = 0
FACING_FRONT = 1
FACING_BACK = 2


class MeshError(ValueError):
    pass


class MeshParseError(MeshError):
    def __init__(self, line_no, message):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class EmptyMeshError(MeshError):
    pass


@dataclass(frozen=True)
class TriangleMesh:
    """Immutable triangle soup with per-face unit normals (geometry.py:41-64)."""

    vertices: np.ndarray   # (V, 3) float64
    triangles: np.ndarray  # (T, 3) int32
    normals: np.ndarray    # (T, 3) float64
    dropped: int = 0

    @property
    def bounds(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    @property
    def num_triangles(self):
        return len(self.triangles)

    def transformed(self, transform):
        m = np.asarray(transform, dtype=np.float64)
        if m.shape != (3, 4):
            raise MeshError(f"transform must be 3x4, got {m.shape}")
        return make_mesh(self.vertices @ m[:, :3].T + m[:, 3], self.triangles,
                         dropped=self.dropped)


def _face_normals(vertices, triangles):
    a = vertices[triangles[:, 0]]
    n = np.cross(vertices[triangles[:, 1]] - a, vertices[triangles[:, 2]] - a)
    return n, np.linalg.norm(n, axis=1)


def make_mesh(vertices, triangles, dropped=0) -> TriangleMesh:
    """Drop faces with area < 1e-12 and attach unit normals (geometry.py:76-91)."""
    vertices = np.ascontiguousarray(vertices, dtype=np.float64)
    triangles = np.ascontiguousarray(triangles, dtype=np.int32)
    if triangles.ndim != 2 or triangles.shape[1] != 3:
        raise MeshError("triangles must be (T, 3)")
    if len(triangles) and triangles.max() >= len(vertices):
        raise MeshError("triangle index out of range")
    n, lengths = _face_normals(vertices, triangles)
    keep = lengths * 0.5 >= DEGENERATE_AREA
    n_dropped = int((~keep).sum()) + dropped
    triangles = triangles[keep]
    if len(triangles) == 0:
        raise EmptyMeshError("no non-degenerate triangles")
    return TriangleMesh(vertices, triangles, n[keep] / lengths[keep][:, None], n_dropped)


def _parse_obj(text):
    verts, faces = [], []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        fields = raw.split()
        if not fields or fields[0].startswith("#"):
            continue
        tag = fields[0]
        if tag == "v":
            if len(fields) < 4:
                raise MeshParseError(line_no, f"vertex needs 3 coordinates: {raw!r}")
            try:
                verts.append([float(fields[1]), float(fields[2]), float(fields[3])])
            except ValueError as exc:
                raise MeshParseError(line_no, f"bad vertex coordinate: {exc}") from None
        elif tag == "f":
            if len(fields) < 4:
                raise MeshParseError(line_no, f"face needs >= 3 vertices: {raw!r}")
            ids = []
            for tok in fields[1:]:
                try:
                    i = int(tok.split("/")[0])
                except ValueError:
                    raise MeshParseError(line_no, f"bad face index {tok!r}") from None
                i = len(verts) + i if i < 0 else i - 1  # OBJ: 1-based, negatives relative
                if not 0 <= i < len(verts):
                    raise MeshParseError(line_no, f"face index {tok!r} out of range")
                ids.append(i)
            faces.extend([ids[0], ids[q], ids[q + 1]] for q in range(1, len(ids) - 1))
    return verts, faces


def load_mesh(source, transform=None) -> TriangleMesh:
    """OBJ subset (v/f records, fan triangulation); geometry.py:94-163."""
    if isinstance(source, bytes):
        text = source.decode("utf-8", errors="replace")
    elif isinstance(source, str) and "\n" not in source and source.endswith(".obj"):
        with open(source, "r") as fh:
            text = fh.read()
    elif hasattr(source, "read"):
        text = source.read()
        if isinstance(text, bytes):
            text = text.decode("utf-8", errors="replace")
    else:
        text = str(source)
    verts, faces = _parse_obj(text)
    if not faces:
        raise EmptyMeshError("OBJ contains no faces")
    vertices = np.array(verts, dtype=np.float64)
    if transform is not None:
        m = np.asarray(transform, dtype=np.float64)
        if m.shape != (3, 4):
            raise MeshError(f"transform must be 3x4, got {m.shape}")
        vertices = vertices @ m[:, :3].T + m[:, 3]
    mesh = make_mesh(vertices, np.array(faces, dtype=np.int32))
    log.info("loaded mesh: %d triangles kept, %d degenerate dropped, %d vertices",
             mesh.num_triangles, mesh.dropped, len(mesh.vertices))
    return mesh


def identity_transform():
    return np.hstack([np.eye(3), np.zeros((3, 1))])


@dataclass(frozen=True)
class BvhIndex:
    """Flat BVH (geometry.py:177-199) plus its packed device copy.

    The numpy fields are the reference's arrays (same tree, same order);
    `packed` is the device traversal buffer (64 B nodes + 128 B triangles).
    """

    mesh: TriangleMesh
    node_lo: np.ndarray
    node_hi: np.ndarray
    node_left: np.ndarray
    node_right: np.ndarray
    order: np.ndarray
    tri_a: np.ndarray
    tri_e1: np.ndarray
    tri_e2: np.ndarray
    tri_n: np.ndarray
    packed: torch.Tensor = dc_field(repr=False, compare=False, default=None)
    normals_dev: torch.Tensor = dc_field(repr=False, compare=False, default=None)
    # K6 search tree (binned SAH) in the packed device layout, and its node count
    search: torch.Tensor = dc_field(repr=False, compare=False, default=None)
    search_nodes: int = 0
    search_nodes4: int = 0  # > 0: BVH4 records (8 octant copies per node) appended to `search`
    search_stack4: int = 0  # > 0: stack entries its traversal can need (3 per level)

    @property
    def num_nodes(self):
        return len(self.node_left)

    @property
    def num_tris(self):
        return len(self.order)


def build_bvh(mesh: TriangleMesh) -> BvhIndex:
    """Median split over the longest node axis, stable ties, leaf <= 4."""
    if mesh.num_triangles == 0:
        raise EmptyMeshError("cannot build BVH over empty mesh")
    v, tris = mesh.vertices, mesh.triangles
    p0, p1, p2 = v[tris[:, 0]], v[tris[:, 1]], v[tris[:, 2]]
    tri_lo = np.ascontiguousarray(np.minimum(np.minimum(p0, p1), p2))
    tri_hi = np.ascontiguousarray(np.maximum(np.maximum(p0, p1), p2))
    T = len(tris)
    cap = 2 * T
    node_lo = np.empty((cap, 3), np.float64)
    node_hi = np.empty((cap, 3), np.float64)
    left = np.empty(cap, np.int32)
    right = np.empty(cap, np.int32)
    order = np.empty(T, np.int32)
    L = _lib.lib()
    n = L.rtsdf_bvh_build_host(_lib.host_ptr(tri_lo), _lib.host_ptr(tri_hi), T,
                               _lib.host_ptr(node_lo), _lib.host_ptr(node_hi),
                               _lib.host_ptr(left), _lib.host_ptr(right), _lib.host_ptr(order))
    if n < 0:
        raise EmptyMeshError(L.rtsdf_last_error().decode())
    node_lo, node_hi, left, right = node_lo[:n].copy(), node_hi[:n].copy(), left[:n].copy(), right[:n].copy()
    if tree_depth(left, right) >= 64:  # RTSDF_STACK (csrc/common.cuh)
        raise MeshError("BVH deeper than the traversal stack (64 levels)")
    a = np.ascontiguousarray(p0[order])
    e1 = np.ascontiguousarray(p1[order] - a)
    e2 = np.ascontiguousarray(p2[order] - a)
    tn = np.ascontiguousarray(mesh.normals[order])
    packed = upload_bvh(node_lo, node_hi, left, right, order, a, e1, e2, tn)
    # the K6 search tree (binned SAH): same triangles, any tree gives the same
    # brute-force-equivalent closest hit (csrc/trace.cuh)
    slo, shi = np.empty((cap, 3)), np.empty((cap, 3))
    sl, sr = np.empty(cap, np.int32), np.empty(cap, np.int32)
    so = np.empty(T, np.int32)
    ns = L.rtsdf_bvh_build_sah_host(_lib.host_ptr(tri_lo), _lib.host_ptr(tri_hi), T, SAH_MAX_LEAF,
                                    *[_lib.host_ptr(x) for x in (slo, shi, sl, sr, so)])
    if ns < 0:
        raise MeshError(L.rtsdf_last_error().decode())
    slo, shi, sl, sr = slo[:ns], shi[:ns], sl[:ns], sr[:ns]
    if tree_depth(sl, sr) >= 40:  # RTSDF_FAST_STACK (csrc/trace.cuh)
        raise MeshError("SAH BVH deeper than the traversal stack (40 levels)")
    sa = np.ascontiguousarray(p0[so])
    search = upload_bvh(slo, shi, sl, sr, so, sa, np.ascontiguousarray(p1[so] - sa),
                        np.ascontiguousarray(p2[so] - sa), np.ascontiguousarray(mesh.normals[so]))
    # 4-wide collapse of the search tree, appended after the packed layout
    n4 = 0
    if USE_BVH4:
        slo_c, shi_c = np.ascontiguousarray(slo), np.ascontiguousarray(shi)
        sl_c, sr_c = np.ascontiguousarray(sl), np.ascontiguousarray(sr)
        nodes4 = np.empty((8 * max(int(ns), 1), 128), dtype=np.uint8)  # 8 octant records per node
        n4 = int(L.rtsdf_bvh4_collapse_host(*[_lib.host_ptr(x) for x in (slo_c, shi_c, sl_c, sr_c)],
                                            int(ns), _lib.host_ptr(nodes4), nodes4.shape[0]))
        stack4 = 3 * _depth4(nodes4[:n4]) if n4 > 0 else 0
        if n4 > 0 and stack4 < 40:  # RTSDF_FAST_STACK pushes
            search = torch.cat([search, to_device(nodes4[:n4].reshape(-1))])
        else:
            n4, stack4 = 0, 0
    else:
        stack4 = 0
    return BvhIndex(mesh, node_lo, node_hi, left, right, order, a, e1, e2, tn, packed,
                    to_device(mesh.normals), search, int(ns), n4, stack4)


class DeviceBvh:
    """The K6 search tree built ON THE DEVICE (rtsdf_lbvh_build): the per-frame
    tree of dynamic scenes (the reference rebuilds its tree in Python every
    animated frame, scenes.py:56-93 -> geometry.py:202-267).  Same closest
    hits as any other tree (geometry.py:3-6).  Rigid or deforming motion with
    an unchanged triangle list refits the previous topology (boxes and
    triangle records only); `rebuild_every` frames force a fresh build.

    The reference-order tree (the validation APIs: ray_query fast=False,
    exact_distance, reference_visibility) is built on the host on first use.
    """

    device_built = True
    search_nodes4 = 0
    search_stack4 = 0

    def __init__(self, mesh: TriangleMesh, verts_dev, tris_dev, state: dict | None = None,
                 rebuild_every: int = 8):
        if mesh.num_triangles == 0:
            raise EmptyMeshError("cannot build BVH over empty mesh")
        L = _lib.lib()
        T = int(mesh.num_triangles)
        self.mesh = mesh
        self.num_tris = T
        self.search_nodes = int(L.rtsdf_lbvh_nodes(T))
        self.normals_dev = to_device(mesh.normals)
        dev = self.normals_dev.device
        st = state if state is not None else {}
        if st.get("T") != T:
            st.clear()
            st.update(T=T, ws=torch.empty(int(L.rtsdf_lbvh_ws_bytes(T)), dtype=torch.uint8, device=dev),
                      bufs=[None, None], flip=0, age=None,
                      depth=torch.zeros(1, dtype=torch.int32, device=dev), checked=False)
        refit = st["age"] is not None and st["age"] < rebuild_every - 1
        st["flip"] ^= 1
        nbytes = int(L.rtsdf_bvh_packed_bytes(self.search_nodes, T))
        if st["bufs"][st["flip"]] is None:
            st["bufs"][st["flip"]] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.search = st["bufs"][st["flip"]]  # ping-pong: the previous view's tree stays valid
        _lib.check(L.rtsdf_lbvh_build(_lib.ptr(verts_dev), _lib.ptr(tris_dev), _lib.ptr(self.normals_dev),
                                      T, 1 if refit else 0, _lib.ptr(self.search), nbytes,
                                      _lib.ptr(st["ws"]), st["ws"].numel(), _lib.ptr(st["depth"]),
                                      _lib.stream()), "lbvh_build")
        st["age"] = st["age"] + 1 if refit else 0
        if not st["checked"]:  # once per scene: the traversal stack bounds the depth
            if int(st["depth"].item()) >= 40:  # RTSDF_FAST_STACK (csrc/trace.cuh)
                raise MeshError("device BVH deeper than the traversal stack (40 levels)")
            st["checked"] = True
        self.refit = refit
        self._ref = None

    def reference_tree(self) -> "BvhIndex":
        if self._ref is None:
            self._ref = build_bvh(self.mesh)
        return self._ref

    def __getattr__(self, name):
        # node_lo / order / packed / num_nodes / ...: the reference-order tree
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.reference_tree(), name)


def _depth4(nodes4: np.ndarray) -> int:
    child = nodes4.view(np.int32).reshape(-1, 32)[:, 24:28]
    frontier, depth = np.array([0]), 0
    while len(frontier):
        depth += 1
        c = child[frontier].reshape(-1)
        frontier = c[(c >= 0) & (c != 0x7FFFFFFF)]
    return depth


def tree_depth(left: np.ndarray, right: np.ndarray) -> int:
    """Number of levels of the flat tree (leaves: left < 0)."""
    frontier = np.array([0], dtype=np.int64)
    depth = 0
    while len(frontier):
        depth += 1
        internal = frontier[left[frontier] >= 0]
        frontier = np.concatenate([left[internal], right[internal]]).astype(np.int64)
    return depth


def upload_bvh(node_lo, node_hi, left, right, order, a, e1, e2, tn) -> torch.Tensor:
    """Upload the flat arrays and pack them into the device traversal layout."""
    n, T = len(left), len(order)
    L = _lib.lib()
    packed = torch.empty(int(L.rtsdf_bvh_packed_bytes(n, T)), dtype=torch.uint8,
                         device=to_device(np.zeros(1)).device)
    dev = [to_device(x) for x in (node_lo, node_hi, left, right, order, a, e1, e2, tn)]
    _lib.check(L.rtsdf_bvh_pack(*[_lib.ptr(x) for x in dev], n, T, _lib.ptr(packed),
                                _lib.stream()), "bvh_pack")
    torch.cuda.current_stream().synchronize()  # the staging tensors die here
    return packed


@dataclass(frozen=True)
class RayHit:
    hit: bool
    t: float = 0.0
    triangle: int = -1
    facing: int = FACING_NONE


def ray_query_many(bvh: BvhIndex, origins, directions, t_max=np.inf, fast=False):
    """Batched closest-hit queries: (t, id, facing) arrays; t < 0 = miss.

    fast=False: the reference's traversal order verbatim (fp64);
    fast=True: the refinement's K6 search (brute-force-equivalent result).
    """
    o = to_device(np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3))
    d = to_device(np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3))
    n = o.shape[0]
    t = torch.empty(n, dtype=torch.float64, device=o.device)
    ids = torch.empty(n, dtype=torch.int32, device=o.device)
    fac = torch.empty(n, dtype=torch.int32, device=o.device)
    buf, nn = (bvh.search, bvh.search_nodes) if fast else (bvh.packed, bvh.num_nodes)
    mode = (2 if bvh.search_nodes4 > 0 and fast != "binary" else 1) if fast else 0
    _lib.check(_lib.lib().rtsdf_ray_query(_lib.ptr(buf), nn, bvh.num_tris,
                                          mode, _lib.ptr(o),
                                          _lib.ptr(d), n, float(t_max), _lib.ptr(t),
                                          _lib.ptr(ids), _lib.ptr(fac), _lib.stream()),
               "ray_query")
    return to_numpy(t), to_numpy(ids), to_numpy(fac)


def ray_query(bvh: BvhIndex, origin, direction, t_max=np.inf) -> RayHit:
    """Nearest intersection with t <= t_max (geometry.py:395-410)."""
    d = np.asarray(direction, dtype=np.float64)
    norm = np.linalg.norm(d)
    if abs(norm - 1.0) > 1e-6:
        raise ValueError(f"direction must be unit length, |d| = {norm}")
    t, ids, fac = ray_query_many(bvh, np.asarray(origin, dtype=np.float64)[None], d[None], t_max)
    if t[0] < 0.0:
        return RayHit(False)
    return RayHit(True, float(t[0]), int(ids[0]), int(fac[0]))


# ---------------------------------------------------------------------------
# Exact point-to-mesh distance (validation oracle)
# ---------------------------------------------------------------------------

def exact_distance_many(bvh: BvhIndex, points) -> np.ndarray:
    """Exact unsigned point-to-mesh distance per point (geometry.py:588-594):
    Eberly's region tests over the reference-order BVH in the reference's
    traversal order and pruning rule -- bit-exact with the reference."""
    pts = to_device(np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3))
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=pts.device)
    _lib.check(_lib.lib().rtsdf_exact_distance(_lib.ptr(bvh.packed), bvh.num_nodes, _lib.ptr(pts),
                                               pts.shape[0], _lib.ptr(out), _lib.stream()),
               "exact_distance")
    return to_numpy(out)


def exact_distance(bvh: BvhIndex, point) -> float:
    """Exact unsigned point-to-mesh distance (geometry.py:579-585)."""
    return float(exact_distance_many(bvh, np.asarray(point, dtype=np.float64)[None])[0])


__all__ = ["DEGENERATE_AREA", "FACING_NONE", "FACING_FRONT", "FACING_BACK", "MeshError",
           "MeshParseError", "EmptyMeshError", "TriangleMesh", "make_mesh", "load_mesh",
           "identity_transform", "BvhIndex", "DeviceBvh", "build_bvh", "RayHit", "ray_query",
           "ray_query_many", "to_numpy", "exact_distance", "exact_distance_many"]
