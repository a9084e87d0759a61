"""ctypes front end of the CPU parity oracle (oracle/rtsdf_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.
numpy in, numpy out, same array layouts as the reference (`sdfshadow`):
C-order (nx, ny, nz), int32 linear seeds, fp64 geometry.  Each wrapper names
the reference function it restates.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "librtsdf_oracle.so"

P, I, I64, U64, D = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
_SIGS = {
    "oracle_num_threads": (I, []),
    "oracle_set_threads": (None, [I]),
    "oracle_tri_box_overlap": (I, [P, P, P, P, P]),
    "oracle_voxelize": (None, [P, P, P, I64, P, D, D, D, I, I, I, P]),
    "oracle_jfa_init": (I64, [P, I64, P]),
    "oracle_jfa_step": (None, [P, P, I, I, I, I, D, D, D]),
    "oracle_jfa_step_range": (None, [P, P, I, I, I, I, D, D, D, I, I]),
    "oracle_seeds_to_sdf": (None, [P, P, I, I, I, D, D, D, D]),
    "oracle_trilinear": (D, [P, I, I, I, D, D, D, D, D, D, D, D, D]),
    "oracle_resample_mask": (None, [P, I, I, I, D, D, D, D, D, D, D, D, D, I, I, I, D, P, P]),
    "oracle_stream_key": (U64, [U64, U64, U64]),
    "oracle_uniform": (D, [U64, U64]),
    "oracle_unit_sphere_dir": (None, [U64, U64, P]),
    "oracle_dir_table": (None, [U64, P, I64, I64, I, P]),
    "oracle_libm_sincos": (None, [P, I64, P, P]),
    "oracle_bvh_build": (I64, [P, P, I64, P, P, P, P, P]),
    "oracle_ray_query": (None, [P, P, P, P, P, P, P, P, P, P, P, I64, D, P, P, P]),
    "oracle_ray_brute": (None, [P, P, P, P, P, P, P, P, P, I64, P, P, I64, D, P, P, P]),
    "oracle_sample_masked": (None, [P, P, P, P, P, P, P, P, P, P, I64, D, D, D, D, D, D, I, I, I,
                                    U64, I64, D, P, P, P, P]),
    "oracle_update_fine": (None, [P, P, P, P, I64, P, P, P, P, I64, P, P, P, D, P]),
    "oracle_march": (I, [P, I, I, I, D, D, D, D, D, D, D, D, D, D, D, D, D, I, D, D, D, D, P, P,
                         P]),
    "oracle_occlusion": (None, [P, I, I, I, D, D, D, D, D, D, P, P, P, I, I, D, D, D, D, I, D, D,
                                D, D, D, I, U64, P]),
    "oracle_gbuffer": (None, [P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, D, D, I, I, P, P, P,
                              P]),
    "oracle_exact_distance_many": (None, [P, P, P, P, P, P, P, P, P, P, I64, P]),
    "oracle_reference_visibility": (None, [P, P, P, P, P, P, P, P, P, P, P, P, I, I, D, D, D, D, D,
                                           D, D, D, D, D, I, U64, P]),
}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        src = HERE / "rtsdf_oracle.c"
        if not LIB.exists() or (src.exists() and src.stat().st_mtime > LIB.stat().st_mtime):
            build()
        h = C.CDLL(str(LIB))
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def set_threads(n: int):
    lib().oracle_set_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ------------------------------------------------------------------ voxel.py
def voxelize(verts, tris, dims, bounds):
    """voxel.py:150-181 -> occupancy uint8 (nx, ny, nz); raises on OOB."""
    verts = _c(verts, np.float64)
    tris = np.asarray(tris)
    p0, p1, p2 = (_c(verts[tris[:, c]], np.float64) for c in range(3))
    lo = _c(bounds[0], np.float64)
    hi = _c(bounds[1], np.float64)
    tlo = np.minimum(np.minimum(p0, p1), p2)
    thi = np.maximum(np.maximum(p0, p1), p2)
    bad = np.any(tlo < lo, axis=1) | np.any(thi > hi, axis=1)
    if bad.any():
        raise ValueError(f"triangles outside voxel bounds: {np.nonzero(bad)[0].tolist()[:16]}")
    dims = tuple(int(n) for n in dims)
    occ = np.zeros(dims, dtype=np.uint8)
    h = (hi - lo) / np.array(dims, dtype=np.float64)
    lib().oracle_voxelize(_p(p0), _p(p1), _p(p2), len(p0), _p(lo), h[0], h[1], h[2], *dims, _p(occ))
    return occ


# -------------------------------------------------------------------- jfa.py
def jfa_init(occ):
    seed = np.empty(occ.shape, dtype=np.int32)
    n = lib().oracle_jfa_init(_p(_c(occ, np.uint8)), occ.size, _p(seed))
    if n == 0:
        raise ValueError("voxel grid has no occupied cells")
    return seed


def jfa_offsets(dims):
    n = 1
    while n < max(dims):
        n *= 2
    out, s = [], n // 2
    while s >= 1:
        out.append(s)
        s //= 2
    return out


def jfa_step(seed, offset, h):
    seed = _c(seed, np.int32)
    dst = np.empty_like(seed)
    lib().oracle_jfa_step(_p(seed), _p(dst), *seed.shape, int(offset), float(h[0]), float(h[1]),
                          float(h[2]))
    return dst


def jfa_run(occ, h):
    seed = jfa_init(occ)
    for off in jfa_offsets(seed.shape):
        seed = jfa_step(seed, off, h)
    return seed


def seeds_to_sdf(seed, h, beta=0.0):
    seed = _c(seed, np.int32)
    out = np.empty(seed.shape, dtype=np.float32)
    lib().oracle_seeds_to_sdf(_p(seed), _p(out), *seed.shape, float(h[0]), float(h[1]),
                              float(h[2]), float(beta))
    return out


# -------------------------------------------------------- field / raysample
def trilinear(data, lo, h, p):
    data = _c(data, np.float32)
    return lib().oracle_trilinear(_p(data), *data.shape, *map(float, lo), *map(float, h),
                                  *map(float, p))


def resample_mask(coarse, clo, chi, fine_dims, d):
    """raysample.py:108-119 -> (c_fine f32, mask bool)."""
    coarse = _c(coarse, np.float32)
    clo = np.asarray(clo, np.float64)
    chi = np.asarray(chi, np.float64)
    ch = (chi - clo) / np.array(coarse.shape, dtype=np.float64)
    fine_dims = tuple(int(n) for n in fine_dims)
    fh = (chi - clo) / np.array(fine_dims, dtype=np.float64)
    out = np.empty(fine_dims, np.float32)
    mask = np.empty(fine_dims, np.uint8)
    lib().oracle_resample_mask(_p(coarse), *coarse.shape, *map(float, clo), *map(float, ch),
                               *map(float, fh), *fine_dims, float(d), _p(out), _p(mask))
    return out, mask.astype(bool)


def stream_key(seed, stream, tick):
    return int(lib().oracle_stream_key(int(seed) & (2**64 - 1), int(stream) & (2**64 - 1),
                                       int(tick) & (2**64 - 1)))


def uniform(key, counter):
    return float(lib().oracle_uniform(int(key), int(counter)))


def dir_table(seed, idx, frame, x):
    """(M, x, 3) directions keyed like raysample.py:170 (glibc cos/sin)."""
    idx = _c(idx, np.int64)
    out = np.empty((len(idx), int(x), 3), np.float64)
    lib().oracle_dir_table(int(seed) & (2**64 - 1), _p(idx), len(idx), int(frame), int(x), _p(out))
    return out


def libm_sincos(x):
    """The host libm's (sin, cos) of every element (the reference's rng.py:53 calls)."""
    x = _c(x, np.float64)
    s, c = np.empty_like(x), np.empty_like(x)
    lib().oracle_libm_sincos(_p(x), x.size, _p(s), _p(c))
    return s, c


# ----------------------------------------------------------------- geometry
def face_normals(verts, tris):
    a = verts[tris[:, 0]]
    n = np.cross(verts[tris[:, 1]] - a, verts[tris[:, 2]] - a)
    return n / np.linalg.norm(n, axis=1)[:, None]


def bvh_build(verts, tris, normals=None):
    """geometry.py:202-267 -> dict of the flat BVH arrays."""
    verts = _c(verts, np.float64)
    tris = np.asarray(tris)
    p0, p1, p2 = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    tri_lo = _c(np.minimum(np.minimum(p0, p1), p2), np.float64)
    tri_hi = _c(np.maximum(np.maximum(p0, p1), p2), np.float64)
    T = len(tris)
    node_lo = np.empty((2 * T, 3)); node_hi = np.empty((2 * T, 3))
    left = np.empty(2 * T, np.int32); right = np.empty(2 * T, np.int32)
    order = np.empty(T, np.int32)
    n = lib().oracle_bvh_build(_p(tri_lo), _p(tri_hi), T, _p(node_lo), _p(node_hi), _p(left),
                               _p(right), _p(order))
    if normals is None:
        normals = face_normals(verts, tris)
    a = _c(p0[order], np.float64)
    return dict(node_lo=node_lo[:n].copy(), node_hi=node_hi[:n].copy(), node_left=left[:n].copy(),
                node_right=right[:n].copy(), order=order, tri_a=a, tri_e1=_c(p1[order] - a, np.float64),
                tri_e2=_c(p2[order] - a, np.float64), tri_n=_c(np.asarray(normals)[order], np.float64))


def _bvh_args(b):
    return [_p(b[k]) for k in ("node_lo", "node_hi", "node_left", "node_right", "order", "tri_a",
                               "tri_e1", "tri_e2", "tri_n")]


def ray_query(b, origins, dirs, t_max=np.inf):
    o = _c(origins, np.float64).reshape(-1, 3)
    d = _c(dirs, np.float64).reshape(-1, 3)
    n = len(o)
    t = np.empty(n); ids = np.empty(n, np.int32); fac = np.empty(n, np.int32)
    lib().oracle_ray_query(*_bvh_args(b), _p(o), _p(d), n, float(t_max), _p(t), _p(ids), _p(fac))
    return t, ids, fac


def ray_brute(b, origins, dirs, t_max=np.inf):
    """Closest hit over every triangle (no BVH): the traversal contract."""
    o = _c(origins, np.float64).reshape(-1, 3)
    d = _c(dirs, np.float64).reshape(-1, 3)
    n = len(o)
    t = np.empty(n); ids = np.empty(n, np.int32); fac = np.empty(n, np.int32)
    lib().oracle_ray_brute(*_bvh_args(b), len(b["order"]), _p(o), _p(d), n, float(t_max), _p(t),
                           _p(ids), _p(fac))
    return t, ids, fac


def sample_masked(b, idx, lo, fh, fine_dims, x, seed, frame, t_max, dirs=None):
    """raysample.py:155-176 -> (min t, front, back) per masked texel."""
    idx = _c(idx, np.int64)
    M = len(idx)
    smin = np.empty(M); sf = np.empty(M, np.int32); sb = np.empty(M, np.int32)
    if dirs is not None:
        dirs = _c(dirs, np.float64)
    lib().oracle_sample_masked(*_bvh_args(b), _p(idx), M, *map(float, lo), *map(float, fh),
                               int(fine_dims[1]), int(fine_dims[2]), int(x), int(seed) & (2**64 - 1),
                               int(frame), float(t_max), _p(dirs), _p(smin), _p(sf), _p(sb))
    return smin, sf, sb


def empty_accum(fine_dims):
    return dict(min_dist=np.full(fine_dims, np.inf, np.float32), front=np.zeros(fine_dims, np.int32),
                back=np.zeros(fine_dims, np.int32), mask=np.zeros(fine_dims, bool))


def update_fine(prev, coarse, clo, chi, b, x, d, alpha, seed, frame, accum=None, t_max=None,
                dirs=None):
    """raysample.py:247-305 on numpy arrays; returns (fine f32, accum dict, idx)."""
    prev = _c(prev, np.float32)
    fine_dims = prev.shape
    if accum is None:
        accum = empty_accum(fine_dims)
    clo = np.asarray(clo, np.float64); chi = np.asarray(chi, np.float64)
    c_fine, mask_new = resample_mask(coarse, clo, chi, fine_dims, d)
    idx = np.flatnonzero(mask_new.ravel()).astype(np.int64)
    if t_max is None:
        t_max = float(np.linalg.norm(chi - clo))
    fh = (chi - clo) / np.array(fine_dims, dtype=np.float64)
    if x > 0 and len(idx):
        smin, sf, sb = sample_masked(b, idx, clo, fh, fine_dims, x, seed, frame, t_max, dirs)
    else:
        smin = np.full(len(idx), np.inf); sf = np.zeros(len(idx), np.int32); sb = np.zeros(len(idx), np.int32)
    out = c_fine.copy()
    mo = _c(accum["mask"], np.uint8)
    mn = _c(mask_new, np.uint8)
    lib().oracle_update_fine(_p(prev), _p(c_fine), _p(mo), _p(mn), prev.size, _p(accum["min_dist"]),
                             _p(accum["front"]), _p(accum["back"]), _p(idx), len(idx), _p(smin),
                             _p(sf), _p(sb), float(alpha), _p(out))
    accum["mask"] = mask_new
    return out, accum, idx


# ---------------------------------------------------------- raymarch/render
def march(data, lo, h, o, d, eps, max_iter, max_step, t_max, t0, k):
    data = _c(data, np.float32)
    t = C.c_double(); it = C.c_int(); mt = C.c_double()
    st = lib().oracle_march(_p(data), *data.shape, *map(float, lo), *map(float, h), *map(float, o),
                            *map(float, d), float(eps), int(max_iter), float(max_step), float(t_max),
                            float(t0), float(k), C.byref(t), C.byref(it), C.byref(mt))
    return st, t.value, it.value, mt.value


def occlusion(data, lo, h, g_pos, g_nrm, g_cov, light, eps, max_iter, max_step, t_max, k, jitter,
              offset, draws, seed):
    data = _c(data, np.float32)
    g_pos = _c(g_pos, np.float64); g_nrm = _c(g_nrm, np.float64); g_cov = _c(g_cov, np.uint8)
    hgt, wid = g_cov.shape
    out = np.empty((hgt, wid))
    lib().oracle_occlusion(_p(data), *data.shape, *map(float, lo), *map(float, h), _p(g_pos),
                           _p(g_nrm), _p(g_cov), hgt, wid, *map(float, light), float(eps),
                           int(max_iter), float(max_step), float(t_max), float(k), float(jitter),
                           float(offset), int(draws), int(seed) & (2**64 - 1), _p(out))
    return out


def gbuffer(b, normals_orig, albedo_orig, pos, fwd, right, up, half_w, half_h, width, height):
    normals_orig = _c(normals_orig, np.float64)
    albedo_orig = _c(albedo_orig, np.float32)
    vec = [_c(v, np.float64) for v in (pos, fwd, right, up)]
    out_pos = np.zeros((height, width, 3)); out_nrm = np.zeros((height, width, 3))
    out_alb = np.zeros((height, width, 3), np.float32); out_cov = np.zeros((height, width), np.uint8)
    lib().oracle_gbuffer(*_bvh_args(b), _p(normals_orig), _p(albedo_orig), *[_p(v) for v in vec],
                         float(half_w), float(half_h), int(width), int(height), _p(out_pos),
                         _p(out_nrm), _p(out_alb), _p(out_cov))
    return out_pos, out_nrm, out_alb, out_cov.astype(bool)


# ------------------------------------------------------------ whole frames
class HybridOracle:
    """FramePipeline.advance (pipeline.py:109-160) on the CPU oracle."""

    def __init__(self, verts, tris, normals, bounds, coarse_dims, fine_dims, x=32, d=0.1,
                 alpha=0.95, seed=0, beta=0.0, mesh_fn=None):
        # mesh_fn(frame) -> (verts, tris, normals): animated scenes re-voxelize
        # and rebuild the BVH every frame (pipeline.py:116-119, scenes.py:56-93)
        self.mesh_fn = mesh_fn
        self.verts, self.tris, self.normals = verts, tris, normals
        self.lo = np.asarray(bounds[0], np.float64)
        self.hi = np.asarray(bounds[1], np.float64)
        self.coarse_dims = tuple(coarse_dims)
        self.fine_dims = tuple(fine_dims)
        self.x, self.d, self.alpha, self.seed, self.beta = x, d, alpha, seed, beta
        self.bvh = bvh_build(verts, tris, normals)
        self.fine = None
        self.accum = None
        self.frame = 0

    def advance(self, dirs_fn=None):
        if self.mesh_fn is not None:
            self.verts, self.tris, self.normals = self.mesh_fn(self.frame)
            self.bvh = bvh_build(self.verts, self.tris, self.normals)
        occ = voxelize(self.verts, self.tris, self.coarse_dims, (self.lo, self.hi))
        h = (self.hi - self.lo) / np.array(self.coarse_dims, dtype=np.float64)
        seeds = jfa_run(occ, h)
        coarse = seeds_to_sdf(seeds, h, self.beta)
        if self.fine is None:
            self.fine = resample_mask(coarse, self.lo, self.hi, self.fine_dims, np.inf)[0]
            self.accum = empty_accum(self.fine_dims)
        dirs = None
        if dirs_fn is not None:
            _, mask = resample_mask(coarse, self.lo, self.hi, self.fine_dims, self.d)
            dirs = dirs_fn(np.flatnonzero(mask.ravel()), self.frame)
        self.fine, self.accum, idx = update_fine(self.fine, coarse, self.lo, self.hi, self.bvh,
                                                 self.x, self.d, self.alpha, self.seed, self.frame,
                                                 self.accum, dirs=dirs)
        self.frame += 1
        return dict(occ=occ, seeds=seeds, coarse=coarse, fine=self.fine, idx=idx)


# ------------------------------------------------------ validation oracles
def exact_distance_many(b, points):
    """geometry.py:588-594: exact unsigned point-to-mesh distance per point."""
    pts = _c(points, np.float64).reshape(-1, 3)
    out = np.empty(len(pts))
    lib().oracle_exact_distance_many(*_bvh_args(b), _p(pts), len(pts), _p(out))
    return out


def cone_basis(light_unit):
    """render.py:237-241 (t1, t2) around the light direction, numpy as the reference."""
    l = np.asarray(light_unit, dtype=np.float64)
    up = np.array([0.0, 1.0, 0.0]) if abs(l[1]) < 0.9 else np.array([1.0, 0.0, 0.0])
    t1 = np.cross(l, up)
    t1 /= np.linalg.norm(t1)
    t2 = np.cross(l, t1)
    return t1, t2


def reference_visibility(b, g_pos, g_nrm, g_cov, light_unit, angular_radius, spp, seed):
    """render.py:195-254: cone-sampled shadow-ray visibility per pixel."""
    import math

    pos = _c(g_pos, np.float64)
    nrm = _c(g_nrm, np.float64)
    cov = _c(g_cov, np.uint8)
    h, w = cov.shape
    l = np.asarray(light_unit, dtype=np.float64)
    t1, t2 = cone_basis(l)
    out = np.empty((h, w))
    lib().oracle_reference_visibility(*_bvh_args(b), _p(pos), _p(nrm), _p(cov), h, w, *map(float, l),
                                      *map(float, t1), *map(float, t2),
                                      math.tan(angular_radius), int(spp), int(seed), _p(out))
    return out


def jfa_step_range(src, dst, offset, h, i0, i1):
    lib().oracle_jfa_step_range(_p(src), _p(dst), *src.shape, int(offset), float(h[0]),
                                float(h[1]), float(h[2]), int(i0), int(i1))


class CpuFrameRunner:
    """Whole C3-style frames on the CPU oracle, timed end to end: the
    reference arm / cpu_baseline of bench.py.  Each step is one complete
    FramePipeline.advance(render=True) (pipeline.py:109-160): voxelize, the
    full JFA schedule, seeds -> SDF, resample + mask, every masked texel's x
    rays, the Eq. 1 update with the temporal state carried frame to frame,
    the G-buffer and the soft-shadow march -- no sampling, no extrapolation.
    The BVH of the static scene is built once, as the reference's memoised
    SceneView does (scenes.py:56-63)."""

    def __init__(self, mesh, albedo, bounds, dims, camera, light_unit, light_angle, x=32, d=0.1,
                 alpha=0.95, bias=0.01):
        import math

        self.mesh, self.albedo = mesh, np.ascontiguousarray(albedo, np.float32)
        self.lo = np.asarray(bounds[0], np.float64)
        self.hi = np.asarray(bounds[1], np.float64)
        self.dims = tuple(dims)
        self.bias = bias
        self.h = (self.hi - self.lo) / np.array(dims, dtype=np.float64)
        self.H = HybridOracle(mesh.vertices, mesh.triangles, mesh.normals, bounds, dims, dims, x=x,
                              d=d, alpha=alpha)
        pos, fwd, right, up = camera.basis()
        half_h = math.tan(math.radians(camera.vfov_deg) * 0.5)
        self.cam = (pos, fwd, right, up, half_h * camera.width / camera.height, half_h,
                    camera.width, camera.height)
        self.light = np.asarray(light_unit, np.float64)
        self.k = 1.0 / math.tan(light_angle)
        self.eps = float(max(self.h))
        self.t_max = float(np.linalg.norm(self.hi - self.lo))
        self.threads = num_threads()

    def step(self) -> float:
        """One full frame; returns its wall time in seconds."""
        import time

        t = time.perf_counter()
        self.H.advance()
        gp, gn, _, gc = gbuffer(self.H.bvh, self.mesh.normals, self.albedo, *self.cam)
        self.occ = occlusion(self.H.fine - np.float32(self.bias), self.lo, self.h, gp, gn, gc,
                             self.light, self.eps, 256, 0.05, self.t_max, self.k, 1.0,
                             2 * self.eps + self.bias, 1, 0)
        return time.perf_counter() - t
