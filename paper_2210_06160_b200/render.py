"""G-buffer, soft-shadow occlusion image and compose -- mirrors sdfshadow.render.

`occlusion_image` is the batched soft-shadow query that consumes the hybrid
field (render.py:155-175, K8 rtsdf_occlusion).  `rasterize_gbuffer` is the
G-buffer primary-visibility pass (render.py:112-128), traced on the device
through the same BVH kernel as the refinement.  Image I/O stays on the host.
`reference_visibility` / `reference_render` are the reference's distributed
ray-traced ground truth (render.py:195-264) on the device -- a validation
oracle for image-quality checks.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import device, to_device, to_numpy
from .field import DistanceField
from .raymarch import MarchParams


@dataclass(frozen=True)
class Camera:
    position: tuple
    look_at: tuple
    up: tuple = (0.0, 1.0, 0.0)
    vfov_deg: float = 45.0
    width: int = 320
    height: int = 240

    def basis(self):
        pos = np.asarray(self.position, dtype=np.float64)
        fwd = np.asarray(self.look_at, dtype=np.float64) - pos
        fwd /= np.linalg.norm(fwd)
        right = np.cross(fwd, np.asarray(self.up, dtype=np.float64))
        right /= np.linalg.norm(right)
        up = np.cross(right, fwd)
        return pos, fwd, right, up


@dataclass(frozen=True)
class DirectionalLight:
    direction: tuple
    angular_radius: float = 0.1

    def unit(self):
        d = np.asarray(self.direction, dtype=np.float64)
        return d / np.linalg.norm(d)


@dataclass(frozen=True)
class DiscLight:
    center: tuple
    radius: float
    normal: tuple = (0.0, -1.0, 0.0)


@dataclass
class GBuffer:
    position: torch.Tensor  # (H, W, 3) float64
    normal: torch.Tensor    # (H, W, 3) float64
    albedo: torch.Tensor    # (H, W, 3) float32
    coverage: torch.Tensor  # (H, W) bool

    @property
    def shape(self):
        return tuple(int(n) for n in self.coverage.shape)

    @classmethod
    def empty(cls, height, width):
        dev = device()
        return cls(torch.zeros((height, width, 3), dtype=torch.float64, device=dev),
                   torch.zeros((height, width, 3), dtype=torch.float64, device=dev),
                   torch.zeros((height, width, 3), dtype=torch.float32, device=dev),
                   torch.zeros((height, width), dtype=torch.bool, device=dev))


def camera_setup(camera: Camera):
    pos, fwd, right, up = camera.basis()
    half_h = math.tan(math.radians(camera.vfov_deg) * 0.5)
    half_w = half_h * camera.width / camera.height
    cam = (_lib.D * 12)(*pos, *fwd, *right, *up)
    return cam, half_w, half_h


def launch_gbuffer(view, camera: Camera, gb: GBuffer, cam_setup=None):
    cam, half_w, half_h = cam_setup or camera_setup(camera)
    bvh = view.bvh
    # device-built (dynamic-scene) trees carry only the search layout
    fast = getattr(bvh, "device_built", False)
    buf, nn = (bvh.search, bvh.search_nodes) if fast else (bvh.packed, bvh.num_nodes)
    _lib.check(_lib.lib().rtsdf_gbuffer(
        _lib.ptr(buf), nn, bvh.num_tris, 1 if fast else 0, _lib.ptr(bvh.normals_dev),
        _lib.ptr(view.albedo_dev),
        cam, half_w, half_h, camera.width, camera.height, _lib.ptr(gb.position),
        _lib.ptr(gb.normal), _lib.ptr(gb.albedo), _lib.ptr(gb.coverage), _lib.stream()),
        "gbuffer")


def rasterize_gbuffer(view, camera: Camera) -> GBuffer:
    """Primary visibility by closest-hit ray casting; deterministic."""
    gb = GBuffer.empty(camera.height, camera.width)
    launch_gbuffer(view, camera, gb)
    return gb


def launch_occlusion(gbuffer: GBuffer, fld: DistanceField, light_unit, params: MarchParams,
                     draws, seed, out, sample_bias: float = 0.0, rows=None):
    """sample_bias: shade `fld` biased by that much (apply_bias fused, f32).
    rows = (row0, nrows): shade only that band of the image (pixel-sharded DL)."""
    h, w = gbuffer.shape
    row0, nrows = rows if rows is not None else (0, h)
    nx, ny, nz = fld.dims
    offset = 2.0 * params.epsilon + (fld.bias + sample_bias)  # render.py:165
    _lib.check(_lib.lib().rtsdf_occlusion(
        _lib.ptr(fld.data), nx, ny, nz, (_lib.D * 3)(*fld.lo), (_lib.D * 3)(*fld.cell_size),
        _lib.ptr(gbuffer.position), _lib.ptr(gbuffer.normal), _lib.ptr(gbuffer.coverage), h, w,
        int(row0), int(nrows), (_lib.D * 3)(*light_unit), float(params.epsilon),
        int(params.max_iterations),
        float(params.max_step), float(params.t_max), params.cone_k, float(params.jitter),
        float(offset), max(1, int(draws)), int(seed) & 0xFFFFFFFFFFFFFFFF,
        float(np.float32(sample_bias)), _lib.ptr(out), _lib.stream()), "occlusion")


def occlusion_image(gbuffer: GBuffer, fld: DistanceField, light: DirectionalLight,
                    params: MarchParams, draws=1, seed=0) -> torch.Tensor:
    """Per-pixel soft-shadow occlusion toward the light (H, W) float64."""
    out = torch.empty(gbuffer.shape, dtype=torch.float64, device=fld.data.device)
    launch_occlusion(gbuffer, fld, light.unit(), params, draws, seed, out)
    return out


def launch_compose(gbuffer: GBuffer, occ: torch.Tensor, light_unit, background, out):
    h, w = gbuffer.shape
    _lib.check(_lib.lib().rtsdf_compose(
        _lib.ptr(gbuffer.normal), _lib.ptr(gbuffer.albedo), _lib.ptr(gbuffer.coverage),
        _lib.ptr(occ), h, w, (_lib.D * 3)(*light_unit), (_lib.D * 3)(*background), _lib.ptr(out),
        _lib.stream()), "compose")


def compose(gbuffer: GBuffer, occlusion, light: DirectionalLight,
            background=(0.05, 0.07, 0.10)) -> torch.Tensor:
    occ = to_device(occlusion, torch.float64)
    out = torch.empty(gbuffer.shape + (3,), dtype=torch.float32, device=occ.device)
    launch_compose(gbuffer, occ, light.unit(), background, out)
    return out


def shade(gbuffer: GBuffer, fld: DistanceField, light: DirectionalLight, params: MarchParams,
          draws=1, seed=0, background=(0.05, 0.07, 0.10)) -> torch.Tensor:
    occ = occlusion_image(gbuffer, fld, light, params, draws=draws, seed=seed)
    return compose(gbuffer, occ, light, background)


def compare(image_a, image_b, mask=None) -> dict:
    a = np.asarray(to_numpy(image_a), dtype=np.float64)
    b = np.asarray(to_numpy(image_b), dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"image dims differ: {a.shape} vs {b.shape}")
    diff = a - b
    if mask is not None:
        m = np.asarray(to_numpy(mask), dtype=bool)
        if m.shape != a.shape[: m.ndim]:
            raise ValueError("mask dims do not match image")
        diff = diff[m]
    if diff.size == 0:
        raise ValueError("empty comparison region")
    return {"rmse": float(np.sqrt(np.mean(diff ** 2))), "mae": float(np.mean(np.abs(diff))),
            "max": float(np.max(np.abs(diff)))}


def write_pfm(path, image):
    img = np.asarray(to_numpy(image), dtype=np.float32)
    if img.ndim == 2:
        header = b"Pf\n"
        img = img[:, :, None]
    elif img.ndim == 3 and img.shape[2] == 3:
        header = b"PF\n"
    else:
        raise ValueError("PFM supports (H, W) or (H, W, 3) images")
    h, w = img.shape[:2]
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(f"{w} {h}\n".encode())
        fh.write(b"-1.0\n")
        fh.write(np.flipud(img).astype("<f4").tobytes())


def read_pfm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        kind = fh.readline().strip()
        if kind not in (b"PF", b"Pf"):
            raise ValueError(f"not a PFM file: {kind!r}")
        w, h = (int(x) for x in fh.readline().split())
        scale = float(fh.readline())
        count = w * h * (3 if kind == b"PF" else 1)
        data = np.frombuffer(fh.read(count * 4), dtype="<f4" if scale < 0 else ">f4")
        if data.size != count:
            raise ValueError("truncated PFM payload")
    img = data.reshape((h, w, 3) if kind == b"PF" else (h, w))
    return np.ascontiguousarray(np.flipud(img)).astype(np.float32)


def write_ppm(path, image, gamma=2.2):
    img = np.asarray(to_numpy(image), dtype=np.float64)
    if img.ndim == 2:
        img = np.repeat(img[:, :, None], 3, axis=2)
    img = np.clip(img, 0.0, 1.0) ** (1.0 / gamma)
    data = (img * 255.0 + 0.5).astype(np.uint8)
    h, w = data.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode())
        fh.write(data.tobytes())


def cone_basis(light_unit):
    """render.py:237-241: (t1, t2) spanning the plane normal to the light."""
    l = np.asarray(light_unit, dtype=np.float64)
    up = np.array([0.0, 1.0, 0.0]) if abs(l[1]) < 0.9 else np.array([1.0, 0.0, 0.0])
    t1 = np.cross(l, up)
    t1 /= np.linalg.norm(t1)
    t2 = np.cross(l, t1)
    return t1, t2


def reference_visibility(view, gbuffer: GBuffer, light: DirectionalLight, spp=256,
                         seed=0) -> torch.Tensor:
    """Fraction of unoccluded cone-sampled shadow rays per pixel (render.py:231-254)."""
    if spp < 1:
        raise ValueError("spp must be >= 1")
    bvh = view.bvh
    l = light.unit()
    t1, t2 = cone_basis(l)
    h, w = gbuffer.shape
    out = torch.empty((h, w), dtype=torch.float64, device=gbuffer.position.device)
    cov = gbuffer.coverage.to(torch.uint8)
    _lib.check(_lib.lib().rtsdf_reference_visibility(
        _lib.ptr(bvh.packed), bvh.num_nodes, _lib.ptr(gbuffer.position), _lib.ptr(gbuffer.normal),
        _lib.ptr(cov), h, w, (_lib.D * 3)(*map(float, l)), (_lib.D * 3)(*map(float, t1)),
        (_lib.D * 3)(*map(float, t2)),
        math.tan(light.angular_radius), int(spp), int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(out),
        _lib.stream()), "reference_visibility")
    return out


def reference_render(view, camera: Camera, light: DirectionalLight, spp=256, seed=0,
                     background=(0.05, 0.07, 0.10)) -> torch.Tensor:
    """Distributed ray-traced ground truth with the same Lambert shading (render.py:257-264)."""
    gb = rasterize_gbuffer(view, camera)
    vis = reference_visibility(view, gb, light, spp=spp, seed=seed)
    return compose(gb, 1.0 - vis, light, background)


__all__ = ["Camera", "DirectionalLight", "DiscLight", "GBuffer", "rasterize_gbuffer",
           "occlusion_image", "compose", "shade", "compare", "write_pfm", "read_pfm", "write_ppm",
           "reference_visibility", "reference_render", "cone_basis"]
