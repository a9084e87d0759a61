"""Counter-based random streams (rng.py:1-53) -- host numpy form + device tables.

The sampler generates its directions on the device: SplitMix64 plus a bit-exact
restatement of the host glibc's cos / sin (csrc/glibc_sincos.cuh), so the
default, benchmarked path draws exactly the reference's directions.  This
module is the host side: the north star's "host-supplied ray-direction table"
(numpy == numba bit for bit), the scalar API helpers
(sample_texel, soft_shadow jitter) and `device_direction_table`, which runs the
sampler's own direction code for a list of texels.
"""

from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)
INV53 = 1.0 / 9007199254740992.0


def mix64(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        return z ^ (z >> np.uint64(31))


def stream_key(seed, stream, tick):
    k = mix64(np.uint64(seed) ^ GOLDEN)
    k = mix64(k ^ np.asarray(stream).astype(np.uint64))
    return mix64(k ^ np.uint64(tick))


def uniform(key, counter):
    with np.errstate(over="ignore"):
        bits = mix64(np.asarray(key, dtype=np.uint64)
                     + np.asarray(counter).astype(np.uint64) * GOLDEN)
    return (bits >> np.uint64(11)).astype(np.float64) * INV53


def unit_sphere_dir(key, counter):
    """(x, y, z) arrays; consumes counters 2c and 2c+1 (rng.py:46-53)."""
    c = np.asarray(counter).astype(np.uint64)
    u = uniform(key, np.uint64(2) * c)
    v = uniform(key, np.uint64(2) * c + np.uint64(1))
    z = 1.0 - 2.0 * u
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = 2.0 * np.pi * v
    return r * np.cos(phi), r * np.sin(phi), z


def direction_table(seed: int, texel_index, frame: int, x: int) -> np.ndarray:
    """(M, x, 3) float64 directions of texels `texel_index` at `frame`."""
    idx = np.asarray(texel_index, dtype=np.int64).reshape(-1)
    keys = stream_key(seed, idx, frame)[:, None]
    r = np.arange(x, dtype=np.uint64)[None, :]
    dx, dy, dz = unit_sphere_dir(keys, r)
    return np.ascontiguousarray(np.stack([dx, dy, dz], axis=-1))


def device_direction_table(seed: int, texel_index, frame: int, x: int) -> np.ndarray:
    """direction_table computed by the device kernels' code path (rtsdf_unit_sphere_dirs)."""
    import torch

    from . import _lib
    from ._device import to_device

    idx = np.asarray(texel_index, dtype=np.int64).reshape(-1)
    keys = to_device(stream_key(seed, idx, frame).astype(np.uint64).view(np.int64))
    out = torch.empty((len(idx), int(x), 3), dtype=torch.float64, device=keys.device)
    _lib.check(_lib.lib().rtsdf_unit_sphere_dirs(_lib.ptr(keys), len(idx), int(x), _lib.ptr(out),
                                                 _lib.stream()), "unit_sphere_dirs")
    return out.cpu().numpy()


__all__ = ["mix64", "stream_key", "uniform", "unit_sphere_dir", "direction_table",
           "device_direction_table"]
