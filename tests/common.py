"""Shared helpers for the test-suite: golden fixtures, digests, scene inputs."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype == np.bool_:
        a = a.astype(np.uint8)
    return hashlib.sha256(a.tobytes()).hexdigest()


@lru_cache(maxsize=1)
def golden() -> dict:
    return json.loads((GOLDEN / "golden.json").read_text())


@lru_cache(maxsize=1)
def golden_arrays():
    with np.load(GOLDEN / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@lru_cache(maxsize=1)
def golden_large() -> dict:
    return json.loads((GOLDEN / "golden_large.json").read_text())


@lru_cache(maxsize=1)
def golden_large_arrays():
    with np.load(GOLDEN / "golden_large.npz") as z:
        return {k: z[k] for k in z.files}


def scene_mesh(name, frame=0):
    """(scene, merged world mesh) built by the product's host-side scene code."""
    from paper_2210_06160_b200 import scenes
    from paper_2210_06160_b200.geometry import make_mesh

    scene = scenes.get_scene(name)
    verts, tris, base = [], [], 0
    for inst in scene.instances:
        m = inst.transform_at(frame)
        v = inst.mesh.vertices @ m[:, :3].T + m[:, 3]
        verts.append(v)
        tris.append(inst.mesh.triangles + base)
        base += len(v)
    return scene, make_mesh(np.vstack(verts), np.vstack(tris))


C1 = dict(scene="sphere", dims=(64, 64, 64), x=32)
C3 = dict(scene="sphere_plane", dims=(400, 200, 400), x=32)
