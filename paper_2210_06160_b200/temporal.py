"""Temporal evaluation of the hybrid field on dynamic scenes.

Mirrors the reference's scenario description and its ghosting experiment
(/root/reference/pkg/src/sdfshadow/bench.py:28-84 Scenario / SIZES,
:300-364 GhostingResult / ghosting_experiment): after `warmup` frames the
orbiting occluder moves one step; fine texels that were on its old surface
split into a c <= d group, whose residual must decay like alpha^k (Eq. 1), and
a c > d group, which must equal the coarse value at once.  The frames run on
the device (FramePipeline); only the per-frame bookkeeping over the vacated
texels is host numpy, on the same float32 arrays and with the same numpy
expressions as the reference, so every reported number is the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from ._device import to_numpy
from .pipeline import FramePipeline, PipelineConfig
from .raysample import SamplingParams, coarse_at_fine
from .scenes import Instance, Scene, get_scene

# named resolutions: coarse / fine (bench.py:28-32)
SIZES = {
    "S": ((64, 64, 64), (128, 128, 128)),
    "M": ((128, 128, 128), (256, 256, 256)),
    "L": ((256, 256, 256), (512, 512, 512)),
}


class ScenarioError(ValueError):
    pass


@dataclass(frozen=True)
class Scenario:
    """bench.py:43-84 (the fields that shape a run; CSV / output options are
    the reference's CLI tooling and out of scope)."""

    scenario_id: str
    scene: str = "sphere_plane"
    size: str = "M"
    coarse_dims: tuple | None = None
    fine_dims: tuple | None = None
    x: int = 5
    d: float = 0.1
    alpha: float = 0.95
    frames: int = 8
    animate: bool = True
    seed: int = 0
    beta: float = 0.0
    bias: float = 0.01
    repeats: int = 5

    def resolved_dims(self):
        if self.coarse_dims and self.fine_dims:
            return tuple(self.coarse_dims), tuple(self.fine_dims)
        if self.size not in SIZES:
            raise ScenarioError(f"unknown size {self.size!r}; expected one of {sorted(SIZES)} "
                                "or explicit coarse_dims/fine_dims")
        return SIZES[self.size]

    def build(self) -> tuple[Scene, PipelineConfig]:
        try:
            scene = get_scene(self.scene)
        except KeyError as exc:
            raise ScenarioError(str(exc)) from None
        if not self.animate:
            scene = replace_tracks_static(scene)
        coarse, fine = self.resolved_dims()
        mask_d = math.inf if self.d == float("inf") else self.d
        cfg = PipelineConfig(coarse_dims=coarse, fine_dims=fine,
                             sampling=SamplingParams(rays_per_frame=self.x, mask_distance=mask_d,
                                                     decay_alpha=self.alpha, seed=self.seed),
                             beta=self.beta, bias=self.bias, repeats=self.repeats)
        return scene, cfg


def replace_tracks_static(scene: Scene) -> Scene:
    """Freeze every instance at its frame-0 transform (bench.py:87-97)."""
    from dataclasses import replace as dc_replace

    frozen = []
    for inst in scene.instances:
        m = inst.transform_at(0)
        frozen.append(Instance(mesh=inst.mesh.transformed(m), albedo=inst.albedo))
    return dc_replace(scene, name=scene.name + "-static", instances=tuple(frozen))


@dataclass
class GhostingResult:
    frames: list              # frame indices after the vacate event
    envelope: list            # alpha^k * initial residual per frame
    residual_in_band: list    # median |mag - c| over tracked c <= d texels
    max_ratio: float          # worst residual / envelope over the window
    outside_exact: bool       # c > d texels equal coarse immediately
    tracked: int

    def decays_within(self, slack=1.1):
        return self.max_ratio <= slack


def _coarse_at_fine(pipe, fine_dims):
    return to_numpy(coarse_at_fine(pipe.coarse, fine_dims))


def ghosting_experiment(scenario: Scenario, warmup=10, window=14, band_lo=0.035) -> GhostingResult:
    """bench.py:310-364 on the device pipeline (same statistics, same numpy)."""
    scene, cfg = scenario.build()
    if not scene.animated:
        raise ScenarioError("ghosting experiment needs an animated scene")
    pipe = FramePipeline(scene, cfg)
    for _ in range(warmup):
        pipe.advance()
    d = cfg.sampling.mask_distance
    c_before = _coarse_at_fine(pipe, cfg.fine_dims)
    fine_before = np.abs(to_numpy(pipe.fine.data))

    pipe.advance()  # the vacate event
    c_after = _coarse_at_fine(pipe, cfg.fine_dims)

    vacated = (fine_before < band_lo) & (c_after > c_before + 0.02)
    in_band = vacated & (c_after <= d)
    out_band = vacated & (c_after > d)
    fine = to_numpy(pipe.fine.data)
    outside_exact = bool(np.array_equal(fine[out_band], c_after[out_band]))

    idx = np.nonzero(in_band)
    r0 = np.abs(np.abs(fine[idx]) - c_after[idx])
    alive = r0 > 1e-4
    frames, env, res, ratios = [], [], [], []
    alpha = cfg.sampling.decay_alpha
    for k in range(1, window + 1):
        pipe.advance()
        c_now = _coarse_at_fine(pipe, cfg.fine_dims)
        fine = to_numpy(pipe.fine.data)
        stable = alive & (np.abs(c_now[idx] - c_after[idx]) < 1e-3)
        if stable.sum() == 0:
            break
        residual = np.abs(np.abs(fine[idx]) - c_now[idx])[stable]
        envelope = (alpha ** k) * r0[stable]
        frames.append(pipe.frame - 1)
        env.append(float(np.median(envelope)))
        res.append(float(np.median(residual)))
        ratios.append(float(np.max(residual / np.maximum(envelope, 1e-9))))
    return GhostingResult(frames=frames, envelope=env, residual_in_band=res,
                          max_ratio=max(ratios) if ratios else float("inf"),
                          outside_exact=outside_exact, tracked=int(alive.sum()))


__all__ = ["SIZES", "Scenario", "ScenarioError", "replace_tracks_static", "GhostingResult",
           "ghosting_experiment"]
