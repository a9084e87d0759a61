"""Run N hybrid C3 frames (the bench step) -- a short command for ncu/compute-sanitizer."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=4)
ap.add_argument("--rays", type=int, default=32)
ap.add_argument("--scene", default="sphere_plane")
ap.add_argument("--dims", default="400,200,400")
a = ap.parse_args()

import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402

dims = tuple(int(v) for v in a.dims.split(","))
cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims,
                        sampling=rt.SamplingParams(rays_per_frame=a.rays))
pipe = rt.FramePipeline(rt.get_scene(a.scene), cfg)
for _ in range(a.frames):
    rec = pipe.advance(render=True, timing=False)
torch.cuda.synchronize()
print("frames", a.frames, "masked", rec.masked_texels, "launches", rt._lib.launch_count())
