"""Animated orbit scene (reference blob.obj) at C3 size: ms/frame with the
per-frame device BVH build / refit (wall clock and CUDA events), and the host
cost of one SceneView (merge + normals + device build launch)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402

scene = rt.get_scene("orbit")
dims = (400, 200, 400)
cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims, sampling=rt.SamplingParams(rays_per_frame=32))
pipe = rt.FramePipeline(scene, cfg)
for f in range(3):
    pipe.advance(render=True, timing=False)
torch.cuda.synchronize()
t0 = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for f in range(20):
    pipe.advance(render=True, timing=False)
e1.record()
torch.cuda.synchronize()
print(f"orbit (animated, device BVH) wall ms/frame {(time.time() - t0) * 50:.2f}  "
      f"gpu-event ms/frame {e0.elapsed_time(e1) / 20:.2f}")
torch.cuda.synchronize()
t0 = time.time()
for f in range(20):
    v = scene.view(100 + f)
torch.cuda.synchronize()
print(f"SceneView (merge + normals + upload + device build/refit) ms {(time.time() - t0) * 50:.3f}")
from paper_2210_06160_b200.geometry import build_bvh  # noqa: E402

t0 = time.time()
for f in range(5):
    build_bvh(scene.view(200 + f).mesh)
print(f"host reference + SAH + BVH4 build ms {(time.time() - t0) * 200:.3f}")
