import sys, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2210_06160_b200 as rt
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
for f in range(10):
    pipe.advance(render=True, timing=False)
e1.record(); torch.cuda.synchronize()
print("orbit (animated) wall ms/frame", (time.time() - t0) * 100, "gpu-event ms/frame", e0.elapsed_time(e1) / 10)
t0 = time.time()
for f in range(10):
    v = scene.view(100 + f); _ = v.bvh
print("host view+bvh build ms", (time.time() - t0) * 100)
