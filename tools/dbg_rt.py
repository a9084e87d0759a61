import sys; sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2210_06160_b200 as rt
scene = rt.get_scene("sphere_plane")
D=(400,200,400)
cfg = rt.PipelineConfig(coarse_dims=D, fine_dims=D, sampling=rt.SamplingParams(rays_per_frame=32))
pipe = rt.FramePipeline(scene, cfg)
for f in range(6):
    pipe.advance(render=True, timing=False)
pipe.join(); torch.cuda.synchronize()
print("m_cap", pipe._m_cap, "graphs", list(getattr(pipe, "_graphs", {}).keys()))
for f in range(2):
    r = pipe.advance(render=True, timing=True); print("timed", r.durations_ns, r.masked_texels)
pipe.overlap_frames = False
for f in range(3):
    pipe.advance(render=True, timing=False)
torch.cuda.synchronize()
for f in range(2):
    r = pipe.advance(render=True, timing=True); print("timed after e2e", r.durations_ns, r.masked_texels)
