"""Experiment: sampler time with on-device RNG directions vs a device-resident
direction table (isolates the cost of direction generation from traversal)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402
from paper_2210_06160_b200 import raysample as RS  # noqa: E402

dims = (400, 200, 400)
scene = rt.get_scene("sphere_plane")
cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims, sampling=rt.SamplingParams(rays_per_frame=32))
pipe = rt.FramePipeline(scene, cfg)
pipe.advance(render=False, timing=False)
b = pipe._buffers()
cb = b["compact"]
m = int(cb.count.item())
idx = cb.idx[:m].cpu().numpy()
t0 = time.time()
dirs = rt.direction_table(0, idx, 1, 32)
print("host table", dirs.shape, f"{time.time() - t0:.1f}s", flush=True)
dirs_d = torch.from_numpy(dirs).cuda()
del dirs
g = RS._RsGeom(pipe.coarse, dims)
view = scene.view(0)
t_max = float(np.linalg.norm(scene.hi - scene.lo))
smin = torch.empty(m, dtype=torch.float64, device="cuda")
sf = torch.empty(m, dtype=torch.int32, device="cuda")
sb = torch.empty(m, dtype=torch.int32, device="cuda")
for name, d in (("device-rng", None), ("table", dirs_d), ("device-rng", None), ("table", dirs_d)):
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        RS.launch_sample_update(view.bvh, g, cb, cfg.sampling, 1, t_max, dirs=d, samp=(smin, sf, sb),
                                m_cap=m)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "ms", [round(t, 3) for t in ts], flush=True)
    ws = RS._SWS[torch.cuda.current_device()]
    print("  queued long rays:", int(ws[:8].view(torch.int64).item()), "of", m * 32, flush=True)
