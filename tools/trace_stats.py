"""Traversal work counters for one C3 sampler launch (needs a library built
with RTSDF_NVCC_EXTRA=-DRTSDF_TRACE_STATS): node visits, leaf visits, fp32
triangle pre-tests and exact fp64 tests, per ray."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402
from paper_2210_06160_b200 import _lib  # noqa: E402
from paper_2210_06160_b200 import raysample as RS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sphere_plane"
dims = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "400,200,400").split(","))
scene = rt.get_scene(name)
cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims, sampling=rt.SamplingParams(rays_per_frame=32))
pipe = rt.FramePipeline(scene, cfg)
pipe.advance(render=False, timing=False)
b = pipe._buffers()
cb = b["compact"]
m = int(cb.count.item())
g = RS._RsGeom(pipe.coarse, dims)
view = scene.view(0)
t_max = float(np.linalg.norm(scene.hi - scene.lo))
smin = torch.empty(m, dtype=torch.float64, device="cuda")
sf = torch.empty(m, dtype=torch.int32, device="cuda")
sb = torch.empty(m, dtype=torch.int32, device="cuda")
fn = _lib.lib().rtsdf_debug_trace_stats
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
out = (ctypes.c_ulonglong * 12)()
fn(out)
RS.launch_sample_update(view.bvh, g, cb, cfg.sampling, 1, t_max, samp=(smin, sf, sb), m_cap=m)
torch.cuda.synchronize()
fn(out)
rays = m * 32
names = ["node visits", "leaf visits", "tri pre-tests", "exact tests"]
for n, v in zip(names, out[:4]):
    print(f"{n:14s} {v:14d}  {v / rays:8.3f} per ray")
hist = list(out[4:])
if sum(hist):
    labels = ["0-1", "2-3", "4-7", "8-15", "16-31", "32-63", "64-127", "128+"]
    tot = sum(hist)
    print("long-ray node visits:", ", ".join(f"{l}: {100.0 * h / tot:.1f}%" for l, h in zip(labels, hist)))
