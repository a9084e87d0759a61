"""Experiment: two sampler launches of a C3 frame (separate workspaces and
outputs) back to back on one stream vs concurrently on two streams -- does
mixing two tracer kernels' warps on the SMs raise throughput?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402
from paper_2210_06160_b200 import _lib  # noqa: E402
from paper_2210_06160_b200 import raysample as RS  # noqa: E402

dims = (400, 200, 400)
scene = rt.get_scene("sphere_plane")
cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims, sampling=rt.SamplingParams(rays_per_frame=32))
pipe = rt.FramePipeline(scene, cfg)
pipe.advance(render=False, timing=False)
b = pipe._buffers()
cb = b["compact"]
m = int(cb.count.item())
g = RS._RsGeom(pipe.coarse, dims)
view = scene.view(0)
t_max = float(np.linalg.norm(scene.hi - scene.lo))
L = _lib.lib()
need = int(L.rtsdf_sample_ws_bytes(m, 32))
ws = [torch.empty(need, dtype=torch.uint8, device="cuda") for _ in range(2)]
outs = [(torch.empty(m, dtype=torch.float64, device="cuda"), torch.empty(m, dtype=torch.int32, device="cuda"),
         torch.empty(m, dtype=torch.int32, device="cuda")) for _ in range(2)]
desc = g.desc()
bvh = view.bvh


def launch(i, stream):
    smin, sf, sb = outs[i]
    _lib.check(L.rtsdf_sample_update(
        _lib.ptr(bvh.search), bvh.search_nodes, bvh.num_tris, bvh.search_nodes4, bvh.search_stack4,
        _lib.ptr(cb.idx),
        _lib.ptr(cb.count), m, desc, 32, 0, 3 + i, None, t_max, None,
        _lib.ptr(smin), _lib.ptr(sf), _lib.ptr(sb), None, None, None, None, None, 0.95, None,
        _lib.ptr(ws[i]), ws[i].numel(), stream.cuda_stream), "sample_update")


s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
for mode in ("serial", "concurrent", "serial", "concurrent"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    if mode == "serial":
        launch(0, s0)
        launch(1, s0)
    else:
        s1.wait_stream(s0)
        launch(0, s0)
        launch(1, s1)
        s0.wait_stream(s1)
    e1.record(s0)
    torch.cuda.synchronize()
    print(mode, round(e0.elapsed_time(e1), 3), "ms for two sampler launches")
