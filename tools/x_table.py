"""Frame time vs rays per texel x at C3 (SURVEY §0 / §7 hard part 3): the bench
step (V + JF + RT + DL, static scene, CUDA-graph frames with the flood-ahead
overlap) timed with CUDA events for x in {0, 1, 4, 8, 16, 32}, plus one
serial event-timed frame for the stage split.  Prints one JSON line per x."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402

D = (400, 200, 400)
scene = rt.get_scene("sphere_plane")
for x in (0, 1, 4, 8, 16, 32):
    cfg = rt.PipelineConfig(coarse_dims=D, fine_dims=D, sampling=rt.SamplingParams(rays_per_frame=x))
    pipe = rt.FramePipeline(scene, cfg)
    for _ in range(4):
        pipe.advance(render=True, timing=False)
    pipe.join()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        pipe.advance(render=True, timing=False)
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    rec = pipe.advance(render=True, timing=True)
    st = {k: round(v / 1e6, 3) for k, v in rec.durations_ns.items()}
    print(json.dumps({"x": x, "ms_per_frame": round(e0.elapsed_time(e1) / n, 3), "stages_ms": st,
                      "rays_per_frame": rec.masked_texels * x}), flush=True)
    del pipe
    torch.cuda.empty_cache()
