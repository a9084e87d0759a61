"""C3 ms/frame with and without cross-frame flood overlap (PipelineConfig.overlap_frames)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402

dims = (400, 200, 400)
for overlap in (True, True):
    cfg = rt.PipelineConfig(coarse_dims=dims, fine_dims=dims, overlap_frames=overlap,
                            sampling=rt.SamplingParams(rays_per_frame=32))
    pipe = rt.FramePipeline(rt.get_scene("sphere_plane"), cfg)
    for _ in range(4):
        pipe.advance(render=True, timing=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        pipe.advance(render=True, timing=False)
    pipe.join()
    e1.record()
    torch.cuda.synchronize()
    print("overlap", overlap, "ms/frame", round(e0.elapsed_time(e1) / 20, 4), flush=True)
    del pipe
    torch.cuda.empty_cache()
