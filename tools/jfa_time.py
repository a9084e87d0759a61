"""Time the C3 JFA schedule (per pass + whole run_sdf call) with CUDA events;
RTSDF_LIB selects an alternative build (tools/build_variants.sh).  Also checks
the final SDF digest against the default run so a variant cannot be faster by
being wrong."""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402
from paper_2210_06160_b200 import jfa as J  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "400,200,400").split(","))
scene = rt.get_scene(sys.argv[2] if len(sys.argv) > 2 else "sphere_plane")
view = scene.view(0)
h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
w = J.integer_weights(*map(float, h), dims)
offs = J.jfa_offsets(dims)
a = torch.empty(dims, dtype=torch.int32, device="cuda")
b = torch.empty_like(a)
out = torch.empty(dims, dtype=torch.float32, device="cuda")


def seed():
    rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)


per = []
for rep in range(5):
    seed()
    src, dst = a, b
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(offs) + 1)]
    ev[0].record()
    for i, off in enumerate(offs):
        J.launch_step(src, dst, off, h, w)
        ev[i + 1].record()
        src, dst = dst, src
    torch.cuda.synchronize()
    per.append([ev[i].elapsed_time(ev[i + 1]) for i in range(len(offs))])
per = np.median(np.array(per), axis=0)
runs = []
for rep in range(7):
    seed()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    J.flood_to_sdf(a, b, out, h)
    e1.record()
    torch.cuda.synchronize()
    runs.append(e0.elapsed_time(e1))
dig = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
tag = os.environ.get("RTSDF_LIB", "default").split("/")[-1]
print(f"{tag:28s} run_sdf {np.median(runs):.4f} ms  passes " + " ".join(f"{t:.3f}" for t in per)
      + f"  sdf {dig}")
