"""C5: 1024^3 JFA-only SDF of box_spheres on ONE GPU (the
config's 8-GPU z-slab form is bench/shard territory): voxelize + full JFA
schedule + seeds -> SDF, Gvox-pass/s and % of the HBM roofline."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_06160_b200 as rt  # noqa: E402
from paper_2210_06160_b200 import jfa as J  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024,1024,1024").split(","))
scene = rt.get_scene("box_spheres")
view = scene.view(0)
h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
a = torch.empty(dims, dtype=torch.int32, device="cuda")
b = torch.empty_like(a)
out = torch.empty(dims, dtype=torch.float32, device="cuda")
vs = rt.voxelize_seeds(view.mesh, dims, scene.bounds, buffers=view.mesh_buffers(), out=a)
occ = int((a != -1).sum().item())
ts = []
for rep in range(4):
    rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    J.flood_to_sdf(a, b, out, h)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts[1:]))
n = int(np.prod(dims))
passes = len(J.jfa_offsets(dims))
gv = n * passes / (ms * 1e-3) / 1e9
peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(json.dumps({"config": f"C5 box_spheres {dims} JFA-only (+ seeds -> SDF fused)", "occupied": occ,
                  "passes": passes, "ms": round(ms, 2), "gvox_pass_per_s": round(gv, 1),
                  "hbm_frac_8B_per_voxel_pass": round(gv * 8 / peak, 4),
                  "exact_fp64_mode": True, "times_ms": [round(t, 2) for t in ts]}))
