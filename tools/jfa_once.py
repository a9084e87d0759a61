"""One C3 (or given) JFA schedule via flood_to_sdf after a warm-up run: the
command profiled by ncu (tools/ncu_jfa.sh).  Usage: jfa_once.py [dims] [scene]"""
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
a = torch.empty(dims, dtype=torch.int32, device="cuda")
b = torch.empty_like(a)
out = torch.empty(dims, dtype=torch.float32, device="cuda")
for _ in range(2):
    rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)
    J.flood_to_sdf(a, b, out, h)
torch.cuda.synchronize()
print("ok", float(out.float().mean()))
