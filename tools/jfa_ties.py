"""Integer-tie cells (re-decided by the fp64 fix-up) per JFA pass at C3: the
fix-up list count the pass leaves at the head of the JFA workspace."""
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
a = torch.empty(dims, dtype=torch.int32, device="cuda")
b = torch.empty_like(a)
rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)
src, dst = a, b
n = int(np.prod(dims))
for off in J.jfa_offsets(dims):
    J.launch_step(src, dst, off, h, w)
    ws = J.workspace(*dims)
    cnt = int(ws[:8].view(torch.int64).item())
    changed = int((src != dst).sum().item())
    print(f"k={off:4d} tie cells {cnt:9d} ({100.0 * cnt / n:5.2f} %)  changed {changed:9d} ({100.0 * changed / n:5.2f} %)")
    src, dst = dst, src
