"""Fraction of non-EMPTY cells in each JFA pass input at C3 (sparse-pass study)."""
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
for off in J.jfa_offsets(dims):
    ne = (src != -1)
    seg = ne.view(dims[0], dims[1], -1)
    # 32-lane z segments (nz = 400 -> 12.5 segments; pad)
    nzb = (dims[2] + 31) // 32
    pad = torch.zeros(dims[0], dims[1], nzb * 32, dtype=torch.bool, device="cuda")
    pad[:, :, :dims[2]] = ne
    segs = pad.view(dims[0], dims[1], nzb, 32).any(dim=3)
    print(f"input of k={off:4d}: non-EMPTY cells {ne.float().mean().item() * 100:6.2f} %, "
          f"non-empty 32-z segments {segs.float().mean().item() * 100:6.2f} %")
    J.launch_step(src, dst, off, h, w)
    src, dst = dst, src
