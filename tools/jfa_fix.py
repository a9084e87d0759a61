"""Per-pass JFA diagnostics at C3: pass time and the size of the integer-tie
fix-up list (first 8 bytes of the JFA workspace) after every pass."""
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
for rep in range(3):
    rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)
    src, dst = a, b
    rows = []
    for off in J.jfa_offsets(dims):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        J.launch_step(src, dst, off, h, w)
        e1.record()
        torch.cuda.synchronize()
        ws = J.workspace(*dims)
        n_fix = int(ws[:8].view(torch.int64).item())
        rows.append((off, e0.elapsed_time(e1), n_fix))
        src, dst = dst, src
    if rep == 2:
        for off, ms, n in rows:
            print(f"k={off:4d}  {ms:7.3f} ms  fix={n:9d} ({100.0 * n / np.prod(dims):.2f}%)")
print("weights", w)
ts = []
for rep in range(5):
    rt.voxelize_seeds(view.mesh, dims, scene.bounds, check=False, buffers=view.mesh_buffers(), out=a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    J.flood_inplace(a, b, h)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("schedule (rtsdf_jfa_run) ms", [round(t, 3) for t in ts])
