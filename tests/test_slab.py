"""z-slab JFA sharding: the exchange plan (pure host logic), a real
world_size-2 gloo run on the CPU (oracle as the per-rank compute), and the
single-GPU loopback of the slab kernel."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from common import scene_mesh

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

from paper_2210_06160_b200 import slab as S  # noqa: E402


@pytest.mark.parametrize("nx,world", [(400, 2), (400, 8), (64, 3), (1024, 8), (10, 4)])
def test_plan_covers_exactly_the_foreign_taps(nx, world):
    bounds = S.slab_bounds(nx, world)
    assert sum(n for _, n in bounds) == nx
    for k in O.jfa_offsets((nx, 1, 1)):
        plan = S.plan_pass(nx, bounds, k)
        for r, (x0, nxl) in enumerate(bounds):
            need = set()
            for i in range(x0, x0 + nxl):
                for q in (i - k, i + k):
                    if 0 <= q < nx and not (x0 <= q < x0 + nxl):
                        need.add(q)
            got = set()
            for t in plan:
                if t.dst != r:
                    continue
                s0, sn = bounds[t.src]
                assert s0 <= t.first and t.first + t.count <= s0 + sn  # sent by its owner
                got.update(range(t.first, t.first + t.count))
            assert got == need, (k, r)


def test_halo_volume_matches_survey_c5():
    # C5 at P = 8 -> up to 894 inbound planes on the worst rank
    planes, _ = S.halo_volume(1024, 1024, 1024, 8)
    assert planes.max() == 894


def _gloo_worker(rank, world, port, occ, h, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = occ.shape
    bounds = S.slab_bounds(nx, world)
    x0, nxl = bounds[rank]
    full = O.jfa_init(occ)
    local = torch.from_numpy(full[x0:x0 + nxl].copy())
    maxh = max(1, max(min(nxl, k) for k in O.jfa_offsets(occ.shape)))
    halo_lo = torch.empty((maxh, ny, nz), dtype=torch.int32)
    halo_hi = torch.empty_like(halo_lo)
    for k in O.jfa_offsets(occ.shape):
        plan = S.plan_pass(nx, bounds, k)
        S.exchange(local, halo_lo, halo_hi, plan, rank, bounds)
        # per-rank compute: the oracle on a grid holding only local + halo planes
        work = np.full(occ.shape, -1, dtype=np.int32)
        work[x0:x0 + nxl] = local.numpy()
        lo, hi = S.halo_ranges(nx, x0, nxl, k)
        work[lo[0]:lo[0] + lo[1]] = halo_lo[:lo[1]].numpy()
        work[hi[0]:hi[0] + hi[1]] = halo_hi[:hi[1]].numpy()
        local = torch.from_numpy(O.jfa_step(work, k, h)[x0:x0 + nxl].copy())
    out = [torch.empty((n, ny, nz), dtype=torch.int32) for _, n in bounds]
    if rank == 0:
        dist.gather(local, out, dst=0)
        ret.put(np.concatenate([t.numpy() for t in out]))
    else:
        dist.gather(local, None, dst=0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_jfa_bit_exact(world):
    scene, mesh = scene_mesh("sphere_plane")
    dims = (48, 24, 40)
    occ = O.voxelize(mesh.vertices, mesh.triangles, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, occ, h, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(got, O.jfa_run(occ, h))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_slab_kernel_c3(world):
    import paper_2210_06160_b200 as rt

    scene, mesh = scene_mesh("sphere_plane")
    dims = (400, 200, 400)
    vs = rt.voxelize_seeds(mesh, dims, scene.bounds)
    h = (scene.hi - scene.lo) / np.array(dims, dtype=np.float64)
    got = S.flood_loopback(vs.seed_packed, world, h)
    want = rt.jfa_run(rt.voxelize(mesh, dims, scene.bounds)).packed
    assert torch.equal(got, want)
