#!/usr/bin/env python
"""Headline benchmark: hybrid SDF ms/frame at 400x200x400 (+ JFA Gvox-pass/s, % HBM).

One step = one FramePipeline.advance(render=True) of the paper-shaped scene
(BASELINE.json configs[2]): voxelize -> 9-pass JFA -> seeds
-> SDF -> resample/mask -> 32 rays per masked texel + Eq. 1 -> G-buffer ->
soft-shadow march 240x180 -> compose, all on the device.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): the z-slab sharded frame (shard.py: each
frame split over the N GPUs, NCCL P2P halo planes per JFA pass, fine slabs
gathered on rank 0 for the shading; "scaling": "strong"), value = max-over-
ranks time / frames; --replicas runs N independent frames instead ("weak").
--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, OpenMP over all host cores): every step is one whole
C3 frame with the temporal state carried over, nothing sampled or
extrapolated.  With WORLD_SIZE unset, --gpus N > 1 re-launches itself under
torch.distributed.run with N ranks (127.0.0.1); under torchrun WORLD_SIZE
must equal --gpus.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

DIMS = (400, 200, 400)
METRIC = "hybrid SDF ms/frame at 400x200x400"
UNIT = "ms/frame"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rays", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-frames", type=int, default=3,
                    help="cpu_baseline: full C3 frames timed (after one warm-up frame)")
    ap.add_argument("--cpu-baseline-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent frames instead of the z-slab sharded frame")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded frame even at N = 1 (under torchrun; tests the glue)")
    return ap.parse_args()


def workload(x):
    return {"workload": "C3 sphere_plane hybrid frame: V + 9-pass JFA + ray-sampled refine "
                        "+ Eq.1 + DL soft shadows 240x180",
            "dims": list(DIMS), "coarse_equals_fine": True, "rays_per_texel": x,
            "mask_distance": 0.1, "decay_alpha": 0.95, "shade": "240x180, 1 draw",
            "l2": "inputs larger than L2 (2 x 128 MB seed grids + 128 MB fields per frame)"}


# --------------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/rtsdf_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r.split(", ") for r in self.path.read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4)
                          if r[5 + i].strip() == "Active"})
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(sm)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


PROFILE = ROOT / "profiles" / "r2zj_frame_kernels_summary.csv"  # ncu --set full, one C3 frame
DENSE_KERNEL = "jfa_pass5_kernel<2, 2, 0"  # K2 v5 (jfa5.cuh), the dense passes k <= 16
DENSE_MAX_K = 16


def _profile_rows(prefix):
    """Rows of the committed per-kernel ncu summary whose kernel starts with prefix."""
    if not PROFILE.exists():
        return None, []
    import csv

    rows = list(csv.reader(PROFILE.read_text().splitlines()))
    return rows[0], [r for r in rows[1:] if r[0].startswith(prefix)]


def jfa_traffic():
    """DRAM bytes (read + write) per dense JFA pass launch (v5, k <= 16) from the
    committed ncu --set full capture of one frame."""
    head, rows = _profile_rows(DENSE_KERNEL)
    if not rows:
        return None, None
    rd, wr = head.index("dram_rd[MB]"), head.index("dram_wr[MB]")
    mb = [float(r[rd]) + float(r[wr]) for r in rows]
    return round(sum(mb) / len(mb) * 1e6), f"profiles/{PROFILE.name} (mean of {len(mb)} dense pass launches)"


def issue_roofline(n_cells, pass_ms, ck):
    """The JFA pass's binding limit: instruction issue.  Warp instructions per
    dense pass launch from the committed capture; peak = 148 SMs x 4 schedulers
    x 1 warp instruction per clock at the measured SM clock."""
    head, rows = _profile_rows(DENSE_KERNEL)
    if not rows:
        return None
    ii = head.index("inst")
    winst = sum(float(r[ii]) for r in rows) / len(rows)
    mhz = (ck or {}).get("sm_mhz") or 1965.0
    t_issue_ms = winst / (148 * 4 * mhz * 1e6) * 1e3
    return {"warp_instr_per_launch": round(winst), "thread_instr_per_cell": round(winst * 32 / n_cells, 1),
            "ms_at_100pct_issue": round(t_issue_ms, 4), "launch_ms": round(pass_ms, 4),
            "frac": round(t_issue_ms / pass_ms, 4),
            "candidate_floor_instr_per_cell": 162,
            "source": f"profiles/{PROFILE.name}"}


def sampler_roofline(rays, sample_ms):
    """K6 is issue / divergence bound (no HBM bound: BVH + triangles in L2):
    rays/s, SIMT efficiency and issue from the committed capture."""
    head, rows = _profile_rows("wf_pass")
    if not rows:
        return None
    ti, ii, si = head.index("thr/inst"), head.index("issue%"), head.index("time[ms]")
    return {"kernel": "wf_pass1_kernel + wf_pass2_kernel (K6)", "bound": "issue",
            "achieved": round(rays / (sample_ms * 1e-3) / 1e9, 2), "unit": "G rays/s",
            "passes": [{"kernel": r[0], "ms_ncu": float(r[si]), "threads_per_instr": float(r[ti]),
                        "issue_pct": float(r[ii])} for r in rows],
            "source": f"profiles/{PROFILE.name}"}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2210_06160_b200 as rt
    from paper_2210_06160_b200 import _lib
    from paper_2210_06160_b200 import jfa as J

    torch.cuda.set_device(local_rank)
    dist = world > 1
    if dist:
        import torch.distributed as tdist

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    scene = rt.get_scene("sphere_plane")
    cfg = rt.PipelineConfig(coarse_dims=DIMS, fine_dims=DIMS,
                            sampling=rt.SamplingParams(rays_per_frame=args.rays, mask_distance=0.1,
                                                       decay_alpha=0.95, seed=0))
    # N > 1: the z-slab sharded frame (each frame split over the N GPUs, NCCL
    # P2P halos per JFA pass, fine slabs gathered for the shading on rank 0);
    # --replicas: N independent frames instead
    sharded = (dist or args.sharded) and not args.replicas
    if sharded:
        from paper_2210_06160_b200.shard import ShardedFramePipeline

        sp = ShardedFramePipeline(scene, cfg, rank, world)

        def step():
            sp.advance(render=True)
    else:
        pipe = rt.FramePipeline(scene, cfg)

        def step():
            pipe.advance(render=True, timing=False)

    def join():  # the frame flooded ahead (V + JF of step K + 1) is inside the timed region
        if not sharded:
            pipe.join()

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for _ in range(args.steps):
        step()
    join()
    e1.record()
    barrier()
    launches = _lib.launch_count() - l0
    ck = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms_total], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms_total = float(t.item())
    frames = args.steps if sharded else args.steps * world
    value = ms_total / frames
    ms_per_step = ms_total / args.steps

    # ---- e2e through the public API with host buffers
    view = scene.view(0)
    mb = view.mesh_buffers()
    hv = torch.from_numpy(view.mesh.vertices.copy()).pin_memory()
    ht = torch.from_numpy(view.mesh.triangles.copy()).pin_memory()
    img_host = torch.empty((scene.camera.height, scene.camera.width, 3), dtype=torch.float32).pin_memory()
    cnt_host = torch.empty(1, dtype=torch.int64).pin_memory()
    h2d = hv.numel() * 8 + ht.numel() * 4
    d2h = img_host.numel() * 4 + 8

    def e2e_step():
        if not sharded:
            # pipelined input: frame f + 1's mesh goes up while frame f traces, and
            # frame f + 1's V + JF (flooded ahead during frame f) reads that upload
            pipe.upload_mesh(pipe.frame + 1, hv, ht)
        else:
            mb.verts.copy_(hv, non_blocking=True)
            mb.tris.copy_(ht, non_blocking=True)
        if sharded:
            cnt, img = sp.advance(render=True)
            if img is not None:
                img_host.copy_(img, non_blocking=True)
            cnt_host.copy_(cnt, non_blocking=True)
        else:
            r = pipe.advance(render=True, timing=False)
            img_host.copy_(pipe.last_image, non_blocking=True)
            cnt_host.copy_(r._masked_dev, non_blocking=True)

    for _ in range(2):
        e2e_step()
    barrier()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        e2e_step()
    z.record()
    barrier()
    e_ms = a.elapsed_time(z)
    if dist:
        t = torch.tensor([e_ms], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = {"value": e_ms / frames, "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "path": ("pinned mesh H2D -> ShardedFramePipeline.advance(render=True) on every rank -> "
                    "image (rank 0) + masked-count D2H") if sharded else
                   ("pinned mesh H2D of frame f+1 (FramePipeline.upload_mesh) -> "
                    "FramePipeline.advance(render=True) of frame f (floods f+1 from that upload) -> "
                    "image + masked-count D2H")}
    if sharded:  # kernel-level detail below runs on a single-GPU pipeline per rank
        del sp
        torch.cuda.empty_cache()
        pipe = rt.FramePipeline(scene, cfg)
        for _ in range(2):
            pipe.advance(render=True, timing=False)

    # ---- per-stage breakdown on this rank (one instrumented frame + standalone kernels)
    rec = pipe.advance(render=True, timing=True)
    stages_ms = {k: v / 1e6 for k, v in rec.durations_ns.items()}
    masked = rec.masked_texels
    b = pipe._buffers()
    h = (scene.hi - scene.lo) / np.array(DIMS, dtype=np.float64)
    w = J.integer_weights(*map(float, h), DIMS)
    offs = J.jfa_offsets(DIMS)
    # JFA: re-run the schedule from fresh seeds, one event pair per pass
    per_pass = []
    for rep in range(3):
        rt.voxelize_seeds(view.mesh, DIMS, scene.bounds, check=False, buffers=view.mesh_buffers(),
                          out=b["seed_a"])
        src, dst = b["seed_a"], b["seed_b"]
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(offs) + 1)]
        ev[0].record()
        for i, off in enumerate(offs):
            J.launch_step(src, dst, off, h, w)
            ev[i + 1].record()
            src, dst = dst, src
        torch.cuda.synchronize()
        per_pass.append([ev[i].elapsed_time(ev[i + 1]) for i in range(len(offs))])
    per_pass = np.median(np.array(per_pass), axis=0)
    # the schedule as the frame runs it (one C call: sparse early passes + v2)
    sched = []
    for rep in range(3):
        rt.voxelize_seeds(view.mesh, DIMS, scene.bounds, check=False, buffers=view.mesh_buffers(),
                          out=b["seed_a"])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        J.flood_inplace(b["seed_a"], b["seed_b"], h)
        e1.record()
        torch.cuda.synchronize()
        sched.append(e0.elapsed_time(e1))
    jfa_ms = float(np.median(sched))
    n_cells = int(np.prod(DIMS))
    gvox = n_cells * len(offs) / (jfa_ms * 1e-3) / 1e9
    # roofline of the pass kernel: its dense launches (k <= 16: v5 + its tie fix-up)
    dense = [float(t) for off, t in zip(offs, per_pass) if off <= DENSE_MAX_K]
    pass_ms = float(np.mean(dense)) if dense else float(np.mean(per_pass))
    hbm, hbm_src = peaks()
    jfa_gbs = gvox * 8.0
    # ray sampler alone (one launch on the current state)
    from paper_2210_06160_b200 import raysample as RS

    g = RS._RsGeom(pipe.coarse, DIMS)
    cb = b["compact"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t_max = float(np.linalg.norm(scene.hi - scene.lo))
    ev[0].record()
    RS.launch_sample_update(view.bvh, g, cb, cfg.sampling, pipe.frame, t_max, prev=pipe.fine.data,
                            accum=pipe.accum, out=pipe.fine.data)
    ev[1].record()
    torch.cuda.synchronize()
    sample_ms = ev[0].elapsed_time(ev[1])
    rays = masked * args.rays

    kernels_ms = {"jfa_pass_total": jfa_ms, "sample_update": sample_ms}
    traffic_b, traffic_src = jfa_traffic()
    dominant = "sample_update" if sample_ms > jfa_ms else "jfa_pass (schedule)"
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": False, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
        "dtype": "f64+i32",
        "data": "synthetic: reference-identical procedural sphere_plane scene (1,282 triangles)",
        "config": workload(args.rays),
        "layout": {"parallelism": (f"z-slab x{world} (NCCL P2P halos per JFA pass, coarse 1-plane "
                                   "halo, fine slabs gathered for DL)") if sharded else
                   (f"replicas x{world}" if world > 1 else "1 GPU"),
                   "frame_overlap": (None if sharded else
                                     "V + JF of frame f+1 on a flood stream during frame f's RT/DL "
                                     "(static scene, BVH <= 16 MB, double-buffered); frame_stages_ms "
                                     "come from one serial event-timed frame; e2e uploads frame f+1's "
                                     "mesh while frame f traces (upload_mesh)")},
        "frame_stages_ms": {k: round(v, 4) for k, v in stages_ms.items()},
        "masked_texels": masked, "rays_per_frame": rays,
        "rays_per_s": round(rays / (sample_ms * 1e-3), 1),
        "jfa": {"ms": round(jfa_ms, 4), "passes": len(offs),
                "per_pass_ms": [round(float(x), 4) for x in per_pass],
                "per_pass_note": "each pass launched alone (pass kernel + tie fix-up); 'ms' is the "
                                 "whole schedule as the frame runs it (sparse early passes)",
                "gvox_pass_per_s": round(gvox, 2), "achieved_gbs": round(jfa_gbs, 1),
                "hbm_frac": round(jfa_gbs / hbm, 4), "weights": list(w),
                "algorithmic_bytes_per_voxel_pass": 8},
        "roofline": {"kernel": "jfa_pass5_kernel (K2 v5, dense passes k <= 16; launch_ms includes "
                               "its tie fix-up kernel)", "bound": "hbm",
                     "binding_limit": "instruction issue (see issue_roofline)",
                     "achieved": round(n_cells * 8 / (pass_ms * 1e-3) / 1e9, 1),
                     "peak": hbm, "unit": "GB/s",
                     "frac": round(n_cells * 8 / (pass_ms * 1e-3) / 1e9 / hbm, 4),
                     "launch_ms": round(pass_ms, 4),
                     "traffic": traffic_b, "traffic_unit": "bytes/launch (DRAM read+write, ncu)",
                     "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": n_cells * 8, "peak_source": hbm_src,
                     "dominant_kernel": dominant,
                     "issue_roofline": issue_roofline(n_cells, pass_ms, ck),
                     "note": "frac is against HBM as the contract asks; the pass is bound by its two "
                             "half-rate integer pipes (ALU + FMA, ~85 % issue): 27 exact candidates "
                             "per cell at 6 instructions each, 3 per pipe "
                             "(candidate_floor_instr_per_cell), put its issue floor far above the "
                             "HBM floor (DESIGN.md section 7)"},
        "roofline_sampler": sampler_roofline(rays, sample_ms),
        "kernels_ms": {k: round(v, 4) for k, v in kernels_ms.items()},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": ck,
    }
    return out


def cpu_runner(x):
    """The CPU oracle (OpenMP over every host core) set up for full C3 frames."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    from paper_2210_06160_b200 import scenes as S
    from paper_2210_06160_b200.geometry import make_mesh

    scene = S.get_scene("sphere_plane")
    verts, tris, alb, base = [], [], [], 0
    for inst in scene.instances:
        verts.append(inst.mesh.vertices)
        tris.append(inst.mesh.triangles + base)
        alb.append(np.tile(np.asarray(inst.albedo, np.float32), (inst.mesh.num_triangles, 1)))
        base += len(inst.mesh.vertices)
    mesh = make_mesh(np.vstack(verts), np.vstack(tris))
    return O.CpuFrameRunner(mesh, np.vstack(alb), scene.bounds, DIMS, scene.camera,
                            scene.light.unit(), scene.light.angular_radius, x=x)


def run_cpu_baseline(args):
    """cpu_baseline: one warm-up + --cpu-frames whole C3 frames on the oracle
    (~3 s each on 16 host threads), median ms/frame."""
    R = cpu_runner(args.rays)
    R.step()
    ts = [R.step() * 1e3 for _ in range(max(1, args.cpu_frames))]
    return {"value": round(float(np.median(ts)), 1), "unit": UNIT, "cores": R.threads,
            "kind": "port",
            "sample": f"{len(ts)} whole C3 frames after 1 warm-up frame (V + 9-pass JFA + s2sdf + "
                      "resample/mask + 76.7 M rays + Eq.1 + G-buffer + 240x180 march, temporal "
                      "state carried), median; C oracle, OpenMP; BVH built once (static scene)"}


def cpu_baseline_subprocess(args):
    """The cpu_baseline leg in its own process (no GPU state, no allocator
    pressure on the timed GPU process)."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-baseline-only",
           "--rays", str(args.rays), "--cpu-frames", str(args.cpu_frames)]
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    for ln in reversed(r.stdout.splitlines()):
        if ln.startswith("{"):
            return json.loads(ln)
    return {"value": None, "unit": UNIT, "kind": "port", "error": (r.stderr or "")[-400:]}


# ------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference's CPU implementation of the path on this box's host cores:
    every step is one whole C3 frame (nothing sampled, nothing extrapolated)."""
    R = cpu_runner(args.rays)
    for _ in range(args.warmup):
        R.step()
    t0 = time.perf_counter()
    ts = [R.step() for _ in range(args.steps)]
    wall = time.perf_counter() - t0
    value = float(np.mean(ts)) * 1e3
    cpu = {"value": round(value, 1), "unit": UNIT, "cores": R.threads, "kind": "port",
           "sample": f"{args.steps} whole C3 frames after {args.warmup} warm-up frames (V + 9-pass "
                     "JFA + s2sdf + resample/mask + 76.7 M rays + Eq.1 + G-buffer + 240x180 march, "
                     "temporal state carried); C oracle, OpenMP; BVH built once (static scene)"}
    return {"impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(value, 1), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+i32",
            "data": "synthetic: reference-identical procedural sphere_plane scene (1,282 triangles)",
            "config": workload(args.rays), "layout": f"{R.threads} host threads",
            "timed_wall_s": round(wall, 2), "cpu_baseline": cpu,
            "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse()
    if args.cpu_baseline_only:
        print(json.dumps(run_cpu_baseline(args)), flush=True)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun ourselves
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                  f"--master-port={_free_port()}", str(Path(__file__).resolve()),
                                  *sys.argv[1:]])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    group = world > 1 or args.sharded
    if group:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu:
            out["cpu_baseline"] = cpu_baseline_subprocess(args)
        print(json.dumps(out), flush=True)
    if group:
        import torch.distributed as tdist

        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
