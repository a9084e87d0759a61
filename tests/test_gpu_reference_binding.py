"""INTEGRATION.md §2 in practice: the UNMODIFIED reference package (installed
into baseline/_ref by `pip install --target baseline/_ref`, which travels to
the GPU box) with ONE numba kernel swapped for the C-ABI entry that replaces
it -- jfa.py:136's `_jfa_step_kernel(...)` -> `rtsdf_jfa_step` through ctypes,
exactly as the INTEGRATION.md binding shows -- gives the reference's own
results: seeds of every pass schedule and the reference pipeline's frame.

Skipped when baseline/_ref is absent (it is git-ignored; `__graft_entry__`
documents the install).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from common import digest, golden

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sdfshadow():
    if not (REF / "sdfshadow").exists():
        pytest.skip("baseline/_ref (the pip-installed reference) is not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtsdf_numba_cache")
    sys.path.insert(0, str(REF))
    try:
        import sdfshadow as ref
    except Exception as exc:  # numba missing on this box, ...
        pytest.skip(f"reference not importable: {exc}")
    return ref


def _binding():
    """INTEGRATION.md §2's sdfshadow/_b200.py, verbatim in substance."""
    lib = C.CDLL(str(ROOT / "paper_2210_06160_b200" / "librtsdf.so"))
    P, I, D, SZ = C.c_void_p, C.c_int, C.c_double, C.c_size_t
    lib.rtsdf_jfa_step.argtypes = [P, P, I, I, I, I, D, D, D, I, I, I, P, SZ, P]
    lib.rtsdf_jfa_ws_bytes.argtypes = [I, I, I]
    lib.rtsdf_jfa_ws_bytes.restype = SZ
    lib.rtsdf_seeds_linear_to_packed.argtypes = [P, P, I, I, I, P]
    lib.rtsdf_seeds_packed_to_linear.argtypes = [P, P, I, I, I, P]
    lib.rtsdf_last_error.restype = C.c_char_p
    calls = []

    def jfa_step_kernel(src_np, dst_np, offset, hx, hy, hz):
        from paper_2210_06160_b200.jfa import integer_weights

        nx, ny, nz = src_np.shape
        weights = integer_weights(float(hx), float(hy), float(hz), (nx, ny, nz))
        s = torch.cuda.current_stream().cuda_stream
        lin = torch.from_numpy(np.ascontiguousarray(src_np)).cuda()
        a, b = torch.empty_like(lin), torch.empty_like(lin)
        lib.rtsdf_seeds_linear_to_packed(P(lin.data_ptr()), P(a.data_ptr()), nx, ny, nz, P(s))
        ws = torch.empty(lib.rtsdf_jfa_ws_bytes(nx, ny, nz), dtype=torch.uint8, device="cuda")
        rc = lib.rtsdf_jfa_step(P(a.data_ptr()), P(b.data_ptr()), nx, ny, nz, int(offset), hx, hy,
                                hz, *weights, P(ws.data_ptr()), ws.numel(), P(s))
        if rc:
            raise RuntimeError(lib.rtsdf_last_error().decode())
        lib.rtsdf_seeds_packed_to_linear(P(b.data_ptr()), P(lin.data_ptr()), nx, ny, nz, P(s))
        dst_np[...] = lin.cpu().numpy()
        calls.append(int(offset))

    return jfa_step_kernel, calls


@pytest.mark.parametrize("name,dims", [("sphere", (64, 64, 64)), ("sphere_plane", (128, 128, 128))])
def test_reference_jfa_with_the_b200_pass_kernel(sdfshadow, monkeypatch, name, dims):
    ref = sdfshadow
    from sdfshadow import jfa as rjfa
    from sdfshadow import scenes as rscenes

    scene = rscenes.get_scene(name)
    vg = ref.voxelize(scene.view(0).mesh, dims, scene.bounds)
    want = rjfa.jfa_run(vg)  # numba
    kernel, calls = _binding()
    monkeypatch.setattr(rjfa, "_jfa_step_kernel", kernel)
    got = rjfa.jfa_run(vg)  # the reference's own jfa_run / jfa_step, our pass kernel
    assert calls == list(rjfa.jfa_offsets(dims))
    np.testing.assert_array_equal(got.seed, want.seed)
    if name == "sphere_plane":  # the fp64 tie cells of Appendix A (128^3)
        assert digest(got.seed) == golden()["sp128"]["seed"]


def test_reference_pipeline_frame_with_the_b200_pass_kernel(sdfshadow, monkeypatch):
    """sdfshadow.FramePipeline.advance (C1) with the swapped kernel == the golden frame."""
    ref = sdfshadow
    from sdfshadow import jfa as rjfa
    from sdfshadow import scenes as rscenes

    kernel, calls = _binding()
    monkeypatch.setattr(rjfa, "_jfa_step_kernel", kernel)
    cfg = ref.PipelineConfig(coarse_dims=(64, 64, 64), fine_dims=(64, 64, 64),
                             sampling=ref.SamplingParams(rays_per_frame=32, mask_distance=0.1,
                                                         decay_alpha=0.95, seed=0))
    pipe = ref.FramePipeline(rscenes.get_scene("sphere"), cfg)
    pipe.advance()
    g = golden()["c1.frame0"]
    assert digest(pipe.coarse.data) == g["coarse"]
    assert digest(pipe.fine.data) == g["fine"]
    assert len(calls) == 6
