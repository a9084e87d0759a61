"""The device directions' cos / sin (csrc/glibc_sincos.cuh) vs the host libm.

The reference draws every ray direction with the host libm's cos/sin
(/root/reference/pkg/src/sdfshadow/rng.py:53).  glibc_sincos.cuh restates
glibc 2.39's FMA build of them (__sin_fma / __cos_fma) step by step; it
compiles for the host too, so this CPU test builds it with g++
(-ffp-contract=off, explicit fma) and compares it bit for bit with the host
libm (through the oracle's libm_sincos) on:

  * 2^22 arguments phi = 2 pi v, v = k 2^-53 -- the only form the directions
    take (rng.py:52);
  * 2^20 log-uniform magnitudes in [2^-40, 2^26] of both signs (every branch:
    |x| < 2^-26, Taylor, table, the pi/2 - x path, reduce_sincos);
  * 4096 neighbours on both sides of every branch threshold and of every
    table knot (k + 1/2) / 128.

The GPU tests check the device build of the same code against the libm and
against the reference's own golden direction tables.
"""

from __future__ import annotations

import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

SRC = r"""
#include "glibc_sincos.cuh"
extern "C" void gs_many(const double* x, long n, double* s, double* c) {
    for (long i = 0; i < n; ++i) {
        s[i] = rtsdf::gs::glibc_sin(x[i]);
        c[i] = rtsdf::gs::glibc_cos(x[i]);
    }
}
"""


@pytest.fixture(scope="module")
def host_gs(tmp_path_factory):
    d = tmp_path_factory.mktemp("gs")
    (d / "gs.cpp").write_text(SRC)
    so = d / "libgs.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared",
                    "-fPIC", "-I", str(ROOT / "paper_2210_06160_b200" / "csrc"), "-o", str(so),
                    str(d / "gs.cpp"), "-lm"], check=True)
    lib = C.CDLL(str(so))
    lib.gs_many.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]

    def run(x):
        x = np.ascontiguousarray(x, np.float64)
        s, c = np.empty_like(x), np.empty_like(x)
        lib.gs_many(x.ctypes.data, x.size, s.ctypes.data, c.ctypes.data)
        return s, c

    return run


def _bits_equal(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _check(host_gs, x):
    s, c = host_gs(x)
    ws, wc = O.libm_sincos(x)
    bad = ~((s.view(np.uint64) == ws.view(np.uint64)) & (c.view(np.uint64) == wc.view(np.uint64)))
    assert not bad.any(), [(float(v).hex(), float(a).hex(), float(b).hex())
                           for v, a, b in zip(x[bad][:5], s[bad][:5], ws[bad][:5])]


def test_direction_arguments(host_gs):
    rng = np.random.default_rng(1)
    k = rng.integers(0, 2**53, size=1 << 22, dtype=np.uint64)
    phi = 6.283185307179586 * (k.astype(np.float64) * (1.0 / 9007199254740992.0))
    _check(host_gs, phi)


def test_all_branches_both_signs(host_gs):
    rng = np.random.default_rng(2)
    m = rng.random(1 << 20)
    e = rng.integers(-40, 27, size=m.size)
    x = np.ldexp(1.0 + m, e) * np.where(rng.random(m.size) < 0.5, -1.0, 1.0)
    x = x[np.abs(x) < 105414350.0]  # glibc's reduce_sincos range (branred not restated)
    _check(host_gs, x)


def test_thresholds_and_table_knots(host_gs):
    th = [2.0**-26, 2.0**-27, 0.126, 0.855469, 2.426265, np.pi / 4, np.pi / 2, np.pi,
          3 * np.pi / 2, 2 * np.pi, 6.283185307179586]
    th += [(k + 0.5) / 128 for k in range(110)]
    xs = []
    for t in th:
        base = np.float64(t)
        steps = np.arange(-2048, 2048, dtype=np.int64)
        v = (base.view(np.int64) + steps).view(np.float64)
        xs += [v, -v]
    _check(host_gs, np.concatenate(xs))


def test_outside_restated_range_is_nan(host_gs):
    s, c = host_gs(np.array([2.0e8, -3.0e9, np.inf]))
    assert np.isnan(s).all() and np.isnan(c).all()


SRC_NB = r"""
#include "glibc_sincos.cuh"
extern "C" void gs_nb_many(const double* x, long n, double* s, double* c) {
    for (long i = 0; i < n; ++i) rtsdf::gs::glibc_sincos_nb(x[i], s[i], c[i]);
}
"""


def test_branch_free_pair_equals_glibc(tmp_path):
    """glibc_sincos_nb (the sampler's straight-line (sin, cos)) == libm sin, cos
    for every non-negative argument form it is used on."""
    (tmp_path / "nb.cpp").write_text(SRC_NB)
    so = tmp_path / "libnb.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared",
                    "-fPIC", "-I", str(ROOT / "paper_2210_06160_b200" / "csrc"), "-o", str(so),
                    str(tmp_path / "nb.cpp"), "-lm"], check=True)
    lib = C.CDLL(str(so))
    lib.gs_nb_many.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(3)
    k = rng.integers(0, 2**53, size=1 << 22, dtype=np.uint64)
    parts = [6.283185307179586 * (k.astype(np.float64) * (1.0 / 9007199254740992.0)),
             np.ldexp(1.0 + rng.random(1 << 18), rng.integers(-60, 27, size=1 << 18)),
             np.array([0.0, 5e-324, 2.0**-1074 * 7])]
    for t in [2.0**-26, 2.0**-27, 0.126, 0.855469, 2.426265, np.pi / 2, np.pi, 2 * np.pi] + \
            [(q + 0.5) / 128 for q in range(110)]:
        parts.append((np.float64(t).view(np.int64) + np.arange(-2048, 2048)).view(np.float64))
    x = np.concatenate(parts)
    x = x[(x >= 0) & (x < 105414350.0)]
    s, c = np.empty_like(x), np.empty_like(x)
    lib.gs_nb_many(x.ctypes.data, x.size, s.ctypes.data, c.ctypes.data)
    ws, wc = O.libm_sincos(x)
    np.testing.assert_array_equal(s.view(np.uint64), ws.view(np.uint64))
    np.testing.assert_array_equal(c.view(np.uint64), wc.view(np.uint64))
