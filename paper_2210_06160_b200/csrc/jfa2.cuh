// jfa2.cuh -- K2 v2: the 27-tap pass as x-streaming register tiles with
// incremental integer keys (INT mode, exact; see jfa.cu header for why the
// integer order is the reference's fp64 order).
//
// Work unit (one warp): 32 consecutive z (one per lane) x a chain of RY rows
// j0, j0 + k, ..., j0 + (RY-1)k x a segment of L planes i0, i0 + k, ...,
// i0 + (L-1)k of one residue class.  With offset k every tap of an output in
// the unit is itself on the unit's lattice (or its one-step halo), so each
// plane of (RY + 2) x 3 taps is loaded ONCE and folded into every output that
// sees it: 3 planes in flight x RY rows.
//
// For a loaded seed s at tap plane a / tap row bt, the key of output (a', b')
//     Key = |s|^2_w - 2 w . (x * s) = q(s, x) - |x|^2_w
// is B - (a' - a) Gx - (b' - bt) Gy with B, Gx = 2 wx k si, Gy = 2 wy k sj
// computed once per value: every candidate costs one IADD3 plus the compare.
// The minimum integer key is the reference's fp64 minimum; an integer tie
// between different seeds (a few % of cells in the late passes) takes a rare
// branch that applies the reference's fp64 rule (jfa.py:116-124) in place.
#pragma once
#include "common.cuh"

namespace rtsdf {

struct Jfa2Task {
    int nzb, jres, jgroups, ires, isegs, L;
};

__device__ __forceinline__ void jfa2_consider(int K, int32_t v, int& Km, int32_t& W, int oi,
                                              int oj, int oz, double hx, double hy, double hz) {
    if (K < Km) {
        Km = K;
        W = v;
    } else if (K == Km && v != W) {  // rare: integer tie between distinct seeds
        double dv = center_d2(oi - unpack_i(v), oj - unpack_j(v), oz - unpack_k(v), hx, hy, hz);
        double dw = center_d2(oi - unpack_i(W), oj - unpack_j(W), oz - unpack_k(W), hx, hy, hz);
        if (dv < dw || (dv == dw && v < W)) W = v;
    }
}

template <int RY, bool FINAL, bool SLAB>
__global__ void __launch_bounds__(128) jfa_pass2_kernel(PlaneSrc src, int32_t* __restrict__ dst,
                                                        float* __restrict__ dst_sdf, JfaGeom g,
                                                        Jfa2Task T, double beta,
                                                        int64_t* __restrict__ empty_count) {
    const int lane = threadIdx.x & 31;
    int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t total = (int64_t)T.nzb * T.jres * T.jgroups * T.ires * T.isegs;
    if (t >= total) return;
    const int zb = (int)(t % T.nzb);
    t /= T.nzb;
    const int jslot = (int)(t % ((int64_t)T.jres * T.jgroups));
    const int islot = (int)(t / ((int64_t)T.jres * T.jgroups));
    const int rj = jslot % T.jres, gj = jslot / T.jres;
    const int ri = islot % T.ires, si = islot / T.ires;
    const int k = g.offset;
    const int L = T.L;
    const int i_first = g.x0 + ri + si * L * k;  // global plane of output a = 0
    const int i_end = g.x0 + g.nxl;              // outputs only on owned planes
    if (i_first >= i_end) return;
    const int z = zb * 32 + lane;
    const bool zok = z < g.nz;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int j_base = rj + gj * RY * k;  // row of output b = 0
    const int cz = -2 * g.wz * z;
    const int gxk = 2 * g.wx * k, gyk = 2 * g.wy * k;

    int Km[3][RY];
    int32_t W[3][RY];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int b = 0; b < RY; ++b) {
            Km[s][b] = 0x7fffffff;
            W[s][b] = RTSDF_EMPTY;
        }

    // the (RY + 2) x 3 taps of one plane, loaded as independent (predicated)
    // loads; the next plane is fetched while the current one is folded in
    int32_t cur[RY + 2][3], nxt[RY + 2][3];
    auto load_plane = [&](int a, int32_t (&vals)[RY + 2][3]) {
        const int pi = i_first + a * k;
        const int32_t* pl = nullptr;
        if (pi >= 0 && pi < g.nx && a <= L)
            pl = SLAB ? plane_ptr(src, g, pi, plane) : src.local + (int64_t)pi * plane;
#pragma unroll
        for (int bt = -1; bt <= RY; ++bt) {
            const int tj = j_base + bt * k;
            const bool rok = pl != nullptr && tj >= 0 && tj < g.ny && zok;
#pragma unroll
            for (int c = -1; c <= 1; ++c) {
                const int tz = z + c * k;
                vals[bt + 1][c + 1] = (rok && tz >= 0 && tz < g.nz)
                                          ? __ldg(pl + (int64_t)tj * g.nz + tz)
                                          : RTSDF_EMPTY;
            }
        }
    };
    load_plane(-1, cur);

    int empties = 0;
    // tap planes a = -1 .. L; after plane a, output a - 1 is complete
    for (int a = -1; a <= L; ++a) {
        const int pi = i_first + a * k;        // tap plane (global)
        if (a >= 1 && i_first + (a - 1) * k >= i_end) break;  // no further outputs
        load_plane(a + 1, nxt);
        const int cx = -2 * g.wx * pi;
        {
#pragma unroll
            for (int bt = -1; bt <= RY; ++bt) {
                const int tj = j_base + bt * k;
                const int cy = -2 * g.wy * tj;
#pragma unroll
                for (int c = -1; c <= 1; ++c) {
                    const int32_t v = cur[bt + 1][c + 1];
                    if (v == RTSDF_EMPTY) continue;
                    const int sx = unpack_i(v), sy = unpack_j(v), sk = unpack_k(v);
                    // B = Key at (tap plane, tap row, this lane's z)
                    const int B = sx * (g.wx * sx + cx) + sy * (g.wy * sy + cy) + sk * (g.wz * sk + cz);
                    const int Gx = gxk * sx, Gy = gyk * sy;
#pragma unroll
                    for (int s = 0; s < 3; ++s) {  // slot s <-> output a' = a - 1 + s
                        const int da = s - 1;       // a' - a
                        const int oa = a + da;
                        if (oa < 0 || oa >= L) continue;
#pragma unroll
                        for (int db = -1; db <= 1; ++db) {  // output row b' = bt + db
                            const int b = bt + db;
                            if (b < 0 || b >= RY) continue;
                            const int K = B - da * Gx - db * Gy;
                            jfa2_consider(K, v, Km[s][b], W[s][b], i_first + oa * k,
                                          j_base + b * k, z, g.hx, g.hy, g.hz);
                        }
                    }
                }
            }
        }
        // output a - 1 (slot 0) is complete
        const int oa = a - 1;
        const int oi = i_first + oa * k;
        if (oa >= 0 && oa < L && oi < i_end && zok) {
#pragma unroll
            for (int b = 0; b < RY; ++b) {
                const int oj = j_base + b * k;
                if (oj >= g.ny) continue;
                const int64_t cell = (int64_t)(oi - g.x0) * plane + (int64_t)oj * g.nz + z;
                const int32_t w = W[0][b];
                if (FINAL) {
                    empties += w == RTSDF_EMPTY;
                    double d2 = center_d2(oi - unpack_i(w), oj - unpack_j(w), z - unpack_k(w),
                                          g.hx, g.hy, g.hz);
                    dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
                } else {
                    dst[cell] = w;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < RY; ++b) {
            Km[0][b] = Km[1][b];
            W[0][b] = W[1][b];
            Km[1][b] = Km[2][b];
            W[1][b] = W[2][b];
            Km[2][b] = 0x7fffffff;
            W[2][b] = RTSDF_EMPTY;
        }
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt)
#pragma unroll
            for (int c = 0; c < 3; ++c) cur[bt][c] = nxt[bt][c];
    }
    if (FINAL && empty_count) {
        for (int o = 16; o; o >>= 1) empties += __shfl_xor_sync(0xffffffffu, empties, o);
        if (lane == 0 && empties) atomicAdd((unsigned long long*)empty_count, (unsigned long long)empties);
    }
}

}  // namespace rtsdf
