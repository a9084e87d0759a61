// jfa3.cuh -- K2 v3: select-free 27-tap pass for grids <= 512 per axis.
//
// Same work decomposition as jfa2.cuh (x-streaming register tiles, incremental
// integer keys), but every output keeps FIVE running minima instead of a
// compare/select chain:
//
//     e_k = 1024 * Key + L_k,   L_k in [0, 1023] an exact offset field of d = s - x
//     L_1 = dz + 512,  L_2 = 511 - dz,  L_3 = dy + 512,  L_4 = 511 - dy,  L_5 = dx + 512
//
// (|d| <= 511 because every axis has <= 512 cells; |Key| <= qmax < 2^21 so
// 1024 Key + L fits int32 -- see jfa3_ok).  The min of each e_k first minimises
// Key, so all five share Key_min and their low bits give, over the seeds that
// reach Key_min, min dz, max dz, min dy, max dy and min dx.  If dz and dy are
// single-valued, every such seed has the same |dx| (same Key), i.e. the set is
// {s} or a mirror pair with bit-identical fp64 d2, and the reference's rule
// (fp64 d2, then lexicographic; jfa.py:116-124) picks the smaller dx: the
// winner is x + (dx_min, dy, dz), rebuilt from the keys -- no argmin
// bookkeeping at all.  If dz or dy differ, two different seeds tie on the
// integer key: the cell goes to the exact fix-up list (jfa_fixup_kernel).
// Each candidate costs 5 adds + 2.5 three-input mins (VIMNMX3), spread over
// the FMA and ALU pipes, instead of ~8 ALU compare/select instructions.
#pragma once
#include "jfa2.cuh"

#define JFA3_EMPTY_B ((1 << 21) - 8)  // key base of EMPTY taps: above every real |Key|

namespace rtsdf {

template <int RY, bool FINAL, bool SLAB>
__global__ void __launch_bounds__(128) jfa_pass3_kernel(PlaneSrc src, int32_t* __restrict__ dst,
                                                        float* __restrict__ dst_sdf, JfaGeom g,
                                                        Jfa2Task T, double beta,
                                                        int64_t* __restrict__ empty_count,
                                                        JfaFixList fix) {
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
    const int i_first = g.x0 + ri + si * L * k;
    const int i_end = g.x0 + g.nxl;
    if (i_first >= i_end) return;
    const int z = zb * 32 + lane;
    const bool zok = z < g.nz;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int j_base = rj + gj * RY * k;
    const int cz = -2 * g.wz * z;
    const int gxk = 2 * g.wx * k, gyk = 2 * g.wy * k;

    // e[key][slot][row]
    int e[5][3][RY];
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
        for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int b = 0; b < RY; ++b) e[q][s][b] = 0x7fffffff;

    int offs[RY + 2][3];
    unsigned okmask = 0;
#pragma unroll
    for (int bt = 0; bt < RY + 2; ++bt) {
        const int tj = j_base + (bt - 1) * k;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int tz = z + (c - 1) * k;
            const bool ok = zok && tj >= 0 && tj < g.ny && tz >= 0 && tz < g.nz;
            offs[bt][c] = ok ? tj * g.nz + tz : 0;
            okmask |= (ok ? 1u : 0u) << (bt * 3 + c);
        }
    }
    int32_t cur[RY + 2][3], nxt[RY + 2][3];
    auto load_plane = [&](int a, int32_t(&vals)[RY + 2][3]) {
        const int pi = i_first + a * k;
        const int32_t* pl = src.local;
        unsigned m = 0;
        if (pi >= 0 && pi < g.nx && a <= L) {
            const int32_t* q = SLAB ? plane_ptr(src, g, pi, plane) : src.local + (int64_t)pi * plane;
            if (q != nullptr) {
                pl = q;
                m = okmask;
            }
        }
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                vals[bt][c] = (m >> (bt * 3 + c)) & 1u ? __ldg(pl + offs[bt][c]) : RTSDF_EMPTY;
    };
    load_plane(-1, cur);

    int empties = 0;
    for (int a = -1; a <= L; ++a) {
        if (a >= 1 && i_first + (a - 1) * k >= i_end) break;
        load_plane(a + 1, nxt);
        const int ia = i_first + a * k;  // tap plane
        const int cx = -2 * g.wx * ia;
#pragma unroll
        for (int bt = -1; bt <= RY; ++bt) {
            const int jt = j_base + bt * k;  // tap row
            const int cy = -2 * g.wy * jt;
#pragma unroll
            for (int c = -1; c <= 1; ++c) {
                const int32_t v = cur[bt + 1][c + 1];
                if (__all_sync(0xffffffffu, v == RTSDF_EMPTY)) continue;
                const bool ok = v != RTSDF_EMPTY;
                const int sx = unpack_i(v), sy = unpack_j(v), sk = unpack_k(v);
                const int B0 = sx * (g.wx * sx + cx) + sy * (g.wy * sy + cy) + sk * (g.wz * sk + cz);
                // EMPTY: a base above every real key (|Key| < 2^20), no increments
                const int B = ok ? B0 : JFA3_EMPTY_B;
                const int Gx = ok ? gxk * sx : 0, Gy = ok ? gyk * sy : 0;
                const int E = 1024 * B;
                const int dz = sk - z, dy = sy - jt, dx = sx - ia;  // relative to (tap plane, tap row)
                const int base[5] = {E + dz + 512, E + 511 - dz, E + dy + 512, E + 511 - dy,
                                     E + dx + 512};
                const int X = 1024 * Gx, Y = 1024 * Gy;
                // e_q(da, db) = base_q - da * (X + kx_q) - db * (Y + ky_q); da = a' - a, db = b' - bt
                const int ix[5] = {X, X, X, X, X + k};
                const int iy[5] = {Y, Y, Y + k, Y - k, Y};
#pragma unroll
                for (int q = 0; q < 5; ++q) {
                    const int rs[3] = {base[q] + ix[q], base[q], base[q] - ix[q]};  // slot 0,1,2
#pragma unroll
                    for (int s = 0; s < 3; ++s) {
#pragma unroll
                        for (int db = -1; db <= 1; ++db) {
                            const int b = bt + db;
                            if (b < 0 || b >= RY) continue;
                            const int ev = db == 0 ? rs[s] : (db < 0 ? rs[s] + iy[q] : rs[s] - iy[q]);
                            e[q][s][b] = min(e[q][s][b], ev);
                        }
                    }
                }
            }
        }
        // output a - 1 (slot 0) complete
        const int oa = a - 1;
        const int oi = i_first + oa * k;
        if (oa >= 0 && oa < L && oi < i_end) {
#pragma unroll
            for (int b = 0; b < RY; ++b) {
                const int oj = j_base + b * k;
                const bool live = zok && oj < g.ny;
                const int64_t cell = (int64_t)(oi - g.x0) * plane + (int64_t)oj * g.nz + z;
                const int e1 = e[0][0][b];
                const bool none = e1 >= JFA3_EMPTY_B * 1024 - 4096;  // only EMPTY taps
                const int dzmin = (e1 & 1023) - 512, dzmax = 511 - (e[1][0][b] & 1023);
                const int dymin = (e[2][0][b] & 1023) - 512, dymax = 511 - (e[3][0][b] & 1023);
                const int dxmin = (e[4][0][b] & 1023) - 512;
                const int32_t w = none ? RTSDF_EMPTY : pack_ijk(oi + dxmin, oj + dymin, z + dzmin);
                const bool flag = live && !none && (dzmin != dzmax || dymin != dymax);
                if (live) {
                    if (FINAL) {
                        empties += none;
                        double d2 = center_d2(-dxmin, -dymin, -dzmin, g.hx, g.hy, g.hz);
                        dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
                    } else {
                        dst[cell] = w;
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, flag);
                if (m) {
                    int64_t bse = 0;
                    if (lane == 0) bse = (int64_t)atomicAdd((unsigned long long*)fix.count,
                                                            (unsigned long long)__popc(m));
                    bse = __shfl_sync(0xffffffffu, bse, 0);
                    if (flag) {
                        int64_t slot = bse + __popc(m & ((1u << lane) - 1));
                        if (slot < fix.cap) fix.cells[slot] = (int32_t)cell;
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 5; ++q)
#pragma unroll
            for (int b = 0; b < RY; ++b) {
                e[q][0][b] = e[q][1][b];
                e[q][1][b] = e[q][2][b];
                e[q][2][b] = 0x7fffffff;
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

// v3 applies when every axis has <= 512 cells (|d| <= 511) and |Key| <= qmax
// stays below the EMPTY base (1024 * base + L must fit int32).
inline bool jfa3_ok(const JfaGeom& g) {
    if (g.nx > 512 || g.ny > 512 || g.nz > 512) return false;
    double qmax = (double)g.wx * (g.nx - 1) * (g.nx - 1) + (double)g.wy * (g.ny - 1) * (g.ny - 1) +
                  (double)g.wz * (g.nz - 1) * (g.nz - 1);
    return qmax < (double)(JFA3_EMPTY_B - 8);
}

}  // namespace rtsdf
