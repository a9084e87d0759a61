// jfa4.cuh -- K2 v4: the 27-tap JFA pass (jfa.py:79-125) on residue-chain
// lanes with the z +- k candidates passed between neighbour lanes.
//
// Work unit (one warp): 32 lanes on consecutive positions of the z residue
// chains laid end to end (position q -> residue r, chain index p, z = r +
// p k), so a lane's z - k / z + k taps sit in its neighbour lanes; a chain of
// RY rows j0, j0 + k, ... (registers); a segment of L planes i0, i0 + k, ...
// streamed along x with 3 output slots in flight (v2's x/y structure).  Each
// lane loads and decodes only its OWN z column -- (RY + 2) / RY values per
// output instead of v2's 3 (RY + 2) / RY -- and receives its neighbours'
// decoded values (key base already moved to its own z, x / y increments,
// seed) by 4 + 4 shuffles; then every output evaluates its 27 candidates
// exactly as v2 does.  Warps overlap by one halo lane on each side (30 outputs
// per warp); a lane at a chain start / end takes itself as its missing
// neighbour.
//
// Taps outside the grid are CLAMPED to an in-grid tap of the same output
// instead of being predicated off: a clamped row / plane / neighbour re-reads
// the output's own row / plane / column, i.e. a candidate the output
// evaluates anyway, and a repeated (key, seed) pair cannot change the running
// minimum, the winner or the tie mark.  Keys always use the output's nominal
// coordinates, so the loads are unpredicated and branch-free.
//
// Keys and the integer-tie mark are v2's (jfa2.cuh jfa2_eval): the minimum
// integer key is the reference's fp64 minimum; a tie between DIFFERENT seeds
// marks the running key odd.  Marked cells are re-decided with the
// reference's own rule (fp64 d2, then lexicographic; jfa.py:108-124) by the
// same warp at the end of its task (one cell per lane, queued in shared
// memory), while the taps are still in L1/L2 -- no DRAM re-read of the source
// grid; a full queue spills to the global list that jfa_fixup_kernel drains
// after the pass.
#pragma once
#include "common.cuh"
#include "jfa2.cuh"

namespace rtsdf {

#define JFA4_KINIT 0x7ffffffe  // even, above every real (doubled) key (< 2^29)

struct Jfa4Task {
    int nz_pos;   // positions = nz (all residue chains end to end)
    int single;   // nz <= 32: one warp holds every position, no halo lanes
    int zw;       // z warps
    int lc;       // longest chain length ceil(nz / k) (>= 1)
    int nlong;    // residues of length lc
    int jres, jgroups, ires, isegs, L;
    int one, zero;
    int skip;     // warp-uniform all-EMPTY value skip (sparse inputs, k >= 16)
};

template <int RY, bool FINAL, bool SLAB, bool EXACT, bool NAT>
__global__ void __launch_bounds__(128, 4) jfa_pass4_kernel(PlaneSrc src, int32_t* __restrict__ dst,
                                                           float* __restrict__ dst_sdf, JfaGeom g,
                                                           Jfa4Task T, double beta,
                                                           int64_t* __restrict__ empty_count,
                                                           JfaFixList overflow) {
    __shared__ int32_t fixq_all[4][JFA_TIEQ];
    const int lane = threadIdx.x & 31;
    int32_t* fixq = fixq_all[(threadIdx.x >> 5) & 3];
    int nfix = 0;  // warp-uniform
    int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t total = (int64_t)T.zw * T.jres * T.jgroups * T.ires * T.isegs;
    if (t >= total) return;
    const int zwi = (int)(t % T.zw);
    t /= T.zw;
    const int jslot = (int)(t % ((int64_t)T.jres * T.jgroups));
    const int islot = (int)(t / ((int64_t)T.jres * T.jgroups));
    const int rj = jslot % T.jres, gj = jslot / T.jres;
    const int ri = islot % T.ires, si = islot / T.ires;
    const int k = g.offset;
    const int L = T.L;
    const int i_first = g.ox0 + ri + si * L * k;
    const int i_end = g.ox0 + g.onx;
    if (i_first >= i_end) return;

    // ---- z: chain position of this lane
    int q = T.single ? lane : zwi * 30 - 1 + lane;
    const bool own_q = T.single ? q < T.nz_pos : (lane >= 1 && lane <= 30 && q < T.nz_pos);
    q = q < 0 ? 0 : (q >= T.nz_pos ? T.nz_pos - 1 : q);
    int r, p, len;
    if (q < T.nlong * T.lc) {
        r = q / T.lc;
        p = q - r * T.lc;
        len = T.lc;
    } else {
        const int q2 = q - T.nlong * T.lc;
        r = T.nlong + q2 / (T.lc - 1);
        p = q2 - (r - T.nlong) * (T.lc - 1);
        len = T.lc - 1;
    }
    const int z = r + p * k;
    const bool own = own_q;
    // neighbour lanes on the same chain (else the lane stands in for itself)
    const int src_l = (lane > 0 && p > 0) ? lane - 1 : lane;
    const int src_r = (lane < 31 && p < len - 1) ? lane + 1 : lane;
    const bool has_l = src_l != lane, has_r = src_r != lane;

    const int64_t plane = (int64_t)g.ny * g.nz;
    const int j_base = rj + gj * RY * k;
    const int wsc = EXACT ? 1 : 2;
    const int wx = wsc * g.wx, wy = wsc * g.wy, wz = wsc * g.wz;
    const int one = T.one, zero = T.zero;
    const int cz = -2 * wz * z;
    const int gxk = 2 * wx * k, gyk = 2 * wy * k, gzk = 2 * wz * k;

    // clamped tap rows (task-uniform): row bt -> j_base + (bt - 1) k
    int roff[RY + 2];
    {
        int jlast = j_base;
#pragma unroll
        for (int b = 1; b < RY; ++b)
            if (j_base + b * k < g.ny) jlast = j_base + b * k;
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt) {
            int tj = j_base + (bt - 1) * k;
            tj = tj < 0 ? j_base : (tj >= g.ny ? jlast : tj);
            roff[bt] = tj * g.nz + z;
        }
    }
    auto plane_base = [&](int a) -> const int32_t* {
        int pi = i_first + a * k;
        if (pi < 0) pi = i_first;
        else if (pi >= g.nx) pi = pi - k;
        return SLAB ? plane_ptr(src, g, pi, plane) : src.local + (int64_t)pi * plane;
    };

    int Km[3][RY];
    int32_t W[3][RY];
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int b = 0; b < RY; ++b) {
            Km[s][b] = JFA4_KINIT;
            W[s][b] = RTSDF_EMPTY;
        }

    int32_t cur[RY + 2], nxt[RY + 2];
    {
        const int32_t* pl = plane_base(-1);
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt) cur[bt] = __ldg(pl + roff[bt]);
    }
    int empties = 0;
    int a_last = L - 1;
    if (i_first + a_last * k >= i_end) a_last = (i_end - 1 - i_first) / k;
    for (int a = -1; a <= a_last + 1; ++a) {
        if (a <= a_last) {
            const int32_t* pl = plane_base(a + 1);
#pragma unroll
            for (int bt = 0; bt < RY + 2; ++bt) nxt[bt] = __ldg(pl + roff[bt]);
        }
        const int cx = -2 * wx * (i_first + a * k);
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt) {
            const int32_t v = cur[bt];
            if (T.skip && __all_sync(0xffffffffu, v == RTSDF_EMPTY)) continue;
            const int sx = unpack_i(v), sy = unpack_j(v), sk = unpack_k(v);
            const int cy = -2 * wy * (j_base + (bt - 1) * k);
            const int B0 = sx * (wx * sx + cx) + sy * (wy * sy + cy) + sk * (wz * sk + cz);
            const int B = NAT || v != RTSDF_EMPTY ? B0 : JFA2_EMPTY_KEY;
            const int Gx = gxk * sx, Gy = gyk * sy, Gz = gzk * sk;
            // the neighbours' values, key base moved to this lane's z: the left
            // lane's seed sits at z - k relative to its own output, so its key at
            // z is its B - Gz; the right lane's is its B + Gz
            const int Bl0 = __shfl_sync(0xffffffffu, B - Gz, src_l);
            const int Br0 = __shfl_sync(0xffffffffu, B + Gz, src_r);
            const int Gxl = __shfl_sync(0xffffffffu, Gx, src_l), Gxr = __shfl_sync(0xffffffffu, Gx, src_r);
            const int Gyl = __shfl_sync(0xffffffffu, Gy, src_l), Gyr = __shfl_sync(0xffffffffu, Gy, src_r);
            const int32_t vl = __shfl_sync(0xffffffffu, v, src_l), vr = __shfl_sync(0xffffffffu, v, src_r);
            const int Bl = has_l ? Bl0 : B, Br = has_r ? Br0 : B;
            const int Bc[3] = {Bl, B, Br};
            const int Gxc[3] = {Gxl, Gx, Gxr};
            const int Gyc[3] = {Gyl, Gy, Gyr};
            const int32_t vc[3] = {vl, v, vr};
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // slot s <-> output plane a - 1 + s; row b <-> tap row bt - 1 + db
                const int Bs[3] = {Bc[c] + Gxc[c], Bc[c], Bc[c] - Gxc[c]};
#pragma unroll
                for (int s = 0; s < 3; ++s) {
#pragma unroll
                    for (int db = -1; db <= 1; ++db) {
                        const int b = bt - 1 + db;
                        if (b < 0 || b >= RY) continue;  // compile-time
                        const int K = db == 0 ? Bs[s] : (db < 0 ? Bs[s] + Gyc[c] : Bs[s] - Gyc[c]);
                        if (EXACT)
                            jfa2_eval_exact(K, vc[c], Km[s][b], W[s][b], zero);
                        else
                            jfa2_eval(K, vc[c], Km[s][b], W[s][b], one, zero);
                    }
                }
            }
        }
        // output plane a - 1 (slot 0) is complete
        const int oa = a - 1;
        if (oa >= 0) {
            const int oi = i_first + oa * k;
            const int64_t cbase = (int64_t)(oi - g.ox0) * plane + z;
#pragma unroll
            for (int b = 0; b < RY; ++b) {
                const int oj = j_base + b * k;
                const bool live = own && oj < g.ny;
                const int32_t w = W[0][b];
                const bool tie = !EXACT && live && w != RTSDF_EMPTY && (Km[0][b] & 1);
                const int64_t cell = cbase + (int64_t)oj * g.nz;
                if (live && !tie) {
                    if (FINAL) empties += w == RTSDF_EMPTY;
                    jfa_store_out<FINAL>(dst, dst_sdf, g, cell, oi, oj, z, w, beta);
                }
                if (!EXACT) {
                    // queue the tie cells; a full queue spills to the global list
                    // (re-decided by jfa_fixup_kernel after the pass) so that no
                    // fix-up runs while the tile's state is live in registers
                    const unsigned m = __ballot_sync(0xffffffffu, tie);
                    if (m) {
                        const int before = __popc(m & ((1u << lane) - 1));
                        if (nfix + __popc(m) <= JFA_TIEQ) {
                            if (tie) fixq[nfix + before] = (int32_t)cell;
                            nfix += __popc(m);
                        } else {
                            int64_t base = 0;
                            if (lane == __ffs(m) - 1)
                                base = (int64_t)atomicAdd((unsigned long long*)overflow.count,
                                                          (unsigned long long)__popc(m));
                            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
                            if (tie && base + before < overflow.cap)
                                overflow.cells[base + before] = (int32_t)cell;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < RY; ++b) {
            Km[0][b] = Km[1][b];
            W[0][b] = W[1][b];
            Km[1][b] = Km[2][b];
            W[1][b] = W[2][b];
            Km[2][b] = JFA4_KINIT;
            W[2][b] = RTSDF_EMPTY;
        }
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt) cur[bt] = nxt[bt];
    }
    if (!EXACT && nfix) {
        __syncwarp();
        jfa_flush_ties<FINAL, SLAB>(src, dst, dst_sdf, g, beta, fixq, nfix, lane);
    }
    if (FINAL && empty_count) {
        for (int o = 16; o; o >>= 1) empties += __shfl_xor_sync(0xffffffffu, empties, o);
        if (lane == 0 && empties) atomicAdd((unsigned long long*)empty_count, (unsigned long long)empties);
    }
}

}  // namespace rtsdf
