// jfa2.cuh -- K2 v2: the 27-tap pass as x-streaming register tiles with
// incremental integer keys (INT mode, exact; see jfa.cu header for why the
// integer order is the reference's fp64 order).
//
// Work unit (one warp): 32 consecutive z (one per lane) x a chain of RY rows
// j0, j0 + k, ..., j0 + (RY-1)k x a segment of L planes i0, i0 + k, ...,
// i0 + (L-1)k of one residue class.  With offset k every tap of an output in
// the unit is itself on the unit's lattice (or its one-step halo), so each
// plane of (RY + 2) x 3 taps is loaded ONCE (as independent loads, the next
// plane in flight while the current one is folded in) and folded into every
// output that sees it: 3 planes in flight x RY rows.
//
// For a loaded seed s at tap plane a / tap row bt, the key of output (a', b')
//     Key = |s|^2_w - 2 w . (x * s) = q(s, x) - |x|^2_w
// is B - (a' - a) Gx - (b' - bt) Gy with B, Gx = 2 wx k si, Gy = 2 wy k sj
// computed once per value: every candidate costs its key (one IMAD) plus the
// 5-instruction update of jfa2_eval (4 with jfa2_eval_exact).  The minimum
// integer key is the reference's fp64 minimum.  An integer tie between two
// DIFFERENT seeds (a few % of cells in the late passes) only marks the output
// (odd running key, jfa2_eval); marked cells are appended to a list and
// re-decided by jfa_fixup_kernel with the reference's own rule (fp64 d2, then
// lexicographic; jfa.py:108-124), so the hot loop has no fp64 and no
// divergent branch.
#pragma once
#include "common.cuh"

#ifndef JFA2_FULL_LOADS
#define JFA2_FULL_LOADS 0
#endif
#ifndef JFA2_MINB
#define JFA2_MINB 4  // 128 registers: 4 resident 128-thread blocks per SM
#endif

#ifndef JFA2_SKIP_MODE
#define JFA2_SKIP_MODE 1
#endif
#define JFA2_EMPTY_KEY (1 << 30)  // larger than any real (doubled) key: |key| < 2^29

namespace rtsdf {

struct Jfa2Task {
    int nzb, jres, jgroups, ires, isegs, L;
    int one, zero;  // = 1, 0 (opaque to ptxas, see jfa2_eval)
    int skip;       // pass input may hold all-EMPTY tap segments (k >= 16)
};

// One candidate against one output's running (Km, W).  Keys are even (the
// non-EXACT pass doubles the weights); an integer tie between a DIFFERENT seed
// and the running minimum marks Km odd.  An odd Km = 2m - 1 orders exactly
// like 2m against every (even) key, so later equal keys are neither smaller
// nor equal (already tied) and a strictly smaller key clears the mark: at the
// end Km is odd iff >= 2 distinct seeds share the minimum (and W, which a tie
// also overwrites, is then re-decided by the fix-up).  With
//     p = K <= Km  and  v != W
// both cases are one update: Km = min(Km - 1, K) (K < Km: K; K == Km: Km - 1)
// and W = v.  A repeat of the winner (v == W, hence K == Km) changes nothing.
// 6 instructions: the key, 2 predicate compares and IMNMX (ALU), Km - 1 and
// the predicated winner move as IMADs (FMA pipe; `one` / `zero` are opaque to
// ptxas, which would otherwise turn the moves into ALU selects).
__device__ __forceinline__ void jfa2_eval(int K, int32_t v, int& Km, int32_t& W, int one, int zero) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .s32 km1;\n\t"
        "setp.le.s32 p, %2, %0;\n\t"
        "setp.ne.and.s32 p, %3, %1, p;\n\t"
        "mad.lo.s32 km1, %0, %4, -1;\n\t"
        "@p min.s32 %0, km1, %2;\n\t"
        "@p mad.lo.s32 %1, %1, %5, %3;\n\t}"
        : "+r"(Km), "+r"(W)
        : "r"(K), "r"(v), "r"(one), "r"(zero));
}

// EXACT mode (host-proven: every fp64 operation of center_d2 is exact for the
// grid's spacings and extents, e.g. dyadic spacings such as 4/512): fp64 d2 is
// then exactly proportional to the integer key, so the reference's rule
// (fp64 d2, then lexicographic) IS the lexicographic order of (key, packed
// seed) -- ties resolve in the hot loop, no flags, no fix-up.  (K, v) < (Km, W)
// with the seed compared unsigned (EMPTY = 0xffffffff is the largest): one
// 64-bit signed compare of {K : v} (key high, seed low -- the low word counts
// unsigned), i.e. ISETP.U32 + ISETP.EX, and the two moves as predicated IMADs
// on the FMA pipe: 5 instructions per candidate with its key.
__device__ __forceinline__ void jfa2_eval_exact(int K, int32_t v, int& Km, int32_t& W, int zero) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 a, b;\n\t"
        "mov.b64 a, {%3, %2};\n\t"
        "mov.b64 b, {%1, %0};\n\t"
        "setp.lt.s64 p, a, b;\n\t"
        "@p mad.lo.s32 %0, %0, %4, %2;\n\t"
        "@p mad.lo.s32 %1, %1, %4, %3;\n\t}"
        : "+r"(Km), "+r"(W)
        : "r"(K), "r"(v), "r"(zero));
}

struct JfaFixList {
    int32_t* cells;  // local linear cell indices needing the exact rule
    int64_t* count;  // device counter
    int64_t cap;
};

// Integer-tie cells of the v4 pass (jfa4.cuh) are queued per warp and
// re-decided at the end of its task (a full queue spills to the global list
// drained by jfa_fixup_kernel).  The same end-of-task queue in v2 measured
// slower than v2's separate fix-up kernel (C3 schedule 4.40 vs 3.66 ms: the
// latency-bound gathers stall warps that hold the SM), so v2 keeps the kernel.
#define JFA_TIEQ 256

// jfa.py:108-124 on the 27 taps of one cell, integer pre-filter (jfa2.cuh
// jfa_fixup_kernel's rule); returns the reference's seed.
template <bool SLAB>
__device__ __forceinline__ int32_t jfa_exact_cell(const PlaneSrc& src, const JfaGeom& g, int i,
                                                   int j, int z) {
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int k = g.offset;
    const int32_t* pl[3];
#pragma unroll
    for (int di = 0; di < 3; ++di) {
        const int qi = i + (di - 1) * k;
        pl[di] = nullptr;
        if (qi >= 0 && qi < g.nx)
            pl[di] = SLAB ? plane_ptr(src, g, qi, plane) : src.local + (int64_t)qi * plane;
    }
    const bool jok[3] = {j - k >= 0, true, j + k < g.ny};
    const bool zok[3] = {z - k >= 0, true, z + k < g.nz};
    int32_t c[27];
#pragma unroll
    for (int di = 0; di < 3; ++di)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj)
#pragma unroll
            for (int dk = 0; dk < 3; ++dk) {
                const bool ok = pl[di] != nullptr && jok[dj] && zok[dk];
                const int off = (j + (dj - 1) * k) * g.nz + z + (dk - 1) * k;
                c[(di * 3 + dj) * 3 + dk] = ok ? __ldg(pl[di] + off) : RTSDF_EMPTY;
            }
    auto ikey = [&](int32_t v) {
        const int dx = i - unpack_i(v), dy = j - unpack_j(v), dz = z - unpack_k(v);
        return v == RTSDF_EMPTY ? 0x7fffffff : g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
    };
    int km = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < 27; ++t) km = min(km, ikey(c[t]));
    int32_t best = RTSDF_EMPTY;
    double bd = 1e300;
#pragma unroll
    for (int t = 0; t < 27; ++t) {
        if (c[t] == RTSDF_EMPTY || c[t] == best || ikey(c[t]) != km) continue;
        const double d2 = center_d2(i - unpack_i(c[t]), j - unpack_j(c[t]), z - unpack_k(c[t]),
                                    g.hx, g.hy, g.hz);
        if (d2 < bd || (d2 == bd && best != RTSDF_EMPTY && c[t] < best)) {
            best = c[t];
            bd = d2;
        }
    }
    return best;
}

template <bool FINAL>
__device__ __forceinline__ void jfa_store_out(int32_t* dst, float* dst_sdf, const JfaGeom& g,
                                           int64_t cell, int i, int j, int z, int32_t w,
                                           double beta) {
    if (FINAL) {
        const double d2 = center_d2(i - unpack_i(w), j - unpack_j(w), z - unpack_k(w), g.hx, g.hy, g.hz);
        dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
    } else {
        dst[cell] = w;
    }
}

template <bool FINAL, bool SLAB>
__device__ __forceinline__ void jfa_flush_ties(const PlaneSrc& src, int32_t* dst, float* dst_sdf,
                                           const JfaGeom& g, double beta, const int32_t* q, int n,
                                           int lane) {
    const int64_t plane = (int64_t)g.ny * g.nz;
    for (int t = lane; t < n; t += 32) {
        const int32_t cell = q[t];  // slab-local linear cell (< 2^31)
        const int il = (int)(cell / plane);
        const int rem = (int)(cell - (int64_t)il * plane);
        const int j = rem / g.nz, z = rem - j * g.nz;
        const int i = g.ox0 + il;
        const int32_t w = jfa_exact_cell<SLAB>(src, g, i, j, z);
        jfa_store_out<FINAL>(dst, dst_sdf, g, cell, i, j, z, w, beta);
    }
    __syncwarp();
}

// NAT: the host proved that the packed EMPTY (-1) decodes to a virtual seed
// (4095, 1023, 1023) whose key exceeds every real seed's key at every cell of
// the grid (jfa.cu natural_empty_ok), so an EMPTY tap needs no select: it can
// neither win nor tie, and a run of EMPTY taps leaves (Km, W) = (init, EMPTY).
template <int RY, bool FINAL, bool SLAB, bool EXACT, bool NAT = false>
__global__ void __launch_bounds__(128, JFA2_MINB) jfa_pass2_kernel(PlaneSrc src, int32_t* __restrict__ dst,
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
    const int i_first = g.ox0 + ri + si * L * k;  // global plane of output a = 0
    const int i_end = g.ox0 + g.onx;              // outputs only on owned planes
    if (i_first >= i_end) return;
    const int z = zb * 32 + lane;
    const bool zok = z < g.nz;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int j_base = rj + gj * RY * k;  // row of output b = 0
    // non-EXACT: doubled weights, so every real key is even (jfa2_eval's tie mark)
    const int wsc = EXACT ? 1 : 2;
    const int wx = wsc * g.wx, wy = wsc * g.wy, wz = wsc * g.wz;
    const int one = T.one, zero = T.zero;
    const int cz = -2 * wz * z;
    const int gxk = 2 * wx * k, gyk = 2 * wy * k;

    int Km[3][RY];
    int32_t W[3][RY];  // winner (non-EXACT: Km odd = integer tie, jfa2_eval)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
        for (int b = 0; b < RY; ++b) {
            Km[s][b] = 0x7fffffff;
            W[s][b] = RTSDF_EMPTY;
        }

    // the in-plane offsets of the (RY + 2) x 3 taps and their validity are
    // loop invariants of the task: a plane load is 18 address adds + loads
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
            // slab mode: the prefetch can run one plane past the last output's
            // taps, which need not be resident -> treat as absent
            const int32_t* q = SLAB ? plane_ptr(src, g, pi, plane) : src.local + (int64_t)pi * plane;
            if (q != nullptr) {
                pl = q;
                m = okmask;
            }
        }
#if JFA2_FULL_LOADS
        if (m == (1u << (3 * (RY + 2))) - 1u) {  // interior plane (warp-uniform): plain loads
#pragma unroll
            for (int bt = 0; bt < RY + 2; ++bt)
#pragma unroll
                for (int c = 0; c < 3; ++c) vals[bt][c] = __ldg(pl + offs[bt][c]);
            return;
        }
#endif
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                vals[bt][c] = (m >> (bt * 3 + c)) & 1u ? __ldg(pl + offs[bt][c]) : RTSDF_EMPTY;
    };
    load_plane(-1, cur);

    int empties = 0;
    // tap planes a = -1 .. L; after plane a, output a - 1 is complete
    for (int a = -1; a <= L; ++a) {
        if (a >= 1 && i_first + (a - 1) * k >= i_end) break;  // no further outputs (uniform)
        load_plane(a + 1, nxt);
        const int cx = -2 * wx * (i_first + a * k);
        // Column-constant plane: every tap row holds the same seed in every lane
        // (seeds constant along y, e.g. above a floor).  A candidate's key
        // depends only on (seed, output), so the RY + 2 copies of a tap column
        // are one candidate per output: 3 columns x 3 slots x RY rows instead
        // of the 3 x 3 x 3 x RY tap/row pairs (repeats of a (key, seed) pair
        // cannot change the running minimum, the winner or the tie mark).
        // Only tried in the sparse early passes (k >= 64): after them, rows of
        // different residue classes hold different provisional seeds and the
        // test (15 compares + a vote per plane) almost never succeeds.
        bool ycon = k >= 64;
#pragma unroll
        for (int bt = 1; bt < RY + 2; ++bt)
#pragma unroll
            for (int c = 0; c < 3; ++c) ycon = ycon && cur[bt][c] == cur[0][c];
        if (k >= 64 && __all_sync(0xffffffffu, ycon)) {
            const int cy = -2 * wy * (j_base - k);  // tap row bt = -1
#pragma unroll
            for (int c = -1; c <= 1; ++c) {
                const int32_t v = cur[0][c + 1];
                if (__all_sync(0xffffffffu, v == RTSDF_EMPTY)) continue;
                const int sx = unpack_i(v), sy = unpack_j(v), sk = unpack_k(v);
                const int B0 = sx * (wx * sx + cx) + sy * (wy * sy + cy) + sk * (wz * sk + cz);
                const int B = NAT || v != RTSDF_EMPTY ? B0 : JFA2_EMPTY_KEY;
                const int Gx = gxk * sx, Gy = gyk * sy;
                const int Bs[3] = {B + Gx, B, B - Gx};
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    int K = Bs[s];
#pragma unroll
                    for (int b = 0; b < RY; ++b) {
                        K -= Gy;  // output row b = tap row -1 + (b + 1)
                        if (EXACT)
                            jfa2_eval_exact(K, v, Km[s][b], W[s][b], zero);
                        else
                            jfa2_eval(K, v, Km[s][b], W[s][b], one, zero);
                    }
                }
            }
        } else
#pragma unroll
        for (int bt = -1; bt <= RY; ++bt) {
            const int cy = -2 * wy * (j_base + bt * k);
#pragma unroll
            for (int c = -1; c <= 1; ++c) {
                const int32_t v = cur[bt + 1][c + 1];
#if JFA2_SKIP_MODE == 1
                // the all-EMPTY vote only in passes that can have EMPTY tap
                // segments (uniform branch on the task; dense passes keep the
                // per-tap region boundary, which ptxas schedules better)
                if (T.skip && __all_sync(0xffffffffu, v == RTSDF_EMPTY)) continue;
#else
                if (__all_sync(0xffffffffu, v == RTSDF_EMPTY)) continue;  // warp-uniform skip
#endif
                const int sx = unpack_i(v), sy = unpack_j(v), sk = unpack_k(v);
                const int B0 = sx * (wx * sx + cx) + sy * (wy * sy + cy) + sk * (wz * sk + cz);
                // EMPTY (-1) decodes to (4095, 1023, 1023): its increments stay bounded
                // (|Gx|, |Gy| < 2^23), so an EMPTY base of 2^30 can never beat a real
                // key (|key| < 2^29) -- no per-increment selects
                const int B = NAT || v != RTSDF_EMPTY ? B0 : JFA2_EMPTY_KEY;
                const int Gx = gxk * sx, Gy = gyk * sy;
                // K(a', b') = B - (a' - a) Gx - (b' - bt) Gy; slot s <-> a' = a - 1 + s
                const int Bs[3] = {B + Gx, B, B - Gx};
#pragma unroll
                for (int s = 0; s < 3; ++s) {
#pragma unroll
                    for (int db = -1; db <= 1; ++db) {
                        const int b = bt + db;
                        if (b < 0 || b >= RY) continue;  // compile-time
                        const int K = db == 0 ? Bs[s] : (db < 0 ? Bs[s] + Gy : Bs[s] - Gy);
                        if (EXACT)
                            jfa2_eval_exact(K, v, Km[s][b], W[s][b], zero);
                        else
                            jfa2_eval(K, v, Km[s][b], W[s][b], one, zero);
                    }
                }
            }
        }
        // output a - 1 (slot 0) is complete
        const int oa = a - 1;
        const int oi = i_first + oa * k;
        if (oa >= 0 && oa < L && oi < i_end) {
#pragma unroll
            for (int b = 0; b < RY; ++b) {
                const int oj = j_base + b * k;
                const bool live = zok && oj < g.ny;
                const int64_t cell = (int64_t)(oi - g.ox0) * plane + (int64_t)oj * g.nz + z;
                const int32_t wt = W[0][b];
                const bool tie = !EXACT && wt != RTSDF_EMPTY && (Km[0][b] & 1);
                const int32_t w = wt;
                if (live) {
                    if (FINAL) {
                        empties += w == RTSDF_EMPTY;
                        double d2 = center_d2(oi - unpack_i(w), oj - unpack_j(w), z - unpack_k(w),
                                              g.hx, g.hy, g.hz);
                        dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
                    } else {
                        dst[cell] = w;
                    }
                }
                // integer tie between distinct seeds: defer to the exact rule
                const bool flag = live && tie;
                const unsigned m = __ballot_sync(0xffffffffu, flag);
                if (m) {
                    int64_t base = 0;
                    if (lane == 0) base = (int64_t)atomicAdd((unsigned long long*)fix.count,
                                                             (unsigned long long)__popc(m));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (flag) {
                        int64_t slot = base + __popc(m & ((1u << lane) - 1));
                        if (slot < fix.cap) fix.cells[slot] = (int32_t)cell;
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

// Re-decide the flagged cells with the reference's exact rule (jfa.py:108-124).
// The 27 taps are gathered as independent loads first; the integer key then
// pre-filters them: a strictly larger integer key is a strictly larger exact
// d2, which fp64 rounding cannot invert (relative gap >= 2^-29), so the fp64
// argmin lies among the taps at the minimum integer key -- only those pay fp64.
#ifndef JFA_FIX_MINB
#define JFA_FIX_MINB 8  // latency bound: occupancy over registers (64 regs, measured best)
#endif
template <bool FINAL, bool SLAB>
__global__ void __launch_bounds__(128, JFA_FIX_MINB) jfa_fixup_kernel(PlaneSrc src, int32_t* __restrict__ dst,
                                                        float* __restrict__ dst_sdf, JfaGeom g,
                                                        double beta, JfaFixList fix, FastDiv dnz,
                                                        FastDiv dny) {
    const int64_t n = min(*fix.count, fix.cap);
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int k = g.offset;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        // local linear cell -> (i, j, z); 32-bit (cells <= 1024^3)
        const uint32_t cell = (uint32_t)fix.cells[q];
        const uint32_t row = fdiv(cell, dnz);
        const int z = (int)(cell - row * dnz.d);
        const uint32_t il = fdiv(row, dny);
        const int j = (int)(row - il * dny.d);
        const int i = g.ox0 + (int)il;
        const int32_t* pl[3];
#pragma unroll
        for (int di = 0; di < 3; ++di) {
            const int qi = i + (di - 1) * k;
            pl[di] = nullptr;
            if (qi >= 0 && qi < g.nx)
                pl[di] = SLAB ? plane_ptr(src, g, qi, plane) : src.local + (int64_t)qi * plane;
        }
        const bool jok[3] = {j - k >= 0, true, j + k < g.ny};
        const bool zok[3] = {z - k >= 0, true, z + k < g.nz};
        // all 27 taps as independent loads, then the integer pre-filter
        int32_t c[27];
#pragma unroll
        for (int di = 0; di < 3; ++di)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj)
#pragma unroll
                for (int dk = 0; dk < 3; ++dk) {
                    const bool ok = pl[di] != nullptr && jok[dj] && zok[dk];
                    const int off = (j + (dj - 1) * k) * g.nz + z + (dk - 1) * k;
                    c[(di * 3 + dj) * 3 + dk] = ok ? __ldg(pl[di] + off) : RTSDF_EMPTY;
                }
        // integer keys recomputed in the second loop (no key[27] array:
        // registers, not ALU, limit this latency-bound kernel)
        auto ikey = [&](int32_t v) {
            const int dx = i - unpack_i(v), dy = j - unpack_j(v), dz = z - unpack_k(v);
            return v == RTSDF_EMPTY ? 0x7fffffff : g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
        };
        int km = 0x7fffffff;
#pragma unroll
        for (int t = 0; t < 27; ++t) km = min(km, ikey(c[t]));
        int32_t best = RTSDF_EMPTY;
        double bd = 1e300;
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            if (c[t] == RTSDF_EMPTY || c[t] == best || ikey(c[t]) != km) continue;
            const double d2 = center_d2(i - unpack_i(c[t]), j - unpack_j(c[t]), z - unpack_k(c[t]),
                                        g.hx, g.hy, g.hz);
            if (d2 < bd || (d2 == bd && best != RTSDF_EMPTY && c[t] < best)) {
                best = c[t];
                bd = d2;
            }
        }
        if (FINAL)
            dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(bd), beta);
        else
            dst[cell] = best;
    }
}

// Re-decide the flagged cells of the v5 pass (jfa5.cuh).  The pass stored, for
// each flagged cell, W = a seed at the cell's minimum integer key K* (in the
// seed output; the FINAL pass in the free ping-pong buffer), so one loop over
// the 27 taps suffices: the candidates at K* are the seeds with that key, and
// the reference's rule (fp64 d2, then lexicographic; jfa.py:108-124) picks
// among them -- a strictly larger integer key is a strictly larger exact d2,
// which fp64 rounding cannot invert.  About a third of jfa_fixup_kernel's
// instructions (no separate minimum pass).
template <bool FINAL, bool SLAB>
__global__ void __launch_bounds__(128, JFA_FIX_MINB) jfa_fixup_w_kernel(PlaneSrc src, int32_t* __restrict__ wbuf,
                                                         float* __restrict__ dst_sdf, JfaGeom g,
                                                         double beta, JfaFixList fix, FastDiv dnz,
                                                         FastDiv dny) {
    __shared__ int32_t fix_lst[26 * 128];  // per-thread list of tied seeds (stride 128)
    const int64_t n = min(*fix.count, fix.cap);
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int k = g.offset;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t cell = (uint32_t)fix.cells[q];
        const uint32_t row = fdiv(cell, dnz);
        const int z = (int)(cell - row * dnz.d);
        const uint32_t il = fdiv(row, dny);
        const int j = (int)(row - il * dny.d);
        const int i = g.ox0 + (int)il;
        const int32_t w0 = wbuf[cell];
        const int32_t* pl[3];
#pragma unroll
        for (int di = 0; di < 3; ++di) {
            const int qi = i + (di - 1) * k;
            pl[di] = nullptr;
            if (qi >= 0 && qi < g.nx)
                pl[di] = SLAB ? plane_ptr(src, g, qi, plane) : src.local + (int64_t)qi * plane;
        }
        const bool jok[3] = {j - k >= 0, true, j + k < g.ny};
        const bool zok[3] = {z - k >= 0, true, z + k < g.nz};
        int32_t c[27];
#pragma unroll
        for (int di = 0; di < 3; ++di)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj)
#pragma unroll
                for (int dk = 0; dk < 3; ++dk) {
                    const bool ok = pl[di] != nullptr && jok[dj] && zok[dk];
                    const int off = (j + (dj - 1) * k) * g.nz + z + (dk - 1) * k;
                    c[(di * 3 + dj) * 3 + dk] = ok ? __ldg(pl[di] + off) : RTSDF_EMPTY;
                }
        auto ikey = [&](int32_t v) {
            const int dx = i - unpack_i(v), dy = j - unpack_j(v), dz = z - unpack_k(v);
            return g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
        };
        const int ks = ikey(w0);
        // the other seeds at K* (integer filter, uniform over the warp), listed in
        // shared memory; then the fp64 rule over the short list -- the divergent
        // fp64 work runs max-over-warp(list length) times, not once per tap
        int32_t* lst = fix_lst + threadIdx.x;
        int nl = 0;
#pragma unroll
        for (int t = 0; t < 27; ++t) {
            const int32_t v = c[t];
            const bool m = v != RTSDF_EMPTY && v != w0 && ikey(v) == ks;
            if (m) lst[(nl++) * 128] = v;
        }
        int32_t best = w0;
        double bd = center_d2(i - unpack_i(w0), j - unpack_j(w0), z - unpack_k(w0), g.hx, g.hy, g.hz);
        for (int q = 0; q < nl; ++q) {
            const int32_t v = lst[q * 128];
            const double d2 = center_d2(i - unpack_i(v), j - unpack_j(v), z - unpack_k(v), g.hx, g.hy, g.hz);
            if (d2 < bd || (d2 == bd && v < best)) {
                best = v;
                bd = d2;
            }
        }
        if (FINAL)
            dst_sdf[cell] = (float)__dsub_rn(__dsqrt_rn(bd), beta);
        else
            wbuf[cell] = best;
    }
}

}  // namespace rtsdf
