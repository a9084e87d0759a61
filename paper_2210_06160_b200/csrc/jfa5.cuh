// jfa5.cuh -- K2 v5: the 27-tap pass (jfa.py:79-125) as 3-D register tiles.
//
// Each THREAD owns an RY x ZT block of outputs in one (y, z) residue class of
// the offset-k lattice -- rows j = rj + (gj RY + b) k, columns z = rz +
// (gz ZT + m) k -- and streams the planes of its x residue class, i = ri +
// (si L + a) k, keeping three output planes (slots) in flight.  Per plane it
// loads the (RY + 2) x (ZT + 2) tap block ONCE, decodes each tap value ONCE
// (key base + three gradients) and folds it into every output of the 3 x 3 x 3
// neighbourhood it belongs to: (RY+2)(ZT+2) / (RY ZT) decodes per output
// (2.8 for 3 x 3) where v2 (one column per lane, jfa2.cuh) pays 4.5.
//
// Keys are v2's exact integer keys  K = |s|^2_w - 2 w.(x o s)  (doubled
// weights outside EXACT mode), built once per tap value at the tap's stencil
// position and moved to each output by three gradient adds (one IADD3):
//     K(out) = B - dx Gx - dy Gy - dz Gz,  G = 2 w k s,  d in {-1, 0, 1}.
// Update per candidate (jfa2.cuh's rule): p = K <= Km && v != W ->
// Km = min(Km - 1, K) (one VIADDMNMX), W = v; EXACT: lexicographic (K, seed).
//
// Taps outside the grid are CLAMPED to a tap of the same output (its own
// row / column / plane): a repeated (key, seed) candidate cannot change the
// running minimum, the winner or the tie mark, so there are no load
// predicates and no EMPTY selects.  The keys still use the unclamped stencil
// position, which is what the output sees.  EMPTY (-1) decodes to the far
// virtual seed (4095, 1023, 1023) whose key the host proved larger than every
// real key (natural_empty_ok), so EMPTY taps need no test either.
//
// Integer ties between distinct seeds mark the output (odd Km) and are
// re-decided by jfa2.cuh's jfa_fixup_w_kernel with the reference's fp64 rule;
// the pass leaves the cell's tied winner W (a seed at the minimum key) in the
// seed output for it (FINAL: in the free ping-pong buffer `dst`).
#pragma once
#include "jfa2.cuh"

#ifndef JFA5_MINB
#define JFA5_MINB 6  // 2 x 2 tiles: 85 registers, 24 resident warps per SM (measured best)
#endif

namespace rtsdf {

struct Jfa5Task {
    int zres, zgroups;  // z residues min(k, nz), chain groups of ZT
    int jres, jgroups;  // y residues min(k, ny), chain groups of RY
    int ires, isegs, L; // x residues min(k, onx), segments of L planes
    int tpb;            // threads per (ri, si) block, padded to a multiple of 32
    int one, zero;      // = 1, 0 (opaque to ptxas, see jfa5_eval)
};

// jfa2_eval's rule (K <= Km && v != W -> Km = min(Km - 1, K), W = v) split
// evenly over the two half-rate pipes: the compares and the predicated min on
// the ALU pipe, Km - 1 and the predicated winner move as IMADs on the FMA pipe
// (`one` / `zero` are opaque to ptxas, which would otherwise emit ALU selects:
// five ALU instructions per candidate measured ALU-pipe bound).
__device__ __forceinline__ void jfa5_eval(int K, int32_t v, int& Km, int32_t& W, int one, int zero) {
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

// EXACT: (K, v) < (Km, W) lexicographically, the seed compared unsigned
// (EMPTY = 0xffffffff is the largest): one 64-bit compare of {K : v}.
__device__ __forceinline__ void jfa5_eval_exact(int K, int32_t v, int& Km, int32_t& W, int zero) {
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

template <int RY, int ZT, bool FINAL, bool SLAB, bool EXACT>
__global__ void __launch_bounds__(128, JFA5_MINB)
    jfa_pass5_kernel(PlaneSrc src, int32_t* __restrict__ dst, float* __restrict__ dst_sdf, JfaGeom g,
                     Jfa5Task T, double beta, int64_t* __restrict__ empty_count, JfaFixList fix) {
    const int lane = threadIdx.x & 31;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t blk = tid / T.tpb;  // (ri, si): uniform over the warp (tpb % 32 == 0)
    if (blk >= (int64_t)T.ires * T.isegs) return;
    const int nthr = T.zres * T.zgroups * T.jres * T.jgroups;
    int tin = (int)(tid - blk * T.tpb);
    const bool live = tin < nthr;  // padding lanes repeat a real tile, store nothing
    if (!live) tin = nthr - 1;
    const int rz = tin % T.zres;
    tin /= T.zres;
    const int gz = tin % T.zgroups;
    tin /= T.zgroups;
    const int rj = tin % T.jres;
    const int gj = tin / T.jres;
    const int ri = (int)(blk % T.ires), si = (int)(blk / T.ires);

    const int k = g.offset;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int i_first = g.ox0 + ri + si * T.L * k;  // global plane of output a = 0
    const int i_end = g.ox0 + g.onx;
    int la = (i_end - i_first + k - 1) / k;         // outputs of this residue left in the slab
    if (la > T.L) la = T.L;
    const int clen_z = (g.nz - rz + k - 1) / k;     // chain lengths of this residue class
    const int clen_y = (g.ny - rj + k - 1) / k;
    const int n0 = gz * ZT, jn0 = gj * RY;
    const int z0 = rz + n0 * k, y0 = rj + jn0 * k;  // output (b, m) = (0, 0) of the block

    // non-EXACT: doubled weights, so every real key is even (jfa2_eval's tie mark)
    const int wsc = EXACT ? 1 : 2;
    const int wx = wsc * g.wx, wy = wsc * g.wy, wz = wsc * g.wz;
    const int gxk = 2 * wx * k, gyk = 2 * wy * k, gzk = 2 * wz * k;
    const int cy0 = -2 * wy * y0, cz0 = -2 * wz * z0;

    // tap (bt, m) sits at row y0 + (bt - 1) k, column z0 + (m - 1) k.  Its load
    // address is clamped into the grid (per lane, once per task): an
    // out-of-grid tap then reads a tap of the same outputs -- its inward
    // neighbour, a repeat that cannot change them.
    int rowc[RY + 2], colc[ZT + 2];
#pragma unroll
    for (int bt = 0; bt < RY + 2; ++bt) {
        int n = jn0 + bt - 1;
        n = n < 0 ? 0 : (n >= clen_y ? clen_y - 1 : n);
        rowc[bt] = (rj + n * k) * g.nz;
    }
#pragma unroll
    for (int m = 0; m < ZT + 2; ++m) {
        int n = n0 + m - 1;
        n = n < 0 ? 0 : (n >= clen_z ? clen_z - 1 : n);
        colc[m] = rz + n * k;
    }
    unsigned okmask = 0;  // output (b, m) inside the grid (and a live lane)
#pragma unroll
    for (int b = 0; b < RY; ++b)
#pragma unroll
        for (int m = 0; m < ZT; ++m)
            okmask |= (unsigned)(live && jn0 + b < clen_y && n0 + m < clen_z) << (b * ZT + m);
    const int kz = k * g.nz;  // < 2^20 x 2^9: 32-bit in-plane offsets
    const int64_t cell0 = (int64_t)y0 * g.nz + z0;  // in-plane cell of output (0, 0)

    int Km[3][RY][ZT];
    int32_t W[3][RY][ZT];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int b = 0; b < RY; ++b)
#pragma unroll
            for (int m = 0; m < ZT; ++m) {
                Km[s][b][m] = 0x7fffffff;
                W[s][b][m] = RTSDF_EMPTY;
            }

    int empties = 0;
    // tap planes a = -1 .. la; after plane a, output a - 1 (slot 0) is complete
    for (int a = -1; a <= la; ++a) {
        // the tap plane, clamped onto the plane of an output it feeds
        const int pi = i_first + a * k;
        const int pc = pi < 0 ? pi + k : (pi >= g.nx ? pi - k : pi);
        const int32_t* pl = SLAB ? plane_ptr(src, g, pc, plane) : src.local + (int64_t)pc * plane;
        asm("mov.b64 %0, %0;" : "+l"(pl));  // opaque: one IMAD.WIDE per tap address
        int32_t v[RY + 2][ZT + 2];
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt)
#pragma unroll
            for (int m = 0; m < ZT + 2; ++m) v[bt][m] = __ldg(pl + (unsigned)(rowc[bt] + colc[m]));
        const int cx = -2 * wx * pi;
#pragma unroll
        for (int bt = 0; bt < RY + 2; ++bt) {
#pragma unroll
            for (int m = 0; m < ZT + 2; ++m) {
                const int32_t s = v[bt][m];
                const int sx = unpack_i(s), sy = unpack_j(s), sz = unpack_k(s);
                // key of the seed at output (b, m') of the output plane a - 1 + sl:
                //   K = B0 - (sl - 1) Gx - b Gy - m' Gz  (B0: plane a, row y0, column z0)
                const int B0 = sx * (wx * sx + cx) + sy * (wy * sy + cy0) + sz * (wz * sz + cz0);
                const int Gx = gxk * sx, Gy = gyk * sy, Gz = gzk * sz;
                const int Ys[3] = {0, Gy, Gy + Gy}, Zs[3] = {0, Gz, Gz + Gz};
#pragma unroll
                for (int sl = 0; sl < 3; ++sl) {
                    const int Bs = sl == 0 ? B0 + Gx : (sl == 1 ? B0 : B0 - Gx);
#pragma unroll
                    for (int b = bt - 2; b <= bt; ++b) {
                        if (b < 0 || b >= RY) continue;  // compile-time
#pragma unroll
                        for (int mo = m - 2; mo <= m; ++mo) {
                            if (mo < 0 || mo >= ZT) continue;  // compile-time
                            const int K = Bs - Ys[b] - Zs[mo];  // one IADD3
                            int& km = Km[sl][b][mo];
                            int32_t& w = W[sl][b][mo];
                            if (sl == 2 && bt == b && m == mo) {
                                // first candidate of a fresh output plane
                                km = K;
                                w = s;
                            } else if (EXACT) {
                                jfa5_eval_exact(K, s, km, w, T.zero);
                            } else {
                                jfa5_eval(K, s, km, w, T.one, T.zero);
                            }
                        }
                    }
                }
            }
        }
        // output a - 1 (slot 0) is complete
        const int oa = a - 1;
        if (oa >= 0) {
            const int oi = i_first + oa * k;
            const int64_t ocell0 = (int64_t)(oi - g.ox0) * plane + cell0;
            int32_t* dplane = dst + ocell0;
            float* splane = dst_sdf + ocell0;
            asm("mov.b64 %0, %0;" : "+l"(dplane));
            asm("mov.b64 %0, %0;" : "+l"(splane));
            unsigned tie = 0;
#pragma unroll
            for (int b = 0; b < RY; ++b)
#pragma unroll
                for (int m = 0; m < ZT; ++m) {
                    const bool ok = (okmask >> (b * ZT + m)) & 1u;
                    const int32_t w = W[0][b][m];
                    const unsigned off = (unsigned)(b * kz + m * k);
                    if (FINAL) {
                        if (ok) {
                            empties += w == RTSDF_EMPTY;
                            const int oj = y0 + b * k, oz = z0 + m * k;
                            const double d2 = center_d2(oi - unpack_i(w), oj - unpack_j(w), oz - unpack_k(w),
                                                        g.hx, g.hy, g.hz);
                            splane[off] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
                        }
                    } else if (ok) {
                        dplane[off] = w;
                    }
                    if (!EXACT) tie |= (unsigned)(w != RTSDF_EMPTY && (Km[0][b][m] & 1)) << (b * ZT + m);
                }
            tie &= okmask;
            if (FINAL && !EXACT && tie) {
                // the fix-up's witness of K* (a tied winner), in the free ping-pong buffer
#pragma unroll
                for (int b = 0; b < RY; ++b)
#pragma unroll
                    for (int m = 0; m < ZT; ++m)
                        if ((tie >> (b * ZT + m)) & 1u) dplane[(unsigned)(b * kz + m * k)] = W[0][b][m];
            }
            // integer ties between distinct seeds: one warp-aggregated append
            if (!EXACT && __any_sync(0xffffffffu, tie != 0)) {
                const int cnt = __popc(tie);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                int64_t base = 0;
                if (lane == 31)
                    base = (int64_t)atomicAdd((unsigned long long*)fix.count, (unsigned long long)incl);
                base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
                while (tie) {
                    const int bit = __ffs(tie) - 1;
                    tie &= tie - 1;
                    const int b = bit / ZT, m = bit - b * ZT;
                    if (base < fix.cap) fix.cells[base] = (int32_t)(ocell0 + b * kz + m * k);
                    ++base;
                }
            }
        }
#pragma unroll
        for (int b = 0; b < RY; ++b)
#pragma unroll
            for (int m = 0; m < ZT; ++m) {
                Km[0][b][m] = Km[1][b][m];
                W[0][b][m] = W[1][b][m];
                Km[1][b][m] = Km[2][b][m];
                W[1][b][m] = W[2][b][m];
            }
    }
    if (FINAL && empty_count) {
        for (int o = 16; o; o >>= 1) empties += __shfl_xor_sync(0xffffffffu, empties, o);
        if (lane == 0 && empties) atomicAdd((unsigned long long*)empty_count, (unsigned long long)empties);
    }
}

}  // namespace rtsdf
