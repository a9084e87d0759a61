// jfa.cu -- K2 (JFA pass), jfa_init, K3 (seeds -> SDF) and seed format helpers.
//
// Restates jfa.py:47-181.  Seeds are packed int32 (i<<20 | j<<10 | k) so the
// lexicographic tie rule (jfa.py:116-124) is a plain integer compare and the
// decode is shifts/masks instead of the reference's two integer divisions.
//
// Exactness: the reference orders candidates by fp64 d2
// evaluated as ((dx*hx)^2 + (dy*hy)^2) + (dz*hz)^2 and falls back to the
// lexicographic rule only among fp64-EQUAL values.  When the host proves
// hx^2 : hy^2 : hz^2 = wx : wy : wz exactly (rational arithmetic on the fp64
// cell sizes), the true d2 is s*q with q = wx dx^2 + wy dy^2 + wz dz^2 an
// integer, and fp64's <= 5 ulp relative error cannot reorder distinct q (the
// relative gap is >= 1/q_max ~ 1e-7).  So the INT path orders by q and only
// evaluates the reference's fp64 expression when q ties -- bit-exact, with
// integer work on the common path.  (0,0,0) weights select the FP64 path.
#include <cmath>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace rtsdf {

enum { JFA_INT = 0, JFA_FP64 = 1 };

struct JfaGeom {
    int nx, ny, nz;     // global grid
    int x0, nxl;        // owned planes [x0, x0 + nxl)
    int lo_first, n_lo; // halo planes below
    int hi_first, n_hi; // halo planes above
    int offset;
    double hx, hy, hz;
    int wx, wy, wz;
    bool exact;  // fp64 d2 exact for these spacings (fp64_exact): ties resolve in the pass
    int ox0, onx;  // output planes [ox0, ox0 + onx) (a sub-range of the owned planes;
                   // dst points at plane ox0): interior / boundary launches of a slab
    SeedFmt fmt;   // packed seed layout (seed_fmt_for; the fast kernels assume the fixed one)
};

// True when every fp64 operation of center_d2 (jfa.py:72-76) is exact for all
// offsets |d| < n on each axis: h = m 2^e (m odd) with d*h and (d*h)^2
// representable, and every partial sum of the three terms a multiple of the
// smallest term granularity below 2^53.  Dyadic spacings such as 4/512 or
// 2/1024 qualify (C1, C2, C4, C5); 3.2/400 (C3) does not.
static bool fp64_exact(double hx, double hy, double hz, int nx, int ny, int nz) {
    const double hs[3] = {hx, hy, hz};
    const int ns[3] = {nx, ny, nz};
    int64_t mant[3];
    int ex[3], mb[3];
    int gmin = 1 << 30;
    for (int a = 0; a < 3; ++a) {
        if (!(hs[a] > 0.0) || !std::isfinite(hs[a])) return false;
        int e2;
        const double f = std::frexp(hs[a], &e2);  // h = f 2^e2, f in [0.5, 1)
        int64_t m = (int64_t)std::ldexp(f, 53);
        int e = e2 - 53;
        while ((m & 1) == 0) {
            m >>= 1;
            ++e;
        }
        mant[a] = m;
        ex[a] = e;
        mb[a] = 64 - __builtin_clzll((unsigned long long)m);
        const int db = ns[a] > 1 ? 64 - __builtin_clzll((unsigned long long)(ns[a] - 1)) : 0;
        if (2 * (mb[a] + db) > 53) return false;  // d h and (d h)^2 exact
        if (ns[a] > 1 && 2 * e < gmin) gmin = 2 * e;
    }
    if (gmin == 1 << 30) return true;  // a single cell
    unsigned __int128 sum = 0;
    for (int a = 0; a < 3; ++a) {
        if (ns[a] <= 1) continue;
        const int sh = 2 * ex[a] - gmin;
        if (sh > 60) return false;
        const unsigned __int128 d = (unsigned __int128)(ns[a] - 1);
        sum += d * d * (unsigned __int128)mant[a] * (unsigned __int128)mant[a] << sh;
    }
    return sum < ((unsigned __int128)1 << 53);
}

struct PlaneSrc {
    const int32_t* local;
    const int32_t* halo_lo;
    const int32_t* halo_hi;
};

__device__ __forceinline__ const int32_t* plane_ptr(const PlaneSrc& s, const JfaGeom& g, int q,
                                                    int64_t plane) {
    if (q >= g.x0 && q < g.x0 + g.nxl) return s.local + (int64_t)(q - g.x0) * plane;
    if (q >= g.lo_first && q < g.lo_first + g.n_lo) return s.halo_lo + (int64_t)(q - g.lo_first) * plane;
    if (q >= g.hi_first && q < g.hi_first + g.n_hi) return s.halo_hi + (int64_t)(q - g.hi_first) * plane;
    return nullptr;
}

template <int MODE>
struct Best {
    int32_t p;
    int q;      // INT: weighted integer d2; unused for FP64
    double d2;  // FP64: reference d2; INT: lazily evaluated on ties
};

// Consider candidate seed c for the cell (i, j, k); jfa.py:108-124.
template <int MODE>
__device__ __forceinline__ void consider(Best<MODE>& b, int32_t c, int i, int j, int k,
                                         const JfaGeom& g) {
    if (c == RTSDF_EMPTY || c == b.p) return;
    int dx = i - fmt_i(c, g.fmt), dy = j - fmt_j(c, g.fmt), dz = k - fmt_k(c, g.fmt);
    if (MODE == JFA_INT) {
        int q = g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
        if (q < b.q) {
            b.p = c;
            b.q = q;
        } else if (q == b.q && b.p != RTSDF_EMPTY) {
            // integer tie: decide on the reference's fp64 values
            double dc = center_d2(dx, dy, dz, g.hx, g.hy, g.hz);
            double db = center_d2(i - fmt_i(b.p, g.fmt), j - fmt_j(b.p, g.fmt), k - fmt_k(b.p, g.fmt), g.hx,
                                  g.hy, g.hz);
            if (dc < db || (dc == db && c < b.p)) {
                b.p = c;
                b.q = q;
            }
        }
    } else {
        double d2 = center_d2(dx, dy, dz, g.hx, g.hy, g.hz);
        if (d2 < b.d2 || (d2 == b.d2 && b.p != RTSDF_EMPTY && c < b.p)) {
            b.p = c;
            b.d2 = d2;
        }
    }
}

// One thread per cell; block = 32 (z) x 8 (y), grid.z walks the owned planes.
template <int MODE, bool SLAB>
__global__ void __launch_bounds__(256) jfa_step_kernel(PlaneSrc src, int32_t* __restrict__ dst,
                                                       JfaGeom g) {
    const int k = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * 8 + threadIdx.y;
    const int il = blockIdx.z;  // output plane (relative to g.ox0)
    if (k >= g.nz || j >= g.ny) return;
    const int i = g.ox0 + il;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const int off = g.offset;
    Best<MODE> b;
    b.p = __ldg(src.local + (int64_t)(i - g.x0) * plane + (int64_t)j * g.nz + k);
    if (b.p != RTSDF_EMPTY) {
        int dx = i - fmt_i(b.p, g.fmt), dy = j - fmt_j(b.p, g.fmt), dz = k - fmt_k(b.p, g.fmt);
        if (MODE == JFA_INT) b.q = g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
        else b.d2 = center_d2(dx, dy, dz, g.hx, g.hy, g.hz);
    } else {
        b.q = 0x7fffffff;
        b.d2 = 1e300;
    }
#pragma unroll
    for (int di = -1; di <= 1; ++di) {
        const int qi = i + di * off;
        if (qi < 0 || qi >= g.nx) continue;
        const int32_t* pl = SLAB ? plane_ptr(src, g, qi, plane)
                                 : src.local + (int64_t)qi * plane;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
            const int qj = j + dj * off;
            if (qj < 0 || qj >= g.ny) continue;
            const int32_t* row = pl + (int64_t)qj * g.nz;
#pragma unroll
            for (int dk = -1; dk <= 1; ++dk) {
                if (di == 0 && dj == 0 && dk == 0) continue;
                const int qk = k + dk * off;
                if (qk < 0 || qk >= g.nz) continue;
                consider<MODE>(b, __ldg(row + qk), i, j, k, g);
            }
        }
    }
    dst[(int64_t)il * plane + (int64_t)j * g.nz + k] = b.p;
}

// ---- sparse early passes -----------------------------------------------------
// The first passes (k >= 128 at C3) read grids that are > 99 % EMPTY (0.55 % of
// cells hold a seed).  A byte per 32-cell z-segment records whether the
// segment holds any seed; a warp owns one output segment, its lanes 0..26
// test the 27 tap segments (k is a multiple of 32, so a tap segment is a whole
// segment) and a warp whose taps are all empty writes EMPTY without loading a
// single tap.  Other warps run the per-cell rule of jfa_step_kernel.  The
// output bitmap for the next pass comes out of the same warp vote.

__global__ void __launch_bounds__(256) jfa_seg_bitmap_kernel(const int32_t* __restrict__ src,
                                                             uint8_t* __restrict__ bm, int ny,
                                                             int nz, FastDiv dzb, uint32_t n_seg,
                                                             unsigned long long* __restrict__ n_on) {
    unsigned on_count = 0;
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    // 4 segments per warp per step: independent loads in flight
    for (uint32_t s0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 4; s0 < n_seg; s0 += nwarps * 4) {
        bool on[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t seg = s0 + u;
            const uint32_t row = fdiv(seg, dzb);  // segments < 2^25
            const int z = (int)(seg - row * dzb.d) * 32 + lane;
            on[u] = seg < n_seg && z < nz && __ldg(src + (int64_t)row * nz + z) != RTSDF_EMPTY;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned m = __ballot_sync(0xffffffffu, on[u]);
            if (lane == 0 && s0 + u < n_seg) bm[s0 + u] = m != 0;
            on_count += m != 0;
        }
    }
    if (lane == 0 && on_count) atomicAdd(n_on, (unsigned long long)on_count);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(n_on, 1ull);  // "measured" (+1)
}

// Two-phase sparse pass.  Phase 1, one THREAD per output segment: the 27 tap
// segment bits (k a multiple of 32: whole segments) are OR-ed; a segment no
// seed can reach is filled with EMPTY right away (vector stores, no tap loads)
// and its output bit cleared, the others are appended to an active list.
// Phase 2, one warp per active segment: the per-cell rule (jfa_step_kernel's).
// The thread-per-segment test costs ~100 thread instructions per segment
// where the warp-per-segment form spent ~90 warp instructions.
__global__ void __launch_bounds__(256) jfa_sparse_fill_kernel(int32_t* __restrict__ dst, JfaGeom g,
                                                              const uint8_t* __restrict__ bm_in,
                                                              uint8_t* __restrict__ bm_out,
                                                              FastDiv dzb, FastDiv dny,
                                                              int32_t* __restrict__ active,
                                                              unsigned long long* __restrict__ n_active,
                                                              unsigned long long* __restrict__ n_on) {
    const int nzb = (int)dzb.d;
    const uint32_t n_seg = (uint32_t)g.nx * g.ny * nzb;
    const int off = g.offset, kz = off >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t seg0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); seg0 < n_seg; seg0 += stride) {
        const uint32_t seg = seg0 + lane;
        bool any = false;
        if (seg < n_seg) {
            const uint32_t row = fdiv(seg, dzb);
            const int zb = (int)(seg - row * dzb.d);
            const int i = (int)fdiv(row, dny), j = (int)(row - (uint32_t)i * dny.d);
#pragma unroll
            for (int di = -1; di <= 1; ++di) {
                const int qi = i + di * off;
#pragma unroll
                for (int dj = -1; dj <= 1; ++dj) {
                    const int qj = j + dj * off;
                    if (qi < 0 || qi >= g.nx || qj < 0 || qj >= g.ny) continue;
                    const uint8_t* r = bm_in + ((int64_t)qi * g.ny + qj) * nzb;
#pragma unroll
                    for (int dk = -1; dk <= 1; ++dk) {
                        const int qz = zb + dk * kz;
                        if (qz >= 0 && qz < nzb) any |= __ldg(r + qz) != 0;
                    }
                }
            }
            if (!any) {
                const int z0 = zb * 32, len = min(32, g.nz - z0);
                int32_t* d = dst + (int64_t)row * g.nz + z0;
                if ((((uintptr_t)d) & 15) == 0 && (len & 3) == 0) {
                    const int4 e = make_int4(RTSDF_EMPTY, RTSDF_EMPTY, RTSDF_EMPTY, RTSDF_EMPTY);
                    for (int q = 0; q < len; q += 4) *(int4*)(d + q) = e;
                } else {
                    for (int q = 0; q < len; ++q) d[q] = RTSDF_EMPTY;
                }
                if (bm_out) bm_out[seg] = 0;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, any);
        if (m) {
            unsigned long long base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(n_active, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
            if (any) active[base + __popc(m & ((1u << lane) - 1))] = (int32_t)seg;
        }
    }
    if (n_on && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(n_on, 1ull);  // "measured" (+1)
}

template <int MODE>
__global__ void __launch_bounds__(256) jfa_sparse_active_kernel(const int32_t* __restrict__ src,
                                                                int32_t* __restrict__ dst, JfaGeom g,
                                                                uint8_t* __restrict__ bm_out,
                                                                FastDiv dzb, FastDiv dny,
                                                                const int32_t* __restrict__ active,
                                                                const unsigned long long* __restrict__ n_active,
                                                                unsigned long long* __restrict__ n_on) {
    unsigned on_count = 0;
    const int lane = threadIdx.x & 31;
    const int off = g.offset;
    const int64_t plane = (int64_t)g.ny * g.nz;
    const unsigned long long na = *n_active;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < na; a += nwarps) {
        const uint32_t seg = (uint32_t)active[a];
        const uint32_t row = fdiv(seg, dzb);
        const int zb = (int)(seg - row * dzb.d);
        const int i = (int)fdiv(row, dny), j = (int)(row - (uint32_t)i * dny.d);
        const int k = zb * 32 + lane;
        const int64_t cell = (int64_t)i * plane + (int64_t)j * g.nz + k;
        int32_t out = RTSDF_EMPTY;
        if (k < g.nz) {
            Best<MODE> b;
            b.p = __ldg(src + cell);
            if (b.p != RTSDF_EMPTY) {
                int dx = i - fmt_i(b.p, g.fmt), dy = j - fmt_j(b.p, g.fmt), dz = k - fmt_k(b.p, g.fmt);
                if (MODE == JFA_INT) b.q = g.wx * dx * dx + g.wy * dy * dy + g.wz * dz * dz;
                else b.d2 = center_d2(dx, dy, dz, g.hx, g.hy, g.hz);
            } else {
                b.q = 0x7fffffff;
                b.d2 = 1e300;
            }
#pragma unroll
            for (int di = -1; di <= 1; ++di) {
                const int qi = i + di * off;
                if (qi < 0 || qi >= g.nx) continue;
#pragma unroll
                for (int dj = -1; dj <= 1; ++dj) {
                    const int qj = j + dj * off;
                    if (qj < 0 || qj >= g.ny) continue;
                    const int32_t* rw = src + (int64_t)qi * plane + (int64_t)qj * g.nz;
#pragma unroll
                    for (int dk = -1; dk <= 1; ++dk) {
                        if (di == 0 && dj == 0 && dk == 0) continue;
                        const int qk = k + dk * off;
                        if (qk < 0 || qk >= g.nz) continue;
                        consider<MODE>(b, __ldg(rw + qk), i, j, k, g);
                    }
                }
            }
            out = b.p;
            dst[cell] = out;
        }
        const unsigned m = __ballot_sync(0xffffffffu, out != RTSDF_EMPTY);
        if (bm_out && lane == 0) bm_out[seg] = m != 0;
        on_count += m != 0;
    }
    if (n_on && lane == 0 && on_count) atomicAdd(n_on, (unsigned long long)on_count);
}

__global__ void jfa_init_kernel(const uint8_t* __restrict__ occ, int ny, int nz, int64_t n,
                                int32_t* __restrict__ seed, int64_t* __restrict__ count, SeedFmt f) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool on = false;
    if (c < n) {
        on = occ[c] != 0;
        int64_t nyz = (int64_t)ny * nz;
        int i = (int)(c / nyz), j = (int)((c / nz) % ny), k = (int)(c % nz);
        seed[c] = on ? fmt_pack(i, j, k, f) : RTSDF_EMPTY;
    }
    if (count) {
        unsigned m = __ballot_sync(0xffffffffu, on);
        if ((threadIdx.x & 31) == 0 && m) atomicAdd((unsigned long long*)count, (unsigned long long)__popc(m));
    }
}

// jfa.py:148-160: f32(sqrt(d2_fp64) - beta)
__global__ void seeds_to_sdf_kernel(const int32_t* __restrict__ seed, float* __restrict__ out,
                                    int x0, int ny, int nz, double hx, double hy, double hz,
                                    double beta, int64_t* __restrict__ empty_count, SeedFmt f) {
    const int k = blockIdx.x * 32 + threadIdx.x;
    const int j = blockIdx.y * 8 + threadIdx.y;
    const int i = x0 + blockIdx.z;  // global plane (buffers are global-indexed)
    bool empty = false;
    if (k < nz && j < ny) {
        int64_t c = ((int64_t)i * ny + j) * nz + k;
        int32_t s = __ldg(seed + c);
        empty = s == RTSDF_EMPTY;
        double d2 = center_d2(i - fmt_i(s, f), j - fmt_j(s, f), k - fmt_k(s, f), hx, hy, hz);
        out[c] = (float)__dsub_rn(__dsqrt_rn(d2), beta);
    }
    if (empty_count) {
        unsigned m = __ballot_sync(0xffffffffu, empty);
        if (((threadIdx.y * 32 + threadIdx.x) & 31) == 0 && m)
            atomicAdd((unsigned long long*)empty_count, (unsigned long long)__popc(m));
    }
}

__global__ void packed_to_linear_kernel(const int32_t* __restrict__ p, int32_t* __restrict__ l,
                                        int ny, int nz, int64_t n, SeedFmt f) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    int32_t s = p[c];
    l[c] = s == RTSDF_EMPTY ? RTSDF_EMPTY
                            : (int32_t)(((int64_t)fmt_i(s, f) * ny + fmt_j(s, f)) * nz + fmt_k(s, f));
}

__global__ void linear_to_packed_kernel(const int32_t* __restrict__ l, int32_t* __restrict__ p,
                                        int ny, int nz, int64_t n, SeedFmt f) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    int32_t s = l[c];
    if (s == RTSDF_EMPTY) {
        p[c] = RTSDF_EMPTY;
        return;
    }
    int64_t nyz = (int64_t)ny * nz;
    p[c] = fmt_pack((int)(s / nyz), (int)((s / nz) % ny), (int)(s % nz), f);
}

}  // namespace rtsdf

#include "jfa2.cuh"
#include "jfa4.cuh"
#include "jfa5.cuh"

namespace rtsdf {

static bool dims_ok(int nx, int ny, int nz) {
    SeedFmt f;
    if (!seed_fmt_for(nx, ny, nz, &f) || (int64_t)nx * ny * nz >= ((int64_t)1 << 31)) {
        set_error("dims (%d, %d, %d): packed int32 seeds need bits(nx-1) + bits(ny-1) + bits(nz-1) <= 31",
                  nx, ny, nz);
        return false;
    }
    return true;
}
static SeedFmt fmt_of(int nx, int ny, int nz) {
    SeedFmt f = seed_fmt_packed();
    seed_fmt_for(nx, ny, nz, &f);
    return f;
}

// jfa2.cuh NAT: min over the grid of the virtual EMPTY seed's weighted d2
// (taken at the far corner) > the largest real weighted d2 in the grid.
static bool natural_empty_ok(const JfaGeom& g) {
    auto sq = [](double v) { return v * v; };
    const double e = g.wx * sq(4096.0 - g.nx) + g.wy * sq(1024.0 - g.ny) + g.wz * sq(1024.0 - g.nz);
    const double r = g.wx * sq(g.nx - 1.0) + g.wy * sq(g.ny - 1.0) + g.wz * sq(g.nz - 1.0);
    return e > r;
}

// K2 v2 launch (INT mode): task decomposition of jfa2.cuh, then the exact
// re-decision of the (rare) integer-tie cells the pass flagged.
static JfaFixList fix_list(void* ws, int64_t n_cells) {
    JfaFixList f;
    f.count = (int64_t*)ws;
    f.cells = (int32_t*)((char*)ws + 256);
    f.cap = n_cells;
    return f;
}

template <bool FINAL, bool SLAB>
static void launch_pass2(PlaneSrc s, int32_t* dst, float* dst_sdf, const JfaGeom& g, double beta,
                         int64_t* empty_count, void* ws, cudaStream_t st) {
    const int k = g.offset;
    const int chain_y = (g.ny + k - 1) / k;  // longest j chain
    const int ry = chain_y >= 4 ? 4 : (chain_y >= 2 ? 2 : 1);
    // Segment length L: each unit re-loads 2 halo planes per L outputs, so
    // longer is cheaper (measured at C3: L = 24 is ~8 % faster than 8) as long
    // as the grid still fills the GPU for two waves (~16 resident warps / SM).
    const bool nat = natural_empty_ok(g);
    Jfa2Task T;
    T.one = 1;
    T.zero = 0;
#ifndef JFA2_SKIP_K
#define JFA2_SKIP_K 16
#endif
    T.skip = k >= JFA2_SKIP_K;
    T.nzb = (g.nz + 31) / 32;
    T.jres = k < g.ny ? k : g.ny;
    T.jgroups = (chain_y + ry - 1) / ry;
    T.ires = k < g.onx ? k : g.onx;
    const int chain_x = (g.onx + k - 1) / k;
    T.L = 24;
    const int64_t want = (int64_t)num_sms() * 16 * 2;
    while (T.L > 4 &&
           (int64_t)T.nzb * T.jres * T.jgroups * T.ires * ((chain_x + T.L - 1) / T.L) < want)
        T.L /= 2;
    T.isegs = (chain_x + T.L - 1) / T.L;
    JfaFixList fix = fix_list(ws, (int64_t)g.onx * g.ny * g.nz);
    cudaMemsetAsync(fix.count, 0, sizeof(int64_t), st);
    int64_t warps = (int64_t)T.nzb * T.jres * T.jgroups * T.ires * T.isegs;
    unsigned blocks = (unsigned)((warps + 3) / 4);
    if (g.exact) {  // ties resolve inside the pass: no flags, no fix-up
        if (ry == 4)
            nat ? jfa_pass2_kernel<4, FINAL, SLAB, true, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix)
                : jfa_pass2_kernel<4, FINAL, SLAB, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
        else if (ry == 2)
            jfa_pass2_kernel<2, FINAL, SLAB, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
        else
            jfa_pass2_kernel<1, FINAL, SLAB, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
        count_launch(1);
        return;
    }
    if (ry == 4)
        nat ? jfa_pass2_kernel<4, FINAL, SLAB, false, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix)
            : jfa_pass2_kernel<4, FINAL, SLAB, false><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
    else if (ry == 2)
        jfa_pass2_kernel<2, FINAL, SLAB, false><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
    else
        jfa_pass2_kernel<1, FINAL, SLAB, false><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
    // a flagged cell's seed output holds a tied winner (a seed at its minimum
    // key): the one-loop fix-up; the FINAL pass writes no seeds -> the full one
    if (FINAL)
        jfa_fixup_kernel<FINAL, SLAB><<<(unsigned)(num_sms() * 16), 128, 0, st>>>(
            s, dst, dst_sdf, g, beta, fix, make_fastdiv((uint32_t)g.nz), make_fastdiv((uint32_t)g.ny));
    else
        jfa_fixup_w_kernel<FINAL, SLAB><<<(unsigned)(num_sms() * 16), 128, 0, st>>>(
            s, dst, dst_sdf, g, beta, fix, make_fastdiv((uint32_t)g.nz), make_fastdiv((uint32_t)g.ny));
    count_launch(2);
}

// K2 v4 launch (INT mode): residue-chain tiles, integer ties resolved in the kernel.
template <bool FINAL, bool SLAB>
static void launch_pass4(PlaneSrc s, int32_t* dst, float* dst_sdf, const JfaGeom& g, double beta,
                         int64_t* empty_count, void* ws, cudaStream_t st) {
    const int k = g.offset;
    const int chain_y = (g.ny + k - 1) / k;
    const int ry = chain_y >= 4 ? 4 : (chain_y >= 2 ? 2 : 1);
    const bool nat = natural_empty_ok(g);
    Jfa4Task T;
    T.one = 1;
    T.zero = 0;
    T.skip = k >= 16;
    T.nz_pos = g.nz;
    T.single = g.nz <= 32;
    T.zw = T.single ? 1 : (g.nz + 29) / 30;
    T.lc = (g.nz + k - 1) / k;
    T.nlong = g.nz - k * (T.lc - 1);  // residues with lc positions (k >= nz: every z, lc = 1)
    if (T.nlong > k) T.nlong = k;
    T.jres = k < g.ny ? k : g.ny;
    T.jgroups = (chain_y + ry - 1) / ry;
    T.ires = k < g.onx ? k : g.onx;
    const int chain_x = (g.onx + k - 1) / k;
    // segment length L: 2 halo planes per L outputs; halve while the grid
    // would not fill the GPU for two waves (~16 resident warps / SM)
    T.L = 24;
    const int64_t want = (int64_t)num_sms() * 16 * 2;
    while (T.L > 4 && (int64_t)T.zw * T.jres * T.jgroups * T.ires * ((chain_x + T.L - 1) / T.L) < want)
        T.L /= 2;
    T.isegs = (chain_x + T.L - 1) / T.L;
    const int64_t warps = (int64_t)T.zw * T.jres * T.jgroups * T.ires * T.isegs;
    const unsigned blocks = (unsigned)((warps + 3) / 4);
    JfaFixList fix = fix_list(ws, (int64_t)g.onx * g.ny * g.nz);
    if (!g.exact) cudaMemsetAsync(fix.count, 0, sizeof(int64_t), st);
#define RTSDF_P4(RYV, EX, NA) \
    jfa_pass4_kernel<RYV, FINAL, SLAB, EX, NA><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix)
    if (g.exact) {
        if (ry == 4) { if (nat) RTSDF_P4(4, true, true); else RTSDF_P4(4, true, false); }
        else if (ry == 2) { if (nat) RTSDF_P4(2, true, true); else RTSDF_P4(2, true, false); }
        else { if (nat) RTSDF_P4(1, true, true); else RTSDF_P4(1, true, false); }
    } else {
        if (ry == 4) { if (nat) RTSDF_P4(4, false, true); else RTSDF_P4(4, false, false); }
        else if (ry == 2) { if (nat) RTSDF_P4(2, false, true); else RTSDF_P4(2, false, false); }
        else { if (nat) RTSDF_P4(1, false, true); else RTSDF_P4(1, false, false); }
        // the (rare) overflow of the kernel's per-warp tie queues; a no-op when empty
        jfa_fixup_kernel<FINAL, SLAB><<<(unsigned)num_sms(), 128, 0, st>>>(
            s, dst, dst_sdf, g, beta, fix, make_fastdiv((uint32_t)g.nz), make_fastdiv((uint32_t)g.ny));
        count_launch(1);
    }
#undef RTSDF_P4
    count_launch(1);
}

// K2 v5 launch (INT mode, NAT grids): 3-D register tiles (jfa5.cuh), then
// the exact re-decision of the integer-tie cells (non-EXACT only).
#ifndef JFA5_RY
#define JFA5_RY 2
#endif
#ifndef JFA5_ZT
#define JFA5_ZT 2
#endif
template <bool FINAL, bool SLAB>
static void launch_pass5(PlaneSrc s, int32_t* dst, float* dst_sdf, const JfaGeom& g, double beta,
                         int64_t* empty_count, void* ws, cudaStream_t st) {
    const int k = g.offset;
    Jfa5Task T;
    T.zres = k < g.nz ? k : g.nz;
    T.zgroups = ((g.nz + k - 1) / k + JFA5_ZT - 1) / JFA5_ZT;
    T.jres = k < g.ny ? k : g.ny;
    T.jgroups = ((g.ny + k - 1) / k + JFA5_RY - 1) / JFA5_RY;
    T.ires = k < g.onx ? k : g.onx;
    const int64_t nthr = (int64_t)T.zres * T.zgroups * T.jres * T.jgroups;
    T.tpb = (int)((nthr + 31) / 32 * 32);
    T.one = 1;
    T.zero = 0;
    const int chain_x = (g.onx + k - 1) / k;
    // segment length L: 2 halo planes per L outputs; halve while the grid
    // would not fill the GPU for two waves
    // balanced segments of <= 32 planes (each costs L + 2 plane steps), more
    // of them while the grid would not fill the GPU for two waves
    const int64_t want = (int64_t)num_sms() * 128 * JFA5_MINB * 2;
    T.isegs = (chain_x + 31) / 32;
    while ((chain_x + T.isegs - 1) / T.isegs > 4 && (int64_t)T.tpb * T.ires * T.isegs < want) ++T.isegs;
    T.L = (chain_x + T.isegs - 1) / T.isegs;
    T.isegs = (chain_x + T.L - 1) / T.L;
    const int64_t threads = (int64_t)T.tpb * T.ires * T.isegs;
    const unsigned blocks = (unsigned)((threads + 127) / 128);
    JfaFixList fix = fix_list(ws, (int64_t)g.onx * g.ny * g.nz);
    if (g.exact) {
        jfa_pass5_kernel<JFA5_RY, JFA5_ZT, FINAL, SLAB, true><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
        count_launch(1);
        return;
    }
    cudaMemsetAsync(fix.count, 0, sizeof(int64_t), st);
    jfa_pass5_kernel<JFA5_RY, JFA5_ZT, FINAL, SLAB, false><<<blocks, 128, 0, st>>>(s, dst, dst_sdf, g, T, beta, empty_count, fix);
    jfa_fixup_w_kernel<FINAL, SLAB><<<(unsigned)(num_sms() * 16), 128, 0, st>>>(
        s, dst, dst_sdf, g, beta, fix, make_fastdiv((uint32_t)g.nz), make_fastdiv((uint32_t)g.ny));
    count_launch(2);
}

#ifndef JFA5_MAXK
#define JFA5_MAXK 16  // k = 32 / 64 inputs still hold EMPTY regions: v2's all-EMPTY tap votes win there (measured)
#endif
#ifndef JFA5_MAXK_EXACT
#define JFA5_MAXK_EXACT 32  // dyadic grids (no tie fix-up): v5 measured ahead of v4 up to k = 32
#endif
static bool use_v5(const JfaGeom& g) {
    return g.offset <= (g.exact ? JFA5_MAXK_EXACT : JFA5_MAXK) && natural_empty_ok(g);
}

// Pass kernel by offset and grid, measured on B200 (tools/jfa_time.py):
//   v5 (jfa5.cuh, 2 x 2 register tiles): k <= 16 (non-EXACT; C3 0.34 ms per
//      dense pass vs v2's 0.46) and k <= 32 on EXACT (dyadic) grids (C4 late
//      passes 1.01 vs v4's 1.21 ms, C5 7.8 vs 9.2 ms);
//   v2 (jfa2.cuh): non-EXACT k >= 32, whose inputs still hold EMPTY regions
//      (its all-EMPTY tap votes: C3 k = 32 0.375 vs v5's 0.403 ms);
//   v4 (jfa4.cuh): EXACT k >= 64 (C4 k = 64 1.04 vs v5's 1.19 ms).
static bool use_v4(const JfaGeom& g) { return g.exact; }

static int launch_step(PlaneSrc s, int32_t* dst, const JfaGeom& g, bool slab, void* ws,
                       cudaStream_t st) {
    dim3 block(32, 8, 1);
    dim3 grid((g.nz + 31) / 32, (g.ny + 7) / 8, g.onx);
    bool int_mode = g.wx > 0 && g.wy > 0 && g.wz > 0;
    int mdim = g.nx > g.ny ? g.nx : g.ny;
    if (g.nz > mdim) mdim = g.nz;
    // grids beyond the fixed packed layout: the per-cell kernel (runtime fields)
    const bool generic = !seed_fmt_legacy(g.nx, g.ny, g.nz);
    if (int_mode && (generic || 2 * g.offset >= mdim)) {
        // first pass: every lattice chain has <= 2 cells, v2's register tiles
        // cannot amortise their setup -- the per-cell kernel is faster
        if (slab) jfa_step_kernel<JFA_INT, true><<<grid, block, 0, st>>>(s, dst, g);
        else jfa_step_kernel<JFA_INT, false><<<grid, block, 0, st>>>(s, dst, g);
        count_launch();
    } else if (int_mode && use_v5(g)) {
        if (slab) launch_pass5<false, true>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
        else launch_pass5<false, false>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
    } else if (int_mode && use_v4(g)) {
        if (slab) launch_pass4<false, true>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
        else launch_pass4<false, false>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
    } else if (int_mode) {
        if (slab) launch_pass2<false, true>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
        else launch_pass2<false, false>(s, dst, nullptr, g, 0.0, nullptr, ws, st);
    } else {
        if (slab) jfa_step_kernel<JFA_FP64, true><<<grid, block, 0, st>>>(s, dst, g);
        else jfa_step_kernel<JFA_FP64, false><<<grid, block, 0, st>>>(s, dst, g);
        count_launch();
    }
    return check_launch("jfa_step");
}

static bool weights_ok(int nx, int ny, int nz, int wx, int wy, int wz) {
    if (wx == 0 && wy == 0 && wz == 0) return true;
    if (wx <= 0 || wy <= 0 || wz <= 0) return false;
    if (wx > 16 || wy > 16 || wz > 16) return false;  // EMPTY-key bound in jfa2.cuh
    // keys relative to |x|^2 span about 2 qmax plus the increments, and the
    // non-EXACT pass doubles them (jfa2_eval's tie mark): keep 3 bits spare
    double qmax = (double)wx * (nx - 1) * (nx - 1) + (double)wy * (ny - 1) * (ny - 1) +
                  (double)wz * (nz - 1) * (nz - 1);
    return qmax < 268435456.0;
}

static bool ws_ok(void* ws, size_t ws_bytes, int64_t n_cells) {
    if (!ws || ws_bytes < 256 + (size_t)n_cells * sizeof(int32_t)) {
        set_error("jfa: workspace too small (rtsdf_jfa_ws_bytes)");
        return false;
    }
    return true;
}

}  // namespace rtsdf

using namespace rtsdf;

static size_t seg_bitmap_bytes(int nx, int ny, int nz) {
    return (((size_t)nx * ny * ((nz + 31) / 32)) + 255) / 256 * 256;
}

// fix-up list, two segment bitmaps, 32 per-pass segment-count slots
extern "C" size_t rtsdf_jfa_ws_bytes(int nx, int ny, int nz) {
    return 256 + (size_t)nx * ny * nz * sizeof(int32_t) + 2 * seg_bitmap_bytes(nx, ny, nz) + 256;
}

extern "C" int rtsdf_jfa_init(const uint8_t* occ, int nx, int ny, int nz, int32_t* seed,
                              int64_t* count, void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    int64_t n = (int64_t)nx * ny * nz;
    jfa_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(occ, ny, nz, n,
                                                                                  seed, count,
                                                                                  fmt_of(nx, ny, nz));
    count_launch();
    return check_launch("jfa_init");
}

extern "C" int rtsdf_jfa_step(const int32_t* src, int32_t* dst, int nx, int ny, int nz,
                              int offset, double hx, double hy, double hz, int wx, int wy,
                              int wz, void* ws, size_t ws_bytes, void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    if (offset < 1 || !weights_ok(nx, ny, nz, wx, wy, wz)) {
        set_error("jfa_step: bad offset %d or weights (%d,%d,%d)", offset, wx, wy, wz);
        return RTSDF_ERR_INVALID;
    }
    if (!ws_ok(ws, ws_bytes, (int64_t)nx * ny * nz)) return RTSDF_ERR_WORKSPACE;
    JfaGeom g{nx, ny, nz, 0, nx, 0, 0, 0, 0, offset, hx, hy, hz, wx, wy, wz,
              wx > 0 && fp64_exact(hx, hy, hz, nx, ny, nz), 0, nx};
    g.fmt = fmt_of(nx, ny, nz);
    PlaneSrc s{src, nullptr, nullptr};
    return launch_step(s, dst, g, false, ws, (cudaStream_t)stream);
}

extern "C" int rtsdf_jfa_step_slab(const int32_t* local, const int32_t* halo_lo,
                                   const int32_t* halo_hi, int32_t* dst, int nx, int x0, int nxl,
                                   int lo_first, int n_lo, int hi_first, int n_hi, int ny, int nz,
                                   int offset, double hx, double hy, double hz, int wx, int wy,
                                   int wz, int out_first, int out_count, void* ws, size_t ws_bytes,
                                   void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    if (offset < 1 || nxl < 1 || x0 < 0 || x0 + nxl > nx || !weights_ok(nx, ny, nz, wx, wy, wz) ||
        out_first < x0 || out_count < 0 || out_first + out_count > x0 + nxl) {
        set_error("jfa_step_slab: bad slab/offset/weights/output range");
        return RTSDF_ERR_INVALID;
    }
    if (out_count == 0) return RTSDF_OK;
    if (!ws_ok(ws, ws_bytes, (int64_t)nxl * ny * nz)) return RTSDF_ERR_WORKSPACE;
    JfaGeom g{nx,     ny,    nz, x0, nxl, lo_first, n_lo, hi_first, n_hi, offset, hx, hy, hz,
              wx,     wy,    wz, wx > 0 && fp64_exact(hx, hy, hz, nx, ny, nz), out_first, out_count};
    g.fmt = fmt_of(nx, ny, nz);
    PlaneSrc s{local, halo_lo, halo_hi};
    return launch_step(s, dst, g, true, ws, (cudaStream_t)stream);
}

// Per (device, dims) history of the sparse-pass input densities: the counts
// of one call are copied (async, pinned) for the next call with the same grid,
// which then decides its sparse passes without a host sync; the first call for
// a grid syncs once per sparse-eligible pass.  A stale prediction (the scene
// changed) costs speed only, never results, and is corrected by the next call.
struct SparseHistory {
    unsigned long long* counts = nullptr;  // pinned [32]: pass p's input: 0 unknown, else 1 + count
    cudaEvent_t ready = nullptr;           // compute stream -> side stream
    cudaEvent_t done = nullptr;            // counts landed
    cudaStream_t side = nullptr;           // off-critical-path copy stream
    bool valid = false;                    // a copy was published
    unsigned long long last[32];           // the newest counts that have landed
    bool have_last = false;
};

static SparseHistory* sparse_history(int nx, int ny, int nz) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int>, SparseHistory> hist;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    SparseHistory& h = hist[std::make_tuple(dev, nx, ny, nz)];
    if (!h.counts) {
        if (cudaMallocHost(&h.counts, 32 * sizeof(unsigned long long)) != cudaSuccess) {
            h.counts = nullptr;
            return nullptr;
        }
        for (int i = 0; i < 32; ++i) h.counts[i] = 0;
        cudaEventCreateWithFlags(&h.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h.done, cudaEventDisableTiming);
        cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking);
    }
    return &h;
}

// Copy this call's per-pass counts to the pinned history on the side stream
// (after the compute stream's counting kernels; off the critical path).
static bool capturing(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    return cs != cudaStreamCaptureStatusNone;
}

static void publish_counts(SparseHistory* h, const unsigned long long* slots, cudaStream_t st) {
    if (!h || !slots || capturing(st)) return;  // a graph replays the captured decisions
    // the side stream's previous copy must finish before the pinned buffer is reused
    if (h->valid && cudaEventQuery(h->done) != cudaSuccess) return;
    cudaEventRecord(h->ready, st);
    cudaStreamWaitEvent(h->side, h->ready, 0);
    cudaMemcpyAsync(h->counts, slots, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                    h->side);
    cudaEventRecord(h->done, h->side);
    h->valid = true;
}

// The full schedule (jfa.py:140-145) on one device: sparse kernel for the
// passes with k >= sparse_min_k (and k % 32 == 0) while the workspace has room
// for the bitmaps, the v2 pass kernel (INT mode) or the per-cell kernel
// otherwise; the last pass optionally writes the SDF (K3 fused, INT mode).
static int run_schedule(int32_t* a, int32_t* b, float* sdf_out, int nx, int ny, int nz, double hx,
                        double hy, double hz, int wx, int wy, int wz, double beta,
                        int64_t* empty_count, int* which, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
    const bool int_mode = wx > 0 && wy > 0 && wz > 0;
    const bool exact = int_mode && fp64_exact(hx, hy, hz, nx, ny, nz);
    int m = nx > ny ? nx : ny;
    if (nz > m) m = nz;
    int n = 1;
    while (n < m) n *= 2;  // jfa.py:58-68
    if (!seed_fmt_legacy(nx, ny, nz)) {
        // grids beyond the fixed packed layout: every pass with the per-cell
        // kernel (runtime seed fields), then seeds -> SDF
        int32_t* src = a;
        int32_t* dst = b;
        int w = 0;
        for (int off = n / 2; off >= 1; off /= 2) {
            JfaGeom g{nx, ny, nz, 0, nx, 0, 0, 0, 0, off, hx, hy, hz, wx, wy, wz, exact, 0, nx};
            g.fmt = fmt_of(nx, ny, nz);
            const int rc = launch_step(PlaneSrc{src, nullptr, nullptr}, dst, g, false, ws, st);
            if (rc != RTSDF_OK) return rc;
            int32_t* t = src;
            src = dst;
            dst = t;
            w ^= 1;
        }
        if (which) *which = w;
        if (sdf_out) return rtsdf_seeds_to_sdf(src, sdf_out, nx, ny, nz, hx, hy, hz, beta, empty_count, st);
        return RTSDF_OK;
    }
    // Sparse passes while the pass input is sparse (< 5 % of its 32-cell
    // segments hold a seed): a sparse pass only pays off while few segments
    // are active, since its active warps run the per-cell rule instead of the
    // register-tiled pass (C3: 1.1 % for the first two inputs, then 11.7 %;
    // C5: 14 % already before the second pass).  The bitmap kernels count the
    // non-empty segments of each pass input; the first call for a grid reads
    // them back at once (a small sync per eligible pass), later calls decide
    // from the previous call's counts (SparseHistory) without a sync.
    const double sparse_frac = 0.05;
    const int sparse_min_k = 64;
    const bool bm_room = ws_bytes >= rtsdf_jfa_ws_bytes(nx, ny, nz);
    const int nzb = (nz + 31) / 32;
    const int64_t n_seg = (int64_t)nx * ny * nzb;
    uint8_t* bm[2] = {nullptr, nullptr};
    if (bm_room) {
        bm[0] = (uint8_t*)ws + 256 + (size_t)nx * ny * nz * sizeof(int32_t);
        bm[1] = bm[0] + seg_bitmap_bytes(nx, ny, nz);
    }
    bool sparse_on = true;  // until the first dense input
    // inside a CUDA-graph capture: decide from the history as it stands (no
    // event queries, no syncs, no publishing); every decision is exact anyway
    const bool cap = capturing(st);
    SparseHistory* hist = bm_room ? sparse_history(nx, ny, nz) : nullptr;
    unsigned long long pred[32];
    bool predicted = false;
    if (hist) {
        // never wait for the previous call: use its counts if they have landed,
        // else the ones before (one call staler)
        if (!cap && hist->valid && cudaEventQuery(hist->done) == cudaSuccess) {
            for (int i = 0; i < 32; ++i) hist->last[i] = hist->counts[i];
            hist->have_last = true;
        }
        if (hist->have_last) {
            for (int i = 0; i < 32; ++i) pred[i] = hist->last[i];
            predicted = true;
        }
    }
    const bool big = (int64_t)nx * ny * nz >= ((int64_t)1 << 28);
    if (predicted && big && !cap) predicted = false;  // large grids: the sync is noise, measure every call
    int pass = 0;
    unsigned long long* slots = nullptr;  // per-pass input counts (1 + n), device
    if (bm_room) {
        slots = (unsigned long long*)(bm[1] + seg_bitmap_bytes(nx, ny, nz));
        // the previous call's publish copy (side stream) reads these slots:
        // the reset must come after it
        if (hist && hist->valid && !cap) cudaStreamWaitEvent(st, hist->done, 0);
        cudaMemsetAsync(slots, 0, 32 * sizeof(unsigned long long), st);
    }
    bool bm_valid = false;  // bm[0] describes src
    int32_t* src = a;
    int32_t* dst = b;
    int w = 0;
    const int64_t seg_need = (n_seg * 32 + 255) / 256;
    const unsigned seg_blocks = (unsigned)(seg_need < (int64_t)num_sms() * 16 ? seg_need : (int64_t)num_sms() * 16);
    const FastDiv dzb = make_fastdiv((uint32_t)nzb), dny = make_fastdiv((uint32_t)ny);
    for (int off = n / 2; off >= 1; off /= 2) {
        JfaGeom g{nx, ny, nz, 0, nx, 0, 0, 0, 0, off, hx, hy, hz, wx, wy, wz, exact, 0, nx};
        g.fmt = fmt_of(nx, ny, nz);
        PlaneSrc s{src, nullptr, nullptr};
        if (sdf_out && off == 1 && int_mode) {  // last pass writes the SDF directly
            // v5 leaves the tied winners of the flagged cells in the free buffer
            if (use_v5(g)) launch_pass5<true, false>(s, dst, sdf_out, g, beta, empty_count, ws, st);
            else if (use_v4(g)) launch_pass4<true, false>(s, nullptr, sdf_out, g, beta, empty_count, ws, st);
            else launch_pass2<true, false>(s, nullptr, sdf_out, g, beta, empty_count, ws, st);
            publish_counts(hist, slots, st);
            return check_launch("jfa_run_sdf");
        }
        bool sparse = false;
        if (bm_room && sparse_on && off >= sparse_min_k && off % 32 == 0 && pass < 32) {
            const bool need_bm = !bm_valid;
            if (predicted) {
                const unsigned long long v = pred[pass];
                sparse = v != 0 && (double)(v - 1) < sparse_frac * (double)n_seg;
            }
            if (need_bm && (sparse || !predicted)) {
                jfa_seg_bitmap_kernel<<<seg_blocks, 256, 0, st>>>(src, bm[0], ny, nz, dzb,
                                                                  (uint32_t)n_seg, slots + pass);
                count_launch();
            }
            if (!predicted && cap) {
                sparse = false;  // no history to decide from and no sync in a capture: dense
            } else if (!predicted) {  // first call for this grid (or a big grid): measure now
                unsigned long long v = 0;
                cudaMemcpyAsync(&v, slots + pass, sizeof(v), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                sparse = v != 0 && (double)(v - 1) < sparse_frac * (double)n_seg;
            }
            sparse_on = sparse;
        }
        if (sparse) {
            // this pass's output bitmap (+ count) feeds the next pass's decision
            const bool next_sparse = off / 2 >= sparse_min_k && (off / 2) % 32 == 0 && pass + 1 < 32;
            unsigned long long* next_slot = next_sparse ? slots + pass + 1 : nullptr;
            {
                // active list in the (not yet used) fix-up list area, its count in slot 0
                unsigned long long* n_active = (unsigned long long*)ws;
                int32_t* active = (int32_t*)((char*)ws + 256);
                cudaMemsetAsync(n_active, 0, sizeof(unsigned long long), st);
                const unsigned fill_blocks = (unsigned)((n_seg + 255) / 256);
                jfa_sparse_fill_kernel<<<fill_blocks, 256, 0, st>>>(
                    dst, g, bm[0], next_sparse ? bm[1] : nullptr, dzb, dny, active, n_active, next_slot);
                if (int_mode)
                    jfa_sparse_active_kernel<JFA_INT><<<seg_blocks, 256, 0, st>>>(
                        src, dst, g, next_sparse ? bm[1] : nullptr, dzb, dny, active, n_active, next_slot);
                else
                    jfa_sparse_active_kernel<JFA_FP64><<<seg_blocks, 256, 0, st>>>(
                        src, dst, g, next_sparse ? bm[1] : nullptr, dzb, dny, active, n_active, next_slot);
                count_launch(2);
            }
            uint8_t* t = bm[0];
            bm[0] = bm[1];
            bm[1] = t;
            bm_valid = next_sparse;
            int rc = check_launch("jfa_sparse");
            if (rc) return rc;
        } else {
            int rc = launch_step(s, dst, g, false, ws, st);
            if (rc) return rc;
            bm_valid = false;
        }
        int32_t* t = src;
        src = dst;
        dst = t;
        w ^= 1;
        ++pass;
    }
    publish_counts(hist, slots, st);
    if (which) *which = w;
    if (sdf_out) return rtsdf_seeds_to_sdf(src, sdf_out, nx, ny, nz, hx, hy, hz, beta, empty_count, st);
    return RTSDF_OK;
}

extern "C" int rtsdf_jfa_run(int32_t* a, int32_t* b, int nx, int ny, int nz, double hx,
                             double hy, double hz, int wx, int wy, int wz, int* which, void* ws,
                             size_t ws_bytes, void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    if (!weights_ok(nx, ny, nz, wx, wy, wz)) {
        set_error("jfa_run: bad weights (%d,%d,%d)", wx, wy, wz);
        return RTSDF_ERR_INVALID;
    }
    if (!ws_ok(ws, ws_bytes, (int64_t)nx * ny * nz)) return RTSDF_ERR_WORKSPACE;
    return run_schedule(a, b, nullptr, nx, ny, nz, hx, hy, hz, wx, wy, wz, 0.0, nullptr, which, ws,
                        ws_bytes, (cudaStream_t)stream);
}

extern "C" int rtsdf_jfa_run_sdf(int32_t* a, int32_t* b, float* out, int nx, int ny, int nz,
                                 double hx, double hy, double hz, int wx, int wy, int wz,
                                 double beta, int64_t* empty_count, void* ws, size_t ws_bytes,
                                 void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    if (!weights_ok(nx, ny, nz, wx, wy, wz)) {
        set_error("jfa_run_sdf: bad weights");
        return RTSDF_ERR_INVALID;
    }
    if (!ws_ok(ws, ws_bytes, (int64_t)nx * ny * nz)) return RTSDF_ERR_WORKSPACE;
    if (!out) {
        set_error("jfa_run_sdf: out is null");
        return RTSDF_ERR_INVALID;
    }
    return run_schedule(a, b, out, nx, ny, nz, hx, hy, hz, wx, wy, wz, beta, empty_count, nullptr,
                        ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int rtsdf_seeds_to_sdf_range(const int32_t* seed, float* out, int nx, int ny, int nz,
                                        int x0, int nxl, double hx, double hy, double hz,
                                        double beta, int64_t* empty_count, void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    if (x0 < 0 || nxl < 0 || x0 + nxl > nx) {
        set_error("seeds_to_sdf_range: planes [%d, %d) outside 0..%d", x0, x0 + nxl, nx);
        return RTSDF_ERR_INVALID;
    }
    if (nxl == 0) return RTSDF_OK;
    dim3 block(32, 8, 1);
    dim3 grid((nz + 31) / 32, (ny + 7) / 8, nxl);
    seeds_to_sdf_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(seed, out, x0, ny, nz, hx, hy,
                                                                  hz, beta, empty_count,
                                                                  fmt_of(nx, ny, nz));
    count_launch();
    return check_launch("seeds_to_sdf");
}

extern "C" int rtsdf_seeds_to_sdf(const int32_t* seed, float* out, int nx, int ny, int nz,
                                  double hx, double hy, double hz, double beta,
                                  int64_t* empty_count, void* stream) {
    return rtsdf_seeds_to_sdf_range(seed, out, nx, ny, nz, 0, nx, hx, hy, hz, beta, empty_count,
                                    stream);
}

extern "C" int rtsdf_seeds_packed_to_linear(const int32_t* p, int32_t* l, int nx, int ny, int nz,
                                            void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    int64_t n = (int64_t)nx * ny * nz;
    packed_to_linear_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        p, l, ny, nz, n, fmt_of(nx, ny, nz));
    count_launch();
    return check_launch("seeds_packed_to_linear");
}

extern "C" int rtsdf_seeds_linear_to_packed(const int32_t* l, int32_t* p, int nx, int ny, int nz,
                                            void* stream) {
    if (!dims_ok(nx, ny, nz)) return RTSDF_ERR_DIMS;
    int64_t n = (int64_t)nx * ny * nz;
    linear_to_packed_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        l, p, ny, nz, n, fmt_of(nx, ny, nz));
    count_launch();
    return check_launch("seeds_linear_to_packed");
}
