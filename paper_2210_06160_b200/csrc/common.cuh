// common.cuh -- shared device helpers for librtsdf (sm_100a).
//
// Every fp64 expression that must be bit-identical to the reference is
// compiled with --fmad=false (see _build.py) and written in the reference's
// left-to-right order; comments cite the reference line each helper restates.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rtsdf.h"
#include "glibc_sincos.cuh"

#define RTSDF_EMPTY (-1)
#define RTSDF_MAX_DIM 1024

namespace rtsdf {

// ---- error plumbing (api.cu) ------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);
void count_launch(int n = 1);

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// ---- packed seed coordinates --------------------------------------------------
__host__ __device__ __forceinline__ int32_t pack_ijk(int i, int j, int k) {
    return (i << 20) | (j << 10) | k;
}
__device__ __forceinline__ int unpack_i(int32_t p) { return (int)((uint32_t)p >> 20); }
__device__ __forceinline__ int unpack_j(int32_t p) { return (p >> 10) & 1023; }
__device__ __forceinline__ int unpack_k(int32_t p) { return p & 1023; }

// Dims-dependent packed seeds.  Grids with every axis <= RTSDF_MAX_DIM use the
// fixed i<<20 | j<<10 | k layout above (every fast JFA kernel decodes it with
// immediates); larger grids (any axis beyond 1024, bits(nx-1) + bits(ny-1) +
// bits(nz-1) <= 31) pack k in the low bz bits, j above it, i on top, and run
// the per-cell JFA kernel, which decodes with these runtime fields.  In either
// layout numeric order is lexicographic (i, j, k) order and EMPTY = -1.
struct SeedFmt {
    int sx, sy;          // shifts of the i and j fields
    uint32_t mx, my, mz; // field masks
};
__host__ __device__ __forceinline__ SeedFmt seed_fmt_packed() { return SeedFmt{20, 10, 4095u, 1023u, 1023u}; }
__device__ __forceinline__ int fmt_i(int32_t p, const SeedFmt& f) { return (int)(((uint32_t)p >> f.sx) & f.mx); }
__device__ __forceinline__ int fmt_j(int32_t p, const SeedFmt& f) { return (int)(((uint32_t)p >> f.sy) & f.my); }
__device__ __forceinline__ int fmt_k(int32_t p, const SeedFmt& f) { return (int)((uint32_t)p & f.mz); }
__host__ __device__ __forceinline__ int32_t fmt_pack(int i, int j, int k, const SeedFmt& f) {
    return (int32_t)(((uint32_t)i << f.sx) | ((uint32_t)j << f.sy) | (uint32_t)k);
}
inline int bits_for(int n) {  // bits to hold 0 .. n-1 (>= 1)
    int b = 1;
    while (b < 31 && (1 << b) < n) ++b;
    return b;
}
inline bool seed_fmt_legacy(int nx, int ny, int nz) {
    return nx <= RTSDF_MAX_DIM && ny <= RTSDF_MAX_DIM && nz <= RTSDF_MAX_DIM;
}
// false: the grid cannot be packed in 31 bits
inline bool seed_fmt_for(int nx, int ny, int nz, SeedFmt* f) {
    if (nx < 1 || ny < 1 || nz < 1) return false;
    if (seed_fmt_legacy(nx, ny, nz)) {
        *f = seed_fmt_packed();
        return true;
    }
    const int bx = bits_for(nx), by = bits_for(ny), bz = bits_for(nz);
    if (bx + by + bz > 31) return false;
    f->sy = bz;
    f->sx = by + bz;
    f->mx = (1u << bx) - 1u;
    f->my = (1u << by) - 1u;
    f->mz = (1u << bz) - 1u;
    return true;
}

// jfa.py:72-76 _center_d2, fp64, left to right, no contraction
__device__ __forceinline__ double center_d2(int di, int dj, int dk, double hx, double hy,
                                            double hz) {
    double dx = __dmul_rn((double)di, hx);
    double dy = __dmul_rn((double)dj, hy);
    double dz = __dmul_rn((double)dk, hz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// ---- unsigned 32-bit division by a launch-constant divisor -------------------
// q = (umulhi(n, m) + n) >> s with s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1
// (Granlund-Montgomery); exact for every n < 2^31 (t + n cannot wrap).
struct FastDiv {
    uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.s = s;
    f.m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.m) + n) >> f.s;
}

// ---- field.py:95-128 trilinear (f32 samples promoted to fp64) -------------------
struct FieldView {
    const float* data;
    int nx, ny, nz;
    double lox, loy, loz, hx, hy, hz;
    float bias;  // subtracted from every sample in f32 (field.py:161 fused); 0 = none
};

__device__ __forceinline__ double dmin_(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax_(double a, double b) { return a > b ? a : b; }

// One axis of the trilinear lookup: the lower corner index i, the upper j and
// the fraction f (field.py:104-118 for a single coordinate).
struct AxisW {
    int i, j;
    double f;
};

__device__ __forceinline__ AxisW axis_weight(double p, double lo, double h, int n) {
    double g = __dsub_rn(__ddiv_rn(__dsub_rn(p, lo), h), 0.5);
    g = dmin_(dmax_(g, 0.0), (double)n - 1.0);
    AxisW w;
    w.i = n > 1 ? min((int)g, n - 2) : 0;
    w.f = __dsub_rn(g, (double)w.i);
    w.j = n > 1 ? w.i + 1 : w.i;
    return w;
}

__device__ __forceinline__ double trilinear_w(const FieldView& f, const AxisW& x, const AxisW& y,
                                              const AxisW& z) {
    const int64_t sx = (int64_t)f.ny * f.nz, sy = f.nz;
    const float* d = f.data;
    const float b = f.bias;
    double c000 = __fsub_rn(__ldg(d + x.i * sx + y.i * sy + z.i), b);
    double c100 = __fsub_rn(__ldg(d + x.j * sx + y.i * sy + z.i), b);
    double c010 = __fsub_rn(__ldg(d + x.i * sx + y.j * sy + z.i), b);
    double c110 = __fsub_rn(__ldg(d + x.j * sx + y.j * sy + z.i), b);
    double c001 = __fsub_rn(__ldg(d + x.i * sx + y.i * sy + z.j), b);
    double c101 = __fsub_rn(__ldg(d + x.j * sx + y.i * sy + z.j), b);
    double c011 = __fsub_rn(__ldg(d + x.i * sx + y.j * sy + z.j), b);
    double c111 = __fsub_rn(__ldg(d + x.j * sx + y.j * sy + z.j), b);
    const double fx = x.f, fy = y.f, fz = z.f;
    double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy), ofz = __dsub_rn(1.0, fz);
    double c00 = __dadd_rn(__dmul_rn(c000, ofx), __dmul_rn(c100, fx));
    double c10 = __dadd_rn(__dmul_rn(c010, ofx), __dmul_rn(c110, fx));
    double c01 = __dadd_rn(__dmul_rn(c001, ofx), __dmul_rn(c101, fx));
    double c11 = __dadd_rn(__dmul_rn(c011, ofx), __dmul_rn(c111, fx));
    double c0 = __dadd_rn(__dmul_rn(c00, ofy), __dmul_rn(c10, fy));
    double c1 = __dadd_rn(__dmul_rn(c01, ofy), __dmul_rn(c11, fy));
    return __dadd_rn(__dmul_rn(c0, ofz), __dmul_rn(c1, fz));
}

__device__ __forceinline__ double trilinear(const FieldView& f, double px, double py,
                                            double pz) {
    return trilinear_w(f, axis_weight(px, f.lox, f.hx, f.nx), axis_weight(py, f.loy, f.hy, f.ny),
                       axis_weight(pz, f.loz, f.hz, f.nz));
}

// ---- rng.py:18-53 counter-based SplitMix64 --------------------------------------
#define RTSDF_GOLDEN 0x9E3779B97F4A7C15ull
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    uint64_t z = x + RTSDF_GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream,
                                                        uint64_t tick) {
    uint64_t k = mix64(seed ^ RTSDF_GOLDEN);
    k = mix64(k ^ stream);
    return mix64(k ^ tick);
}
__device__ __forceinline__ double uniform01(uint64_t key, uint64_t counter) {
    uint64_t bits = mix64(key + counter * RTSDF_GOLDEN);
    return __dmul_rn((double)(bits >> 11), 1.0 / 9007199254740992.0);
}
__constant__ double k_two_pi = 6.283185307179586;  // a constant-bank operand, not two UMOVs per ray
__device__ __forceinline__ void unit_sphere_dir(uint64_t key, uint64_t counter, double& dx,
                                                double& dy, double& dz) {
    double u = uniform01(key, 2 * counter);
    double v = uniform01(key, 2 * counter + 1);
    double z = __dsub_rn(1.0, __dmul_rn(2.0, u));
    double r = __dsqrt_rn(dmax_(0.0, __dsub_rn(1.0, __dmul_rn(z, z))));
    double phi = __dmul_rn(k_two_pi, v);
    // rng.py:53 calls the host libm's cos / sin: its glibc FMA build, restated
    // bit for bit in glibc_sincos.cuh (CUDA's sincos differs in the last ulp);
    // the straight-line pair form keeps a warp's random phis on one path
    double s, c;
    gs::glibc_sincos_nb(phi, s, c);
    dx = __dmul_rn(r, c);
    dy = __dmul_rn(r, s);
    dz = z;
}

// ---- packed BVH (geometry.py:177-195 re-laid out for the GPU) --------------------
struct __align__(64) BvhNode {
    double lo[3];
    double hi[3];
    int32_t left;   // internal: child index; leaf: -(start + 1)
    int32_t right;  // internal: child index; leaf: count
};
struct __align__(128) BvhTri {
    double a[3], e1[3], e2[3], n[3];
    int32_t orig;
    int32_t pad[7];
};
static_assert(sizeof(BvhNode) == 64, "node layout");
static_assert(sizeof(BvhTri) == 128, "tri layout");

struct BvhView {
    const BvhNode* nodes;
    const BvhTri* tris;
};
__host__ __device__ inline BvhView bvh_view(const void* packed, int64_t n_nodes) {
    BvhView v;
    v.nodes = (const BvhNode*)packed;
    v.tris = (const BvhTri*)((const char*)packed + n_nodes * sizeof(BvhNode));
    return v;
}

// geometry.py:281-299 _ray_box_entry
__device__ __forceinline__ double ray_box_entry(const BvhNode* nd, double ox, double oy,
                                                double oz, double ix, double iy, double iz,
                                                double t_best) {
    double2 l01 = __ldg((const double2*)&nd->lo[0]);
    double2 l2h0 = __ldg((const double2*)&nd->lo[2]);
    double2 h12 = __ldg((const double2*)&nd->hi[1]);
    double t0 = __dmul_rn(__dsub_rn(l01.x, ox), ix), t1 = __dmul_rn(__dsub_rn(l2h0.y, ox), ix);
    double tmin = dmin_(t0, t1), tmax = dmax_(t0, t1);
    t0 = __dmul_rn(__dsub_rn(l01.y, oy), iy);
    t1 = __dmul_rn(__dsub_rn(h12.x, oy), iy);
    tmin = dmax_(tmin, dmin_(t0, t1));
    tmax = dmin_(tmax, dmax_(t0, t1));
    t0 = __dmul_rn(__dsub_rn(l2h0.x, oz), iz);
    t1 = __dmul_rn(__dsub_rn(h12.y, oz), iz);
    tmin = dmax_(tmin, dmin_(t0, t1));
    tmax = dmin_(tmax, dmax_(t0, t1));
    double entry = dmax_(tmin, 0.0);
    if (tmax >= entry && tmin <= t_best) return entry;
    return -1.0;
}

// geometry.py:302-328 _ray_tri (Moller-Trumbore, fp64)
__device__ __forceinline__ double ray_tri(double ox, double oy, double oz, double dx, double dy,
                                          double dz, const BvhTri* tr) {
    // (the record in three 256-bit loads up front measured slower in pass 2:
    // 1.93 -> 1.98 ms, the early-loaded doubles spill)
    const double* a = tr->a;
    const double* e1 = tr->e1;
    const double* e2 = tr->e2;
    double e2x = __ldg(e2), e2y = __ldg(e2 + 1), e2z = __ldg(e2 + 2);
    double e1x = __ldg(e1), e1y = __ldg(e1 + 1), e1z = __ldg(e1 + 2);
    double px = __dsub_rn(__dmul_rn(dy, e2z), __dmul_rn(dz, e2y));
    double py = __dsub_rn(__dmul_rn(dz, e2x), __dmul_rn(dx, e2z));
    double pz = __dsub_rn(__dmul_rn(dx, e2y), __dmul_rn(dy, e2x));
    double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, px), __dmul_rn(e1y, py)), __dmul_rn(e1z, pz));
    if (-1e-14 < det && det < 1e-14) return -1.0;
    double inv = __ddiv_rn(1.0, det);
    double tx = __dsub_rn(ox, __ldg(a)), ty = __dsub_rn(oy, __ldg(a + 1)),
           tz = __dsub_rn(oz, __ldg(a + 2));
    double u = __dmul_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(tx, px), __dmul_rn(ty, py)), __dmul_rn(tz, pz)), inv);
    if (u < 0.0 || u > 1.0) return -1.0;
    double qx = __dsub_rn(__dmul_rn(ty, e1z), __dmul_rn(tz, e1y));
    double qy = __dsub_rn(__dmul_rn(tz, e1x), __dmul_rn(tx, e1z));
    double qz = __dsub_rn(__dmul_rn(tx, e1y), __dmul_rn(ty, e1x));
    double v = __dmul_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(dx, qx), __dmul_rn(dy, qy)), __dmul_rn(dz, qz)), inv);
    if (v < 0.0 || __dadd_rn(u, v) > 1.0) return -1.0;
    double t = __dmul_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), inv);
    if (t < 1e-12) return -1.0;
    return t;
}

// geometry.py:331-392 _bvh_ray: closest hit, ties -> smaller original id,
// near child first (tl <= tr).  Returns t (or -1) with id/facing.
#define RTSDF_STACK 64
__device__ __forceinline__ double bvh_ray(const BvhView& b, double ox, double oy, double oz,
                                          double dx, double dy, double dz, double t_max,
                                          int32_t& out_id, int& out_facing) {
    int32_t stack[RTSDF_STACK];
    double ix = dx != 0.0 ? __ddiv_rn(1.0, dx) : (dx >= 0 ? 1e300 : -1e300);
    double iy = dy != 0.0 ? __ddiv_rn(1.0, dy) : (dy >= 0 ? 1e300 : -1e300);
    double iz = dz != 0.0 ? __ddiv_rn(1.0, dz) : (dz >= 0 ? 1e300 : -1e300);
    double best_t = t_max;
    int32_t best_id = -1;
    int best_facing = 0;
    out_id = -1;
    out_facing = 0;
    if (ray_box_entry(b.nodes, ox, oy, oz, ix, iy, iz, best_t) < 0.0) return -1.0;
    stack[0] = 0;
    int sp = 1;
    while (sp > 0) {
        int32_t node = stack[--sp];
        int2 lr = __ldg((const int2*)&b.nodes[node].left);
        if (lr.x < 0) {
            int start = -lr.x - 1, count = lr.y;
            for (int k = start; k < start + count; ++k) {
                const BvhTri* tr = b.tris + k;
                double t = ray_tri(ox, oy, oz, dx, dy, dz, tr);
                if (t >= 0.0 && t <= best_t) {
                    int32_t orig = __ldg(&tr->orig);
                    if (t < best_t || best_id < 0 || orig < best_id) {
                        best_t = t;
                        best_id = orig;
                        double dot = __dadd_rn(
                            __dadd_rn(__dmul_rn(dx, __ldg(tr->n)), __dmul_rn(dy, __ldg(tr->n + 1))),
                            __dmul_rn(dz, __ldg(tr->n + 2)));
                        best_facing = dot < 0.0 ? 1 : 2;
                    }
                }
            }
        } else {
            double tl = ray_box_entry(b.nodes + lr.x, ox, oy, oz, ix, iy, iz, best_t);
            double tr = ray_box_entry(b.nodes + lr.y, ox, oy, oz, ix, iy, iz, best_t);
            if (tl >= 0.0) {
                if (tr >= 0.0) {
                    if (tl <= tr) {
                        stack[sp] = lr.y;
                        stack[sp + 1] = lr.x;
                    } else {
                        stack[sp] = lr.x;
                        stack[sp + 1] = lr.y;
                    }
                    sp += 2;
                } else {
                    stack[sp++] = lr.x;
                }
            } else if (tr >= 0.0) {
                stack[sp++] = lr.y;
            }
            if (sp > RTSDF_STACK - 2) sp = RTSDF_STACK - 2;  // unreachable for depth < 62
        }
    }
    if (best_id < 0) return -1.0;
    out_id = best_id;
    out_facing = best_facing;
    return best_t;
}

}  // namespace rtsdf
