// trace.cuh -- K6 fast closest-hit traversal for the ray-sampled refinement.
//
// Same result as the reference's _bvh_ray (geometry.py:331-392), whose own
// contract is "traversal must agree with brute-force intersection"
// (geometry.py:3-6): the closest fp64 Moller-Trumbore hit over ALL triangles,
// t in [1e-12, t_max], ties -> smaller original id.  Only the *search* changes:
//
//   * boxes: fp32 slab tests on padded, outward-rounded child boxes stored in
//     the parent (one 64 B node fetch tests both children).  The padding
//     (1e-5 of the scene scale) is ~100x the fp32 rounding of the slab
//     arithmetic, so a box holding a hit point at t <= t_best is never pruned;
//   * triangles: an fp32 Moller-Trumbore pre-test with an a-priori rounding
//     bound (tri_maybe) rejects only triangles the exact test must reject;
//     every survivor is decided by the reference's exact fp64 test (ray_tri).
//
// Hence the visited set covers everything that can change the answer and
// every accepted hit is the reference's bit-exact fp64 (t, id, facing).
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

#ifndef RTSDF_FAST_STACK
#define RTSDF_FAST_STACK 40  // the host rejects search trees deeper than this
#endif

namespace rtsdf {

// Traversal counters for experiments (-DRTSDF_TRACE_STATS builds only):
// [0] node visits, [1] leaf visits, [2] fp32 triangle pre-tests, [3] exact tests
#ifdef RTSDF_TRACE_STATS
// [4..11]: per-ray node-visit histogram of the long-ray traversal (bins 0-1,
// 2-3, 4-7, 8-15, 16-31, 32-63, 64-127, 128+)
static __device__ unsigned long long g_trace_stats[12];
#define RTSDF_TSTAT(i, v) atomicAdd(&g_trace_stats[i], (unsigned long long)(v))
#else
#define RTSDF_TSTAT(i, v) ((void)0)
#endif

struct __align__(64) FastNode {
    float lo0[3], hi0[3];  // child 0 box (padded, outward rounded)
    float lo1[3], hi1[3];  // child 1 box
    int32_t c0, c1;        // child refs: internal >= 0; leaf -(start * 8 + count) - 1
    int32_t v0, v1;        // 1 = child present, 0 = none
};
static_assert(sizeof(FastNode) == 64, "fast node layout");

struct __align__(16) FastTri {
    float a[3];
    float e1[3];
    float e2[3];
    float scale;  // |e1|_1 + |e2|_1 rounded up (rounding bound)
    float amag;   // |a|_1 rounded up (tri_maybe's fp32-vertex error term)
    float pad_;
};
static_assert(sizeof(FastTri) == 48, "fast tri layout");

struct FastBvh {
    const FastNode* nodes;  // n_nodes + 1 entries; [n_nodes] = virtual parent of the root
    const FastTri* tris;
    const BvhTri* exact;    // fp64 triangles for ray_tri
    int32_t root;
};

__host__ __device__ inline size_t fast_offset_nodes(int64_t n_nodes, int64_t n_tris) {
    return (size_t)n_nodes * sizeof(BvhNode) + (size_t)n_tris * sizeof(BvhTri);
}
__host__ __device__ inline size_t fast_offset_tris(int64_t n_nodes, int64_t n_tris) {
    return fast_offset_nodes(n_nodes, n_tris) + (size_t)(n_nodes + 1) * sizeof(FastNode);
}

__host__ __device__ inline FastBvh fast_bvh_view(const void* packed, int64_t n_nodes,
                                                 int64_t n_tris) {
    FastBvh f;
    const char* p = (const char*)packed;
    f.exact = (const BvhTri*)(p + (size_t)n_nodes * sizeof(BvhNode));
    f.nodes = (const FastNode*)(p + fast_offset_nodes(n_nodes, n_tris));
    f.tris = (const FastTri*)(p + fast_offset_tris(n_nodes, n_tris));
    f.root = (int32_t)n_nodes;
    return f;
}

struct RayF {
    float ix, iy, iz;     // clamped reciprocal direction
    float oix, oiy, oiz;  // origin * reciprocal
};

// The reciprocal only steers the conservative box pre-test: MUFU.RCP's <= 1 ulp
// error is far inside the 1e-5 * scene-scale box padding, and every hit is
// confirmed in exact fp64, so the approximate reciprocal cannot change a result.
// For a (near-)zero component the sign of the 1e30 stand-in is irrelevant: the
// slab interval is [min, max] of the two planes either way.
__device__ __forceinline__ float clamp_inv(double d) {
    const float f = (float)d;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
    return fabsf(f) < 1e-30f ? copysignf(1e30f, f) : r;  // |1/f| <= ~1e30 otherwise
}

#define RTSDF_FINF __int_as_float(0x7f800000)

// fp32 upper bound of t_max for the box tests (+inf beyond fp32 range)
__host__ __device__ inline float tmax_bound(double t_max) {
#ifdef __CUDA_ARCH__
    return t_max < 3.0e38 ? __double2float_ru(t_max) : __int_as_float(0x7f800000);
#else
    if (!(t_max < 3.0e38)) return INFINITY;
    float f = (float)t_max;
    return (double)f < t_max ? nextafterf(f, INFINITY) : f;
#endif
}

// Octant of a ray: bit a set when the axis-a inverse direction is negative
// (its sign bit: clamp_inv keeps the sign of a (near-)zero component).
__device__ __forceinline__ int ray_octant(float ix, float iy, float iz) {
    return (int)((__float_as_uint(ix) >> 31) | ((__float_as_uint(iy) >> 31) << 1) |
                 ((__float_as_uint(iz) >> 31) << 2));
}

// Slab test on a ray-octant copy of the boxes (rtsdf_bvh4_collapse_host):
// n* hold the planes nearer along the ray, f* the farther ones.  fmaf is
// monotonic in the plane for a fixed-sign ix, so these are exactly box_entry's
// min / max pairs -- the same entry t bit for bit -- without the six pair
// min / max instructions; t_best folds into the exit side (tmin <= min(tmax,
// t_best) is box_entry's two tests).
__device__ __forceinline__ float box_entry_nf(float nx, float ny, float nz, float fx, float fy,
                                              float fz, const RayF& r, float t_best) {
    const float tx0 = fmaf(nx, r.ix, -r.oix), tx1 = fmaf(fx, r.ix, -r.oix);
    const float ty0 = fmaf(ny, r.iy, -r.oiy), ty1 = fmaf(fy, r.iy, -r.oiy);
    const float tz0 = fmaf(nz, r.iz, -r.oiz), tz1 = fmaf(fz, r.iz, -r.oiz);
    const float tmin = fmaxf(fmaxf(tx0, ty0), fmaxf(tz0, 0.0f));
    const float tmax = fminf(fminf(tx1, ty1), fminf(tz1, t_best));
    return tmin <= tmax ? tmin : RTSDF_FINF;
}

// Padded child box slab test: entry t (>= 0) or +inf if missed / beyond t_best.
__device__ __forceinline__ float box_entry(float lx, float ly, float lz, float hx, float hy,
                                           float hz, const RayF& r, float t_best) {
    float tx0 = fmaf(lx, r.ix, -r.oix), tx1 = fmaf(hx, r.ix, -r.oix);
    float ty0 = fmaf(ly, r.iy, -r.oiy), ty1 = fmaf(hy, r.iy, -r.oiy);
    float tz0 = fmaf(lz, r.iz, -r.oiz), tz1 = fmaf(hz, r.iz, -r.oiz);
    float tmin = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
    float tmax = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fmaxf(tz0, tz1));
    return (tmin <= tmax && tmin <= t_best) ? tmin : RTSDF_FINF;
}

// fp32 Moller-Trumbore on un-normalised values with an a-priori error bound
// eb >= |fp32 - exact| of det, U, V, W (inputs rounded to fp32, ~10 roundings,
// padded ~4x).  Returns false only when the exact test must reject.
// cm > 0: T was formed in fp32 from fp32-rounded origin and vertex (o_f - a_f)
// instead of rounding the fp64 difference; each component then carries an
// extra absolute error <= 2^-24 (|o_c| + |a_c|), i.e. |dT|_1 <= 2^-24 cm with
// cm = |o|_1 + |a|_1, which moves U and V by <= |dT|_1 scale and W by
// <= |dT|_1 scale^2 -- added to eb with a 4x margin.
__device__ __forceinline__ bool tri_maybe(const FastTri& tr, float tx, float ty, float tz,
                                          float dx, float dy, float dz, float t_best,
                                          float cm = 0.0f) {
    float px = __fsub_rn(__fmul_rn(dy, tr.e2[2]), __fmul_rn(dz, tr.e2[1]));
    float py = __fsub_rn(__fmul_rn(dz, tr.e2[0]), __fmul_rn(dx, tr.e2[2]));
    float pz = __fsub_rn(__fmul_rn(dx, tr.e2[1]), __fmul_rn(dy, tr.e2[0]));
    float det = fmaf(tr.e1[0], px, fmaf(tr.e1[1], py, __fmul_rn(tr.e1[2], pz)));
    float U = fmaf(tx, px, fmaf(ty, py, __fmul_rn(tz, pz)));
    float qx = __fsub_rn(__fmul_rn(ty, tr.e1[2]), __fmul_rn(tz, tr.e1[1]));
    float qy = __fsub_rn(__fmul_rn(tz, tr.e1[0]), __fmul_rn(tx, tr.e1[2]));
    float qz = __fsub_rn(__fmul_rn(tx, tr.e1[1]), __fmul_rn(ty, tr.e1[0]));
    float V = fmaf(dx, qx, fmaf(dy, qy, __fmul_rn(dz, qz)));
    float W = fmaf(tr.e2[0], qx, fmaf(tr.e2[1], qy, __fmul_rn(tr.e2[2], qz)));
    float tn = fabsf(tx) + fabsf(ty) + fabsf(tz);
    float eb = 4e-6f * (tn + 1.0f) * tr.scale * (tr.scale + 1.0f) +
               2.4e-7f * cm * tr.scale * fmaxf(1.0f, tr.scale);
    float ad = fabsf(det);
    if (!(ad > 4.0f * eb)) return true;  // ill-conditioned, tiny or NaN: exact test decides
    float s = det > 0.0f ? 1.0f : -1.0f;
    float Us = U * s, Vs = V * s, Ws = W * s;
    if (Us < -eb || Vs < -eb || Ws < -eb) return false;
    if (Us + Vs > ad + 3.0f * eb) return false;
    if (Ws > t_best * (ad + eb) + eb * (1.0f + t_best)) return false;
    return true;
}

// Closest hit, brute-force equivalent.  `stack` is this thread's slot in a
// shared-memory stack with `stride` (= blockDim) between entries.  budget > 0
// bounds the number of internal-node visits: when it runs out the search is
// abandoned and *complete is set false (the caller re-traces the ray later
// with no budget); budget <= 0 = unbounded.
__device__ __forceinline__ double trace_fast(const FastBvh& b, double ox, double oy, double oz,
                                             double dx, double dy, double dz, double t_max,
                                             int32_t* stack, int stride, int32_t& out_id,
                                             int& out_facing, int budget = 0,
                                             bool* complete = nullptr) {
    RayF r;
    r.ix = clamp_inv(dx);
    r.iy = clamp_inv(dy);
    r.iz = clamp_inv(dz);
    r.oix = (float)ox * r.ix;
    r.oiy = (float)oy * r.iy;
    r.oiz = (float)oz * r.iz;
    const float fdx = (float)dx, fdy = (float)dy, fdz = (float)dz;
    double best_t = t_max;
    int32_t best_id = -1;
    int best_facing = 0;
    float tb = t_max < 3.0e38 ? __double2float_ru(t_max) : RTSDF_FINF;
    int sp = 0;
    int32_t node = b.root;
    if (complete) *complete = true;
    while (true) {
        if (node >= 0) {  // internal: test both children, descend into the nearer
            if (budget > 0 && --budget == 0) {
                if (complete) *complete = false;
                break;
            }
            const FastNode* nd = b.nodes + node;
            float4 a0 = __ldg((const float4*)&nd->lo0[0]);  // lo0 xyz, hi0 x
            float4 a1 = __ldg((const float4*)&nd->hi0[1]);  // hi0 yz, lo1 xy
            float4 a2 = __ldg((const float4*)&nd->lo1[2]);  // lo1 z, hi1 xyz
            int4 cc = __ldg((const int4*)&nd->c0);
            float t0 = cc.z ? box_entry(a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, r, tb) : RTSDF_FINF;
            float t1 = cc.w ? box_entry(a1.z, a1.w, a2.x, a2.y, a2.z, a2.w, r, tb) : RTSDF_FINF;
            bool h0 = t0 != RTSDF_FINF, h1 = t1 != RTSDF_FINF;
            if (h0 && h1) {
                bool first0 = t0 <= t1;
                stack[(sp++) * stride] = first0 ? cc.y : cc.x;
                node = first0 ? cc.x : cc.y;
                continue;
            }
            if (h0 || h1) {
                node = h0 ? cc.x : cc.y;
                continue;
            }
        } else {  // leaf: fp32 pre-test, exact fp64 confirm
            int32_t code = -node - 1;
            int start = code >> 3, count = code & 7;
            for (int k = start; k < start + count; ++k) {
                const FastTri* ft = b.tris + k;
                float4 f0 = __ldg((const float4*)&ft->a[0]);
                float4 f1 = __ldg((const float4*)&ft->e1[1]);
                float4 f2 = __ldg((const float4*)&ft->e2[2]);
                FastTri tr;
                tr.e1[0] = f0.w; tr.e1[1] = f1.x; tr.e1[2] = f1.y;
                tr.e2[0] = f1.z; tr.e2[1] = f1.w; tr.e2[2] = f2.x;
                tr.scale = f2.y;
                const BvhTri* ex = b.exact + k;
                // T = o - a in fp64 (exactly the reference's tx/ty/tz), rounded once
                float tx = (float)(ox - __ldg(ex->a)), ty = (float)(oy - __ldg(ex->a + 1)),
                      tz = (float)(oz - __ldg(ex->a + 2));
                if (!tri_maybe(tr, tx, ty, tz, fdx, fdy, fdz, tb)) continue;
                double t = ray_tri(ox, oy, oz, dx, dy, dz, ex);
                if (t >= 0.0 && t <= best_t) {
                    int32_t orig = __ldg(&ex->orig);
                    if (t < best_t || best_id < 0 || orig < best_id) {
                        best_t = t;
                        best_id = orig;
                        double dot = __dadd_rn(
                            __dadd_rn(__dmul_rn(dx, __ldg(ex->n)), __dmul_rn(dy, __ldg(ex->n + 1))),
                            __dmul_rn(dz, __ldg(ex->n + 2)));
                        best_facing = dot < 0.0 ? 1 : 2;
                        tb = __double2float_ru(best_t);
                    }
                }
            }
        }
        if (sp == 0) break;
        node = stack[(--sp) * stride];
    }
    out_id = best_id;
    out_facing = best_facing;
    return best_id < 0 ? -1.0 : best_t;
}

// ---------------------------------------------------------------------------
// 4-wide variant of the same search (BVH4 collapsed from the SAH binary tree):
// half the depth, four independent slab tests per node fetch (more ILP, fewer
// divergent loop trips).  Same conservative padding, same pre-test and exact
// confirm, so the result is the same brute-force closest hit.
// Stored as 8 interleaved ray-octant copies (record 8 i + o, lo / hi swapped
// on the axes set in o): traversal starts at record `octant` and adds it to
// every inner child ref.
struct __align__(128) FastNode4 {
    float lox[4], loy[4], loz[4];
    float hix[4], hiy[4], hiz[4];
    int32_t child[4];  // >= 0 record of copy 0 (8 i); < 0 leaf -(start * 8 + count) - 1; INT_MAX empty
    int32_t pad[4];
};
static_assert(sizeof(FastNode4) == 128, "node4 layout");

// One BVH4 node (128 B, 128-B aligned) in four 256-bit loads (LDG.256,
// sm_100) instead of seven 128-bit ones.
__device__ __forceinline__ void load_node4(const FastNode4* nd, float4& lx, float4& ly, float4& lz,
                                           float4& hx, float4& hy, float4& hz, int4& ch) {
    const float* q = nd->lox;
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(lx.x), "=f"(lx.y), "=f"(lx.z), "=f"(lx.w), "=f"(ly.x), "=f"(ly.y), "=f"(ly.z), "=f"(ly.w)
        : "l"(q));
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(lz.x), "=f"(lz.y), "=f"(lz.z), "=f"(lz.w), "=f"(hx.x), "=f"(hx.y), "=f"(hx.z), "=f"(hx.w)
        : "l"(q + 8));
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(hy.x), "=f"(hy.y), "=f"(hy.z), "=f"(hy.w), "=f"(hz.x), "=f"(hz.y), "=f"(hz.z), "=f"(hz.w)
        : "l"(q + 16));
    ch = __ldg((const int4*)nd->child);
}

struct FastBvh4 {
    const FastNode4* nodes;
    const FastTri* tris;
    const BvhTri* exact;
};

// End of the packed binary search tree, rounded up to 128 B: the BVH4 nodes
// appended there are 128-B aligned (load_node4's 256-bit loads need 32 B).
__host__ __device__ inline size_t fast_packed_bytes(int64_t n_nodes, int64_t n_tris) {
    return (fast_offset_tris(n_nodes, n_tris) + (size_t)n_tris * sizeof(FastTri) + 127) & ~(size_t)127;
}

__host__ __device__ inline FastBvh4 fast_bvh4_view(const void* packed, int64_t n_nodes,
                                                   int64_t n_tris) {
    FastBvh4 f;
    const char* p = (const char*)packed;
    f.exact = (const BvhTri*)(p + (size_t)n_nodes * sizeof(BvhNode));
    f.tris = (const FastTri*)(p + fast_offset_tris(n_nodes, n_tris));
    f.nodes = (const FastNode4*)(p + fast_packed_bytes(n_nodes, n_tris));
    return f;
}

__device__ __forceinline__ bool leaf_tris(const FastTri* __restrict__ tris, const BvhTri* exact,
                                          int32_t ref, double ox, double oy, double oz, double dx,
                                          double dy, double dz, float fdx, float fdy, float fdz,
                                          double& best_t, int32_t& best_id, int& best_facing,
                                          float& tb) {
    const int32_t code = -ref - 1;
    const int start = code >> 3, count = code & 7;
    bool improved = false;
    // (all pre-tests of the leaf first, then the exact tests of the candidates
    // -- fewer divergent exact-path trips, but the pre-tests lose the tighter
    // tb of an earlier exact hit in the same leaf: pass 2 1.93 -> 2.19 ms)
    for (int k = start; k < start + count; ++k) {
        const FastTri* ft = tris + k;
        float4 f0 = __ldg((const float4*)&ft->a[0]);
        float4 f1 = __ldg((const float4*)&ft->e1[1]);
        float4 f2 = __ldg((const float4*)&ft->e2[2]);
        FastTri tr;
        tr.e1[0] = f0.w; tr.e1[1] = f1.x; tr.e1[2] = f1.y;
        tr.e2[0] = f1.z; tr.e2[1] = f1.w; tr.e2[2] = f2.x;
        tr.scale = f2.y;
        const BvhTri* ex = exact + k;
        // T from the fp32 origin and vertex: the fp64 triangle record is only
        // touched by the exact confirmation (the pre-test's error bound covers
        // the two extra roundings, see tri_maybe)
        const float fox = (float)ox, foy = (float)oy, foz = (float)oz;
        const float tx = __fsub_rn(fox, f0.x), ty = __fsub_rn(foy, f0.y), tz = __fsub_rn(foz, f0.z);
        const float cm = fabsf(fox) + fabsf(foy) + fabsf(foz) + f2.z;
        RTSDF_TSTAT(2, 1);
        if (!tri_maybe(tr, tx, ty, tz, fdx, fdy, fdz, tb, cm)) continue;
        RTSDF_TSTAT(3, 1);
        double t = ray_tri(ox, oy, oz, dx, dy, dz, ex);
        if (t >= 0.0 && t <= best_t) {
            int32_t orig = __ldg(&ex->orig);
            if (t < best_t || best_id < 0 || orig < best_id) {
                best_t = t;
                best_id = orig;
                double dot = __dadd_rn(
                    __dadd_rn(__dmul_rn(dx, __ldg(ex->n)), __dmul_rn(dy, __ldg(ex->n + 1))),
                    __dmul_rn(dz, __ldg(ex->n + 2)));
                best_facing = dot < 0.0 ? 1 : 2;
                tb = __double2float_ru(best_t);
                improved = true;
            }
        }
    }
    return improved;
}

// Each stack entry carries its box entry distance (fp16, rounded down: a lower
// bound), and a popped entry is skipped once it lies beyond the current best
// hit's fp32 upper bound tb -- the same conservative test box_entry applied at
// push time, with the tighter tb found since (ties at t == best_t survive).
__device__ __forceinline__ double trace_fast4(const FastBvh4& b, double ox, double oy, double oz,
                                              double dx, double dy, double dz, double t_max,
                                              int32_t* stack, __half* tstack, int stride,
                                              int32_t& out_id, int& out_facing, float tb0,
                                              int budget = 0, bool* complete = nullptr) {
    RayF r;
    r.ix = clamp_inv(dx);
    r.iy = clamp_inv(dy);
    r.iz = clamp_inv(dz);
    r.oix = (float)ox * r.ix;
    r.oiy = (float)oy * r.iy;
    r.oiz = (float)oz * r.iz;
    const float fdx = (float)dx, fdy = (float)dy, fdz = (float)dz;
    double best_t = t_max;
    int32_t best_id = -1;
    int best_facing = 0;
    float tb = tb0;  // tmax_bound(t_max), computed once by the caller
    int sp = 0;
    int32_t node = 0;
    const FastNode4* base = b.nodes + ray_octant(r.ix, r.iy, r.iz);  // this ray's copy
    if (complete) *complete = true;
    while (true) {
        if (node >= 0) {
            if (budget > 0 && --budget == 0) {
                if (complete) *complete = false;
                break;
            }
            const FastNode4* nd = base + node;
            RTSDF_TSTAT(0, 1);
            float4 lx, ly, lz, hx, hy, hz;
            int4 ch;
            load_node4(nd, lx, ly, lz, hx, hy, hz, ch);
            float t[4];
            t[0] = box_entry_nf(lx.x, ly.x, lz.x, hx.x, hy.x, hz.x, r, tb);
            t[1] = box_entry_nf(lx.y, ly.y, lz.y, hx.y, hy.y, hz.y, r, tb);
            t[2] = box_entry_nf(lx.z, ly.z, lz.z, hx.z, hy.z, hz.z, r, tb);
            t[3] = box_entry_nf(lx.w, ly.w, lz.w, hx.w, hy.w, hz.w, r, tb);
            int32_t c[4] = {ch.x, ch.y, ch.z, ch.w};
            // nearest hit child is visited next; the other hits go on the stack
            // (a full sort that pushes them farthest first measured 1.93 ->
            // 2.17 ms in pass 2)
            int nearest = -1;
            float tn = RTSDF_FINF;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (t[q] < tn) {
                    tn = t[q];
                    nearest = q;
                }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (q != nearest && t[q] != RTSDF_FINF) {
                    stack[sp * stride] = c[q];
                    tstack[sp * stride] = __float2half_rd(t[q]);
                    ++sp;
                }
            if (nearest >= 0) {
                // select, not c[nearest]: a dynamic index puts c[] in local
                // memory (a 16-B spill store + reload per visit, measured)
                int32_t cn = c[0];
#pragma unroll
                for (int q = 1; q < 4; ++q) cn = nearest == q ? c[q] : cn;
                node = cn;
                continue;
            }
        } else {
            RTSDF_TSTAT(1, 1);
            leaf_tris(b.tris, b.exact, node, ox, oy, oz, dx, dy, dz, fdx, fdy, fdz, best_t,
                      best_id, best_facing, tb);
        }
        bool more = false;
        while (sp > 0) {
            --sp;
            if (__half2float(tstack[sp * stride]) <= tb) {
                node = stack[sp * stride];
                more = true;
                break;
            }
        }
        if (!more) break;
    }
    out_id = best_id;
    out_facing = best_facing;
    return best_id < 0 ? -1.0 : best_t;
}

}  // namespace rtsdf
