// lbvh.cu -- K5 on the device: linear BVH build and refit for the K6 search
// tree (dynamic scenes rebuild or refit it every frame without the host).
//
// The reference builds its median-split tree in Python for every animated
// frame (geometry.py:202-267 via scenes.py:56-93).  The sampler's search may
// use ANY tree: trace.cuh returns the brute-force closest hit (t, min id,
// facing) whatever the tree (the reference's own contract, geometry.py:3-6),
// so the per-frame tree is a Karras (2012) radix tree over 30-bit Morton codes
// of the triangle-box centroids (geometry.py:211's centroid), one triangle per
// leaf, built in five launches and a radix sort:
//
//   1. per triangle: fp64 box, centroid; centroid bounds by order-preserving
//      64-bit atomics;
//   2. Morton code (10 bits / axis) | triangle id -> unique 64-bit keys;
//   3. cub radix sort of the keys;
//   4. Karras split search per internal node (children, parents);
//   5. leaves upward: each leaf writes its triangle's exact fp64 record in
//      sorted order and climbs; the second child to arrive at a node forms
//      its box (atomic counter), so every box is built once; depth max'd;
//   6. the packed traversal layout (bvh.cu's pack kernels: fp64 nodes and
//      triangles, fp32 padded child boxes and pre-test triangles).
//
// Refit (rigid or deforming motion with the same triangle list) redoes 1, 5
// and 6 on the stored order and topology.  Workspace and packed sizes depend
// on the triangle count only, so neither call syncs.
#include <cub/cub.cuh>

#include "common.cuh"
#include "trace.cuh"

namespace rtsdf {

// implemented in bvh.cu
__global__ void bvh_pack_kernel(const double* __restrict__ node_lo, const double* __restrict__ node_hi,
                                const int32_t* __restrict__ node_left,
                                const int32_t* __restrict__ node_right,
                                const int32_t* __restrict__ order, const double* __restrict__ tri_a,
                                const double* __restrict__ tri_e1, const double* __restrict__ tri_e2,
                                const double* __restrict__ tri_n, int64_t n_nodes, int64_t n_tris,
                                BvhNode* __restrict__ nodes, BvhTri* __restrict__ tris);
__global__ void bvh_pack_fast_kernel(const double* __restrict__ node_lo,
                                     const double* __restrict__ node_hi,
                                     const int32_t* __restrict__ node_left,
                                     const int32_t* __restrict__ node_right,
                                     const double* __restrict__ tri_e1,
                                     const double* __restrict__ tri_e2,
                                     const double* __restrict__ tri_a, int64_t n_nodes,
                                     int64_t n_tris, FastNode* __restrict__ fnodes,
                                     FastTri* __restrict__ ftris);

struct LbvhWs {
    double* tlo;             // [3T] triangle boxes
    double* thi;
    unsigned long long* cb;  // [6] centroid bounds (ordered bits): min xyz, max xyz
    unsigned long long* keys;
    unsigned long long* sorted;
    double* nlo;             // [3N] node boxes, N = 2T - 1
    double* nhi;
    int32_t* left;           // [N]
    int32_t* right;
    int32_t* parent;         // [N]
    int32_t* counter;        // [T] internal-node arrival counters
    int32_t* order;          // [T] original triangle per leaf position
    double* ta;              // [3T] exact records in leaf order
    double* te1;
    double* te2;
    double* tn;
    void* sort_tmp;
    size_t sort_bytes;
};

static size_t sort_temp_bytes(int64_t T) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int)T, 0, 64);
    return b;
}

static size_t al256(size_t b) { return (b + 255) / 256 * 256; }

static LbvhWs lbvh_ws(void* ws, int64_t T) {
    const int64_t N = 2 * T - 1;
    LbvhWs w;
    char* p = (char*)ws;
    auto take = [&](size_t bytes) {
        char* q = p;
        p += al256(bytes);
        return q;
    };
    w.tlo = (double*)take(sizeof(double) * 3 * T);
    w.thi = (double*)take(sizeof(double) * 3 * T);
    w.cb = (unsigned long long*)take(sizeof(unsigned long long) * 6);
    w.keys = (unsigned long long*)take(sizeof(unsigned long long) * T);
    w.sorted = (unsigned long long*)take(sizeof(unsigned long long) * T);
    w.nlo = (double*)take(sizeof(double) * 3 * N);
    w.nhi = (double*)take(sizeof(double) * 3 * N);
    w.left = (int32_t*)take(sizeof(int32_t) * N);
    w.right = (int32_t*)take(sizeof(int32_t) * N);
    w.parent = (int32_t*)take(sizeof(int32_t) * N);
    w.counter = (int32_t*)take(sizeof(int32_t) * T);
    w.order = (int32_t*)take(sizeof(int32_t) * T);
    w.ta = (double*)take(sizeof(double) * 3 * T);
    w.te1 = (double*)take(sizeof(double) * 3 * T);
    w.te2 = (double*)take(sizeof(double) * 3 * T);
    w.tn = (double*)take(sizeof(double) * 3 * T);
    w.sort_bytes = sort_temp_bytes(T);
    w.sort_tmp = take(w.sort_bytes);
    return w;
}

static size_t lbvh_ws_total(int64_t T) {
    LbvhWs w = lbvh_ws(nullptr, T);
    return (size_t)((char*)w.sort_tmp - (char*)nullptr) + al256(w.sort_bytes);
}

// order-preserving map of doubles to unsigned 64-bit (for atomicMin / Max)
__device__ __forceinline__ unsigned long long dord(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunord(unsigned long long u) {
    const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    return __longlong_as_double((long long)b);
}

__global__ void lbvh_tri_kernel(const double* __restrict__ v, const int32_t* __restrict__ tris,
                                int64_t T, LbvhWs w, int bounds) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double c[3] = {0.0, 0.0, 0.0};
    const bool ok = t < T;
    if (ok) {
        const int32_t i0 = tris[3 * t], i1 = tris[3 * t + 1], i2 = tris[3 * t + 2];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double x0 = v[3 * i0 + a], x1 = v[3 * i1 + a], x2 = v[3 * i2 + a];
            const double lo = fmin(fmin(x0, x1), x2), hi = fmax(fmax(x0, x1), x2);
            w.tlo[3 * t + a] = lo;
            w.thi[3 * t + a] = hi;
            c[a] = __dmul_rn(__dadd_rn(lo, hi), 0.5);  // geometry.py:211
        }
    }
    if (!bounds) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        unsigned long long mn = ok ? dord(c[a]) : ~0ull, mx = ok ? dord(c[a]) : 0ull;
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(w.cb + a, mn);
            atomicMax(w.cb + 3 + a, mx);
        }
    }
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0x030000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void lbvh_morton_kernel(int64_t T, LbvhWs w) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    uint32_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = dunord(w.cb[a]), hi = dunord(w.cb[3 + a]);
        const double c = (w.tlo[3 * t + a] + w.thi[3 * t + a]) * 0.5;
        const double ext = hi - lo;
        double u = ext > 0.0 ? (c - lo) / ext : 0.0;
        u = fmin(fmax(u, 0.0), 1.0);
        q[a] = (uint32_t)fmin(u * 1024.0, 1023.0);
    }
    const uint32_t code = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
    w.keys[t] = ((unsigned long long)code << 32) | (unsigned long long)t;
}

__device__ __forceinline__ int lbvh_delta(const unsigned long long* k, int64_t T, int64_t i, int64_t j) {
    if (j < 0 || j >= T) return -1;
    return __clzll((long long)(k[i] ^ k[j]));  // keys are unique: < 64
}

// Karras 2012, internal node i of T - 1; leaves are nodes T - 1 + j
__global__ void lbvh_karras_kernel(int64_t T, LbvhWs w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= T - 1) return;
    const unsigned long long* k = w.sorted;
    const int d = (lbvh_delta(k, T, i, i + 1) - lbvh_delta(k, T, i, i - 1)) >= 0 ? 1 : -1;
    const int dmin = lbvh_delta(k, T, i, i - d);
    int64_t lmax = 2;
    while (lbvh_delta(k, T, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t tt = lmax / 2; tt >= 1; tt /= 2)
        if (lbvh_delta(k, T, i, i + (l + tt) * d) > dmin) l += tt;
    const int64_t j = i + l * d;
    const int dnode = lbvh_delta(k, T, i, j);
    int64_t s = 0;
    int64_t tt = l;
    do {
        tt = (tt + 1) / 2;
        if (lbvh_delta(k, T, i, i + (s + tt) * d) > dnode) s += tt;
    } while (tt > 1);
    const int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
    const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    const int32_t lc = (int32_t)(lo == gamma ? (T - 1) + gamma : gamma);
    const int32_t rc = (int32_t)(hi == gamma + 1 ? (T - 1) + gamma + 1 : gamma + 1);
    w.left[i] = lc;
    w.right[i] = rc;
    w.parent[lc] = (int32_t)i;
    w.parent[rc] = (int32_t)i;
    if (i == 0) w.parent[0] = -1;
}

// leaves upward: exact records in leaf order, leaf boxes, then each internal
// box by the second child to arrive
__global__ void lbvh_up_kernel(const double* __restrict__ v, const int32_t* __restrict__ tris,
                               const double* __restrict__ normals, int64_t T, LbvhWs w,
                               int32_t* __restrict__ depth_out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= T) return;
    const int32_t t = (int32_t)(w.sorted[j] & 0xffffffffull);
    w.order[j] = t;
    const int32_t i0 = tris[3 * t], i1 = tris[3 * t + 1], i2 = tris[3 * t + 2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double pa = v[3 * i0 + a];
        w.ta[3 * j + a] = pa;
        w.te1[3 * j + a] = __dsub_rn(v[3 * i1 + a], pa);  // geometry.py:260-262 (p1 - a, p2 - a)
        w.te2[3 * j + a] = __dsub_rn(v[3 * i2 + a], pa);
        w.tn[3 * j + a] = normals[3 * t + a];
    }
    const int32_t leaf = T == 1 ? 0 : (int32_t)(T - 1 + j);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        w.nlo[3 * leaf + a] = w.tlo[3 * t + a];
        w.nhi[3 * leaf + a] = w.thi[3 * t + a];
    }
    w.left[leaf] = -(int32_t)(j + 1);
    w.right[leaf] = 1;
    int depth = 1;
    int32_t node = T == 1 ? -1 : w.parent[leaf];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&w.counter[node], 1) == 0) break;  // the other child builds it
        __threadfence();
        const int32_t l = w.left[node], r = w.right[node];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            w.nlo[3 * node + a] = fmin(__ldcg(w.nlo + 3 * l + a), __ldcg(w.nlo + 3 * r + a));
            w.nhi[3 * node + a] = fmax(__ldcg(w.nhi + 3 * l + a), __ldcg(w.nhi + 3 * r + a));
        }
        node = w.parent[node];
        ++depth;
    }
    if (depth_out) atomicMax(depth_out, depth);
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" size_t rtsdf_lbvh_ws_bytes(int64_t n_tris) {
    return n_tris < 1 ? 0 : lbvh_ws_total(n_tris) + 256;
}

extern "C" int64_t rtsdf_lbvh_nodes(int64_t n_tris) { return n_tris < 1 ? 0 : 2 * n_tris - 1; }

extern "C" int rtsdf_lbvh_build(const double* verts, const int32_t* tris, const double* normals,
                                int64_t n_tris, int refit, void* packed, size_t packed_bytes, void* ws,
                                size_t ws_bytes, int32_t* depth_out, void* stream) {
    if (n_tris < 1 || n_tris >= ((int64_t)1 << 30) || !verts || !tris || !normals || !packed) {
        set_error("lbvh_build: bad arguments");
        return RTSDF_ERR_INVALID;
    }
    const int64_t T = n_tris, N = 2 * T - 1;
    if (!ws || ws_bytes < rtsdf_lbvh_ws_bytes(T)) {
        set_error("lbvh_build: workspace too small (rtsdf_lbvh_ws_bytes)");
        return RTSDF_ERR_WORKSPACE;
    }
    if (packed_bytes < fast_offset_tris(N, T) + (size_t)T * sizeof(FastTri)) {
        set_error("lbvh_build: packed buffer too small (rtsdf_bvh_packed_bytes)");
        return RTSDF_ERR_WORKSPACE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    LbvhWs w = lbvh_ws(ws, T);
    const unsigned g = (unsigned)((T + 127) / 128);
    int launches = 0;
    if (!refit) {
        cudaMemsetAsync(w.cb, 0xff, 3 * sizeof(unsigned long long), st);
        cudaMemsetAsync(w.cb + 3, 0x00, 3 * sizeof(unsigned long long), st);
    }
    lbvh_tri_kernel<<<g, 128, 0, st>>>(verts, tris, T, w, !refit);
    ++launches;
    if (!refit) {
        lbvh_morton_kernel<<<g, 128, 0, st>>>(T, w);
        size_t tb = w.sort_bytes;
        cub::DeviceRadixSort::SortKeys(w.sort_tmp, tb, w.keys, w.sorted, (int)T, 0, 64, st);
        launches += 2;
        if (T > 1) {
            lbvh_karras_kernel<<<(unsigned)((T - 1 + 127) / 128), 128, 0, st>>>(T, w);
            ++launches;
        }
    }
    if (T > 1) cudaMemsetAsync(w.counter, 0, sizeof(int32_t) * (T - 1), st);
    lbvh_up_kernel<<<g, 128, 0, st>>>(verts, tris, normals, T, w, depth_out);
    ++launches;
    BvhView bv = bvh_view(packed, N);
    const int64_t n = N > T ? N : T;
    bvh_pack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        w.nlo, w.nhi, w.left, w.right, w.order, w.ta, w.te1, w.te2, w.tn, N, T, (BvhNode*)bv.nodes,
        (BvhTri*)bv.tris);
    FastBvh f = fast_bvh_view(packed, N, T);
    const int64_t nf = (N + 1) > T ? N + 1 : T;
    bvh_pack_fast_kernel<<<(unsigned)((nf + 255) / 256), 256, 0, st>>>(
        w.nlo, w.nhi, w.left, w.right, w.te1, w.te2, w.ta, N, T, (FastNode*)f.nodes, (FastTri*)f.tris);
    launches += 2;
    count_launch(launches);
    return check_launch("lbvh_build");
}
