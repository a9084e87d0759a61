// voxel.cu -- K1: triangle -> voxel seed kernel.
//
// Restates voxel.py:117-181 (conservative closed-box 13-axis SAT, fp64, no FMA:
// this file is compiled with --fmad=false) fused with jfa.py:47-55 (self
// seeding).  The reference loops one worker per triangle (voxel.py:120), which
// is badly imbalanced on B200: the sphere_plane ground is 2 triangles covering
// ~150 k cells next to 1,280 tiny sphere triangles.  Here the (triangle, cell)
// work is expanded by a prefix sum over per-triangle bbox cell counts and a
// grid-stride loop hands every thread one (triangle, cell) pair, so all 148
// SMs stay busy whatever the triangle size distribution.
#include <cub/cub.cuh>

#include "common.cuh"

namespace rtsdf {

struct TriRange {
    int i0, j0, k0;
    int ni, nj, nk;
};

// voxel.py:49-59
__device__ __forceinline__ bool axis_sep(double v0x, double v0y, double v0z, double v1x,
                                         double v1y, double v1z, double v2x, double v2y,
                                         double v2z, double ax, double ay, double az, double ex,
                                         double ey, double ez) {
    double p0 = v0x * ax + v0y * ay + v0z * az;
    double p1 = v1x * ax + v1y * ay + v1z * az;
    double p2 = v2x * ax + v2y * ay + v2z * az;
    double r = ex * fabs(ax) + ey * fabs(ay) + ez * fabs(az);
    double mn = dmin_(p0, dmin_(p1, p2));
    double mx = dmax_(p0, dmax_(p1, p2));
    return mn > r || mx < -r;
}

// voxel.py:62-114
__device__ bool tri_box_overlap(const double* a, const double* b, const double* c, double cx,
                                double cy, double cz, double ex, double ey, double ez) {
    double v0x = a[0] - cx, v0y = a[1] - cy, v0z = a[2] - cz;
    double v1x = b[0] - cx, v1y = b[1] - cy, v1z = b[2] - cz;
    double v2x = c[0] - cx, v2y = c[1] - cy, v2z = c[2] - cz;
    if (dmin_(v0x, dmin_(v1x, v2x)) > ex || dmax_(v0x, dmax_(v1x, v2x)) < -ex) return false;
    if (dmin_(v0y, dmin_(v1y, v2y)) > ey || dmax_(v0y, dmax_(v1y, v2y)) < -ey) return false;
    if (dmin_(v0z, dmin_(v1z, v2z)) > ez || dmax_(v0z, dmax_(v1z, v2z)) < -ez) return false;
    double e0x = v1x - v0x, e0y = v1y - v0y, e0z = v1z - v0z;
    double e1x = v2x - v1x, e1y = v2y - v1y, e1z = v2z - v1z;
    double e2x = v0x - v2x, e2y = v0y - v2y, e2z = v0z - v2z;
#define AT(X, Y, Z) axis_sep(v0x, v0y, v0z, v1x, v1y, v1z, v2x, v2y, v2z, X, Y, Z, ex, ey, ez)
    if (AT(0.0, -e0z, e0y)) return false;
    if (AT(0.0, -e1z, e1y)) return false;
    if (AT(0.0, -e2z, e2y)) return false;
    if (AT(e0z, 0.0, -e0x)) return false;
    if (AT(e1z, 0.0, -e1x)) return false;
    if (AT(e2z, 0.0, -e2x)) return false;
    if (AT(-e0y, e0x, 0.0)) return false;
    if (AT(-e1y, e1x, 0.0)) return false;
    if (AT(-e2y, e2x, 0.0)) return false;
#undef AT
    double nx = e0y * e1z - e0z * e1y;
    double ny = e0z * e1x - e0x * e1z;
    double nz = e0x * e1y - e0y * e1x;
    double d = nx * v0x + ny * v0y + nz * v0z;
    double r = ex * fabs(nx) + ey * fabs(ny) + ez * fabs(nz);
    return fabs(d) <= r;
}

struct VoxParams {
    double lo[3], hi[3], h[3];
    int n[3];
    SeedFmt fmt;  // packed seed layout for the grid (common.cuh seed_fmt_for)
};

// Per triangle: gather p0/p1/p2 (voxel.py:168-170), OOB check (:171-175),
// clamped cell range (:121-132) and its cell count.
__global__ void vox_ranges_kernel(const double* __restrict__ verts, const int32_t* __restrict__ tris,
                                  int64_t T, VoxParams P, double* __restrict__ tri_pts,
                                  TriRange* __restrict__ ranges, int64_t* __restrict__ counts,
                                  int64_t* __restrict__ counters, uint8_t* __restrict__ bad_flags) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= T) return;
    double p[3][3];
    for (int v = 0; v < 3; ++v) {
        int64_t vi = tris[3 * t + v];
        for (int a = 0; a < 3; ++a) p[v][a] = verts[3 * vi + a];
    }
    double* out = tri_pts + 9 * t;
    for (int v = 0; v < 3; ++v)
        for (int a = 0; a < 3; ++a) out[3 * v + a] = p[v][a];
    bool bad = false;
    int lo_i[3], cnt[3];
    for (int a = 0; a < 3; ++a) {
        double tlo = dmin_(p[0][a], dmin_(p[1][a], p[2][a]));
        double thi = dmax_(p[0][a], dmax_(p[1][a], p[2][a]));
        bad |= (tlo < P.lo[a]) || (thi > P.hi[a]);
        double f0 = floor((tlo - P.lo[a]) / P.h[a]);
        double f1 = floor((thi - P.lo[a]) / P.h[a]);
        // clamp in fp64 first so huge values cannot overflow the int cast
        f0 = dmax_(f0, 0.0);
        f1 = dmin_(f1, (double)(P.n[a] - 1));
        int i0 = (int)f0, i1 = (int)f1;
        lo_i[a] = i0;
        cnt[a] = i1 >= i0 ? i1 - i0 + 1 : 0;
    }
    if (bad_flags) bad_flags[t] = bad;
    if (bad) {
        atomicAdd((unsigned long long*)&counters[0], 1ull);
        cnt[0] = 0;
    }
    TriRange r;
    r.i0 = lo_i[0];
    r.j0 = lo_i[1];
    r.k0 = lo_i[2];
    r.ni = cnt[0];
    r.nj = cnt[1];
    r.nk = cnt[2];
    ranges[t] = r;
    counts[t] = (int64_t)cnt[0] * cnt[1] * cnt[2];
}

// One (triangle, cell) pair per thread: binary search the inclusive prefix of
// cell counts, SAT-test the cell, self-seed on overlap (voxel.py:138-147).
__global__ void __launch_bounds__(256) vox_cells_kernel(
    const double* __restrict__ tri_pts, const TriRange* __restrict__ ranges,
    const int64_t* __restrict__ prefix, int64_t T, VoxParams P, uint8_t* __restrict__ occ,
    int32_t* __restrict__ seed, int64_t* __restrict__ counters) {
    const int64_t total = T > 0 ? prefix[T - 1] : 0;
    const int64_t nyz = (int64_t)P.n[1] * P.n[2];
    const double ex = 0.5 * P.h[0], ey = 0.5 * P.h[1], ez = 0.5 * P.h[2];
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w - threadIdx.x < total;
         w += stride) {
        bool hit = false;
        if (w < total) {
            // upper_bound: first t with prefix[t] > w
            int64_t lo = 0, hi = T - 1;
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (__ldg(prefix + mid) > w) hi = mid;
                else lo = mid + 1;
            }
            int64_t t = lo;
            int64_t local = w - (t > 0 ? __ldg(prefix + t - 1) : 0);
            TriRange r = ranges[t];
            int dk = (int)(local % r.nk);
            int64_t rest = local / r.nk;
            int dj = (int)(rest % r.nj);
            int di = (int)(rest / r.nj);
            int i = r.i0 + di, j = r.j0 + dj, k = r.k0 + dk;
            double cx = P.lo[0] + ((double)i + 0.5) * P.h[0];
            double cy = P.lo[1] + ((double)j + 0.5) * P.h[1];
            double cz = P.lo[2] + ((double)k + 0.5) * P.h[2];
            const double* pt = tri_pts + 9 * t;
            double a[3] = {pt[0], pt[1], pt[2]}, b[3] = {pt[3], pt[4], pt[5]},
                   c[3] = {pt[6], pt[7], pt[8]};
            if (tri_box_overlap(a, b, c, cx, cy, cz, ex, ey, ez)) {
                int64_t cell = (int64_t)i * nyz + (int64_t)j * P.n[2] + k;
                if (occ) occ[cell] = 1;  // all writers store the same value
                if (seed) seed[cell] = fmt_pack(i, j, k, P.fmt);
                hit = true;
            }
        }
        unsigned m = __ballot_sync(0xffffffffu, hit);
        if ((threadIdx.x & 31) == 0 && m)
            atomicAdd((unsigned long long*)&counters[1], (unsigned long long)__popc(m));
    }
}

}  // namespace rtsdf

using namespace rtsdf;

static size_t vox_scan_tmp_bytes(int64_t T) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (int64_t*)nullptr, (int64_t*)nullptr, (int)T);
    return bytes;
}

static inline size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t rtsdf_voxelize_ws_bytes(int64_t T) {
    if (T < 1) T = 1;
    return align_up(9 * sizeof(double) * T) + align_up(sizeof(TriRange) * T) +
           2 * align_up(sizeof(int64_t) * T) + align_up(vox_scan_tmp_bytes(T));
}

extern "C" int rtsdf_voxelize(const double* verts, int64_t n_verts, const int32_t* tris,
                              int64_t T, const double* lo, const double* hi, int nx, int ny,
                              int nz, uint8_t* occ, int32_t* seed, int64_t* counters,
                              uint8_t* bad_flags, void* ws, size_t ws_bytes, void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    (void)n_verts;
    if (nx < 2 || ny < 2 || nz < 2) {
        set_error("voxelize: dims must be >= 2 per axis");
        return RTSDF_ERR_INVALID;
    }
    SeedFmt fmt;
    if (seed && (!seed_fmt_for(nx, ny, nz, &fmt) || (int64_t)nx * ny * nz >= ((int64_t)1 << 31))) {
        set_error("voxelize: dims (%d, %d, %d) cannot hold packed int32 seeds", nx, ny, nz);
        return RTSDF_ERR_DIMS;
    }
    if (!counters) {
        set_error("voxelize: counters required");
        return RTSDF_ERR_INVALID;
    }
    if (ws_bytes < rtsdf_voxelize_ws_bytes(T)) {
        set_error("voxelize: workspace too small");
        return RTSDF_ERR_WORKSPACE;
    }
    VoxParams P;
    P.fmt = seed_fmt_packed();
    if (seed) P.fmt = fmt;
    int dims[3] = {nx, ny, nz};
    for (int a = 0; a < 3; ++a) {
        P.lo[a] = lo[a];
        P.hi[a] = hi[a];
        P.h[a] = (hi[a] - lo[a]) / (double)dims[a];  // voxel.py:178
        P.n[a] = dims[a];
    }
    const int64_t n_cells = (int64_t)nx * ny * nz;
    cudaMemsetAsync(counters, 0, 2 * sizeof(int64_t), stream);
    if (occ) cudaMemsetAsync(occ, 0, n_cells, stream);
    if (seed) cudaMemsetAsync(seed, 0xff, n_cells * sizeof(int32_t), stream);
    if (T <= 0) return check_launch("voxelize memset");
    char* p = (char*)ws;
    double* tri_pts = (double*)p;
    p += align_up(9 * sizeof(double) * T);
    TriRange* ranges = (TriRange*)p;
    p += align_up(sizeof(TriRange) * T);
    int64_t* counts = (int64_t*)p;
    p += align_up(sizeof(int64_t) * T);
    int64_t* prefix = (int64_t*)p;
    p += align_up(sizeof(int64_t) * T);
    size_t tmp_bytes = vox_scan_tmp_bytes(T);
    vox_ranges_kernel<<<(unsigned)((T + 255) / 256), 256, 0, stream>>>(
        verts, tris, T, P, tri_pts, ranges, counts, counters, bad_flags);
    cub::DeviceScan::InclusiveSum(p, tmp_bytes, counts, prefix, (int)T, stream);
    int blocks = num_sms() * 8;
    vox_cells_kernel<<<blocks, 256, 0, stream>>>(tri_pts, ranges, prefix, T, P, occ, seed,
                                                 counters);
    count_launch(4);  // ranges, CUB scan (init + scan), cells
    return check_launch("voxelize");
}
