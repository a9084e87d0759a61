// validate.cu -- the reference's validation oracles on the GPU:
//
//   * exact_distance_many (geometry.py:588-594): exact unsigned point-to-mesh
//     distance, Eberly's point-triangle regions (geometry.py:417-510) over
//     the reference-order fp64 BVH with the reference's own traversal order
//     and pruning rule (_bvh_closest_d2, geometry.py:521-565) -- where two
//     triangles give d2 values one ulp apart (a shared closest vertex) the
//     pruning decides which one is reported, so the order is part of the
//     bit-exact result;
//   * reference_visibility (render.py:195-254): per covered pixel, the
//     fraction of spp cone-sampled shadow rays with no hit (closest-hit
//     traversal of the reference-order BVH, t_max = inf).  Directions use
//     the bit-exact restatement of the host libm's cos/sin (glibc_sincos.cuh).
//
// One thread per point / pixel, fp64 without contraction (--fmad=false).
#include "common.cuh"

namespace rtsdf {

// geometry.py:417-510 _point_tri_d2
__device__ __forceinline__ double point_tri_d2(double px, double py, double pz, const double* a,
                                               const double* e1_, const double* e2_) {
    const double e1x = __ldg(e1_), e1y = __ldg(e1_ + 1), e1z = __ldg(e1_ + 2);
    const double e2x = __ldg(e2_), e2y = __ldg(e2_ + 1), e2z = __ldg(e2_ + 2);
    const double dx = __ldg(a) - px, dy = __ldg(a + 1) - py, dz = __ldg(a + 2) - pz;
    const double A = e1x * e1x + e1y * e1y + e1z * e1z;
    const double B = e1x * e2x + e1y * e2y + e1z * e2z;
    const double Cc = e2x * e2x + e2y * e2y + e2z * e2z;
    const double D = e1x * dx + e1y * dy + e1z * dz;
    const double E = e2x * dx + e2y * dy + e2z * dz;
    const double det = A * Cc - B * B;
    double s = B * E - Cc * D;
    double t = B * D - A * E;
    if (s + t <= det) {
        if (s < 0.0) {
            if (t < 0.0) {  // region 4
                if (D < 0.0) {
                    t = 0.0;
                    s = -D >= A ? 1.0 : -D / A;
                } else {
                    s = 0.0;
                    t = E >= 0.0 ? 0.0 : (-E >= Cc ? 1.0 : -E / Cc);
                }
            } else {  // region 3
                s = 0.0;
                t = E >= 0.0 ? 0.0 : (-E >= Cc ? 1.0 : -E / Cc);
            }
        } else if (t < 0.0) {  // region 5
            t = 0.0;
            s = D >= 0.0 ? 0.0 : (-D >= A ? 1.0 : -D / A);
        } else {  // region 0
            const double inv = 1.0 / det;
            s *= inv;
            t *= inv;
        }
    } else {
        if (s < 0.0) {  // region 2
            const double tmp0 = B + D, tmp1 = Cc + E;
            if (tmp1 > tmp0) {
                const double numer = tmp1 - tmp0, denom = A - 2.0 * B + Cc;
                s = numer >= denom ? 1.0 : numer / denom;
                t = 1.0 - s;
            } else {
                s = 0.0;
                t = tmp1 <= 0.0 ? 1.0 : (E >= 0.0 ? 0.0 : -E / Cc);
            }
        } else if (t < 0.0) {  // region 6
            const double tmp0 = B + E, tmp1 = A + D;
            if (tmp1 > tmp0) {
                const double numer = tmp1 - tmp0, denom = A - 2.0 * B + Cc;
                t = numer >= denom ? 1.0 : numer / denom;
                s = 1.0 - t;
            } else {
                t = 0.0;
                s = tmp1 <= 0.0 ? 1.0 : (D >= 0.0 ? 0.0 : -D / A);
            }
        } else {  // region 1
            const double numer = (Cc + E) - (B + D);
            if (numer <= 0.0) {
                s = 0.0;
            } else {
                const double denom = A - 2.0 * B + Cc;
                s = numer >= denom ? 1.0 : numer / denom;
            }
            t = 1.0 - s;
        }
    }
    const double qx = dx + s * e1x + t * e2x;
    const double qy = dy + s * e1y + t * e2y;
    const double qz = dz + s * e1z + t * e2z;
    return qx * qx + qy * qy + qz * qz;
}

// geometry.py:512-518 _point_box_d2
__device__ __forceinline__ double point_box_d2(const BvhNode* nd, double px, double py, double pz) {
    const double dx = fmax(fmax(__ldg(nd->lo) - px, 0.0), px - __ldg(nd->hi));
    const double dy = fmax(fmax(__ldg(nd->lo + 1) - py, 0.0), py - __ldg(nd->hi + 1));
    const double dz = fmax(fmax(__ldg(nd->lo + 2) - pz, 0.0), pz - __ldg(nd->hi + 2));
    return dx * dx + dy * dy + dz * dz;
}

__global__ void __launch_bounds__(128) exact_distance_kernel(BvhView b, const double* __restrict__ pts,
                                                             int64_t n, double* __restrict__ out) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double px = pts[3 * q], py = pts[3 * q + 1], pz = pts[3 * q + 2];
    int32_t stack[RTSDF_STACK];
    double best = 1e300;
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const int32_t node = stack[--sp];
        if (point_box_d2(b.nodes + node, px, py, pz) >= best) continue;
        const int2 lr = __ldg((const int2*)&b.nodes[node].left);
        if (lr.x < 0) {
            const int start = -lr.x - 1, count = lr.y;
            for (int k = start; k < start + count; ++k) {
                const BvhTri* tr = b.tris + k;
                const double d2 = point_tri_d2(px, py, pz, tr->a, tr->e1, tr->e2);
                if (d2 < best) best = d2;
            }
        } else {
            const double dl = point_box_d2(b.nodes + lr.x, px, py, pz);
            const double dr = point_box_d2(b.nodes + lr.y, px, py, pz);
            if (dl < dr) {  // nearer child popped first
                stack[sp++] = lr.y;
                stack[sp++] = lr.x;
            } else {
                stack[sp++] = lr.x;
                stack[sp++] = lr.y;
            }
        }
    }
    out[q] = sqrt(best);
}

struct VisParams {
    double lx, ly, lz, t1x, t1y, t1z, t2x, t2y, t2z, tan_r;
    int spp, width, height;
    uint64_t seed;
};

__global__ void __launch_bounds__(128) reference_visibility_kernel(
    BvhView b, const double* __restrict__ pos, const double* __restrict__ nrm,
    const uint8_t* __restrict__ cov, VisParams V, double* __restrict__ out) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)V.width * V.height) return;
    if (!cov[p]) {
        out[p] = 1.0;
        return;
    }
    const double ox = pos[3 * p] + 1e-4 * nrm[3 * p];
    const double oy = pos[3 * p + 1] + 1e-4 * nrm[3 * p + 1];
    const double oz = pos[3 * p + 2] + 1e-4 * nrm[3 * p + 2];
    const uint64_t key = stream_key(V.seed, (uint64_t)p, 1);
    int open = 0;
    for (int s = 0; s < V.spp; ++s) {
        const double u = uniform01(key, 2 * (uint64_t)s);
        const double v = uniform01(key, 2 * (uint64_t)s + 1);
        const double r = V.tan_r * sqrt(u);
        const double phi = 6.283185307179586 * v;  // 2.0 * math.pi folded exactly
        const double sn = gs::glibc_sin(phi), c = gs::glibc_cos(phi);  // render.py's math.cos/sin
        const double dx = V.lx + r * (c * V.t1x + sn * V.t2x);
        const double dy = V.ly + r * (c * V.t1y + sn * V.t2y);
        const double dz = V.lz + r * (c * V.t1z + sn * V.t2z);
        const double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
        int32_t tid;
        int facing;
        bvh_ray(b, ox, oy, oz, dx * inv, dy * inv, dz * inv, __longlong_as_double(0x7ff0000000000000ll),
                tid, facing);
        open += tid < 0;
    }
    out[p] = (double)open / V.spp;
}

__global__ void unit_sphere_dirs_kernel(const uint64_t* __restrict__ keys, int64_t n, int x,
                                        double* __restrict__ dirs) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n * x) return;
    const int64_t t = q / x;
    unit_sphere_dir(keys[t], (uint64_t)(q - t * x), dirs[3 * q], dirs[3 * q + 1], dirs[3 * q + 2]);
}

__global__ void glibc_sincos_kernel(const double* __restrict__ xs, int64_t n, double* __restrict__ s,
                                    double* __restrict__ c) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double x = xs[q];
    s[q] = gs::glibc_sin(x);
    c[q] = gs::glibc_cos(x);
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" int rtsdf_unit_sphere_dirs(const uint64_t* keys, int64_t n, int x, double* dirs,
                                      void* stream) {
    if (n < 0 || x < 0 || (n * x > 0 && (!keys || !dirs))) {
        set_error("unit_sphere_dirs: bad arguments");
        return RTSDF_ERR_INVALID;
    }
    if (n * x == 0) return RTSDF_OK;
    unit_sphere_dirs_kernel<<<(unsigned)((n * x + 127) / 128), 128, 0, (cudaStream_t)stream>>>(keys, n,
                                                                                              x, dirs);
    count_launch();
    return check_launch("unit_sphere_dirs");
}

extern "C" int rtsdf_glibc_sincos(const double* x, int64_t n, double* s, double* c, void* stream) {
    if (n < 0 || (n > 0 && (!x || !s || !c))) {
        set_error("glibc_sincos: bad arguments");
        return RTSDF_ERR_INVALID;
    }
    if (n == 0) return RTSDF_OK;
    glibc_sincos_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(x, n, s, c);
    count_launch();
    return check_launch("glibc_sincos");
}

extern "C" int rtsdf_exact_distance(const void* bvh_packed, int64_t n_nodes, const double* points,
                                    int64_t n, double* out, void* stream) {
    if (!bvh_packed || n_nodes < 1 || n < 0) {
        set_error("exact_distance: bad arguments");
        return RTSDF_ERR_INVALID;
    }
    if (n == 0) return RTSDF_OK;
    exact_distance_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        bvh_view(bvh_packed, n_nodes), points, n, out);
    count_launch();
    return check_launch("exact_distance");
}

extern "C" int rtsdf_reference_visibility(const void* bvh_packed, int64_t n_nodes,
                                          const double* g_pos, const double* g_nrm,
                                          const uint8_t* g_cov, int height, int width,
                                          const double* light, const double* t1, const double* t2,
                                          double tan_r, int spp, uint64_t seed, double* out_vis,
                                          void* stream) {
    if (!bvh_packed || n_nodes < 1 || height < 0 || width < 0 || spp < 1) {
        set_error("reference_visibility: bad arguments (spp must be >= 1)");
        return RTSDF_ERR_INVALID;
    }
    const int64_t np_ = (int64_t)height * width;
    if (np_ == 0) return RTSDF_OK;
    VisParams V{light[0], light[1], light[2], t1[0], t1[1], t1[2], t2[0], t2[1], t2[2],
                tan_r,    spp,      width,    height, seed};
    reference_visibility_kernel<<<(unsigned)((np_ + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        bvh_view(bvh_packed, n_nodes), g_pos, g_nrm, g_cov, V, out_vis);
    count_launch();
    return check_launch("reference_visibility");
}
