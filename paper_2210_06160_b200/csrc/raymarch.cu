// raymarch.cu -- K8: soft-shadow sphere tracing that consumes the fine field,
// plus the G-buffer primary-visibility kernel, compose, bias and point
// sampling.
//
// Restates raymarch.py:83-147 (_march / _shadow_one), render.py:75-152
// (_gbuffer_kernel / _occlusion_kernel), render.py:186-192 (compose),
// field.py:155-161 (apply_bias) and field.py:141-148 (_sample_many).  The march
// samples the f32 field with the reference's fp64 software trilinear: B200
// texture filtering uses 8-bit fixed-point weights and would not match.
#include "common.cuh"
#include "trace.cuh"

namespace rtsdf {

struct MarchArgs {
    double eps;
    int max_iter;
    double max_step;
    double t_max;
    double k;
};

// raymarch.py:83-115; returns status 0 hit / 1 exited / 2 max-iter
__device__ int march(const FieldView& f, double ox, double oy, double oz, double dx, double dy,
                     double dz, const MarchArgs& a, double t0, double& t_out, int& it_out,
                     double& min_term_out) {
    double t = t0, min_term = 1.0, prev_d = -1.0;
    int it = 0;
    while (it < a.max_iter) {
        double px = ox + t * dx, py = oy + t * dy, pz = oz + t * dz;
        double dist = trilinear(f, px, py, pz);
        it += 1;
        if (dist <= a.eps) {
            t_out = t;
            it_out = it;
            min_term_out = 0.0;
            return 0;
        }
        if (t > 0.0) {
            double term = a.k * dist / t;
            if (prev_d > 0.0 && dist < prev_d) {
                double y = dist * dist / (2.0 * prev_d);
                double den = dist * dist - y * y;
                double te = t - y;
                if (den > 0.0 && te > 0.0) term = a.k * sqrt(den) / te;
            }
            if (term < min_term) min_term = dmax_(term, 0.0);
        }
        prev_d = dist;
        double step = dist < a.max_step ? dist : a.max_step;
        t += step;
        if (t > a.t_max) {
            t_out = t;
            it_out = it;
            min_term_out = min_term;
            return 1;
        }
    }
    t_out = t;
    it_out = it;
    min_term_out = min_term;
    return 2;
}

__global__ void occlusion_kernel(FieldView f, const double* __restrict__ g_pos,
                                 const double* __restrict__ g_nrm, const uint8_t* __restrict__ g_cov,
                                 int height, int width, int row0, int nrows, double lx, double ly,
                                 double lz, MarchArgs a, double jitter, double offset, int draws,
                                 uint64_t seed, double* __restrict__ out) {
    // pixels of rows [row0, row0 + nrows) (a pixel-sharded band or the image)
    int64_t p = (int64_t)row0 * width + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)(row0 + nrows) * width || p >= (int64_t)height * width) return;
    if (!g_cov[p]) {
        out[p] = 0.0;
        return;
    }
    double ox = g_pos[3 * p] + offset * g_nrm[3 * p];
    double oy = g_pos[3 * p + 1] + offset * g_nrm[3 * p + 1];
    double oz = g_pos[3 * p + 2] + offset * g_nrm[3 * p + 2];
    uint64_t key = stream_key(seed, (uint64_t)p, 0);  // render.py:145: py * W + px
    double total = 0.0;
    for (int j = 0; j < draws; ++j) {
        double t0 = jitter * a.max_step * uniform01(key, (uint64_t)j);
        double t, mt;
        int it;
        int st = march(f, ox, oy, oz, lx, ly, lz, a, t0, t, it, mt);
        total += st == 0 ? 1.0 : 1.0 - mt;
    }
    out[p] = total / draws;
}

__global__ void sphere_trace_kernel(FieldView f, const double* __restrict__ orig,
                                    const double* __restrict__ dirs, int64_t n, MarchArgs a,
                                    const double* __restrict__ t0s, int32_t* __restrict__ status,
                                    double* __restrict__ t_out, int32_t* __restrict__ it_out,
                                    double* __restrict__ mt_out) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    double t, mt;
    int it;
    int st = march(f, orig[3 * q], orig[3 * q + 1], orig[3 * q + 2], dirs[3 * q], dirs[3 * q + 1],
                   dirs[3 * q + 2], a, t0s ? t0s[q] : 0.0, t, it, mt);
    status[q] = st;
    t_out[q] = t;
    it_out[q] = it;
    mt_out[q] = mt;
}

__global__ void trilinear_many_kernel(FieldView f, const double* __restrict__ pts, int64_t n,
                                      double* __restrict__ out) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    out[q] = trilinear(f, pts[3 * q], pts[3 * q + 1], pts[3 * q + 2]);
}

struct Cam {
    double pos[3], fwd[3], right[3], up[3];
};

// Primary rays through the K6 search tree (trace_fast): the same brute-force
// closest hit (t, min id) as _bvh_ray, so the same G-buffer; used when the
// view's tree was built on the device (dynamic scenes).
__global__ void __launch_bounds__(128) gbuffer_fast_kernel(FastBvh b, const double* __restrict__ normals_orig,
                                    const float* __restrict__ albedo_orig, Cam cam, double half_w,
                                    double half_h, int width, int height, double* __restrict__ out_pos,
                                    double* __restrict__ out_nrm, float* __restrict__ out_alb,
                                    uint8_t* __restrict__ out_cov) {
    __shared__ int32_t stack_mem[RTSDF_FAST_STACK * 128];
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)height * width) return;
    int py = (int)(p / width), px = (int)(p % width);
    double sy = 1.0 - 2.0 * ((double)py + 0.5) / height;
    double sx = 2.0 * ((double)px + 0.5) / width - 1.0;
    double dx = cam.fwd[0] + sx * half_w * cam.right[0] + sy * half_h * cam.up[0];
    double dy = cam.fwd[1] + sx * half_w * cam.right[1] + sy * half_h * cam.up[1];
    double dz = cam.fwd[2] + sx * half_w * cam.right[2] + sy * half_h * cam.up[2];
    double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    dx *= inv;
    dy *= inv;
    dz *= inv;
    int32_t tid;
    int facing;
    double t = trace_fast(b, cam.pos[0], cam.pos[1], cam.pos[2], dx, dy, dz,
                          __longlong_as_double(0x7ff0000000000000ll), stack_mem + threadIdx.x, 128,
                          tid, facing);
    if (tid < 0) {
        out_cov[p] = 0;
        return;
    }
    out_cov[p] = 1;
    out_pos[3 * p] = cam.pos[0] + t * dx;
    out_pos[3 * p + 1] = cam.pos[1] + t * dy;
    out_pos[3 * p + 2] = cam.pos[2] + t * dz;
    for (int c = 0; c < 3; ++c) {
        out_nrm[3 * p + c] = normals_orig[3 * (int64_t)tid + c];
        out_alb[3 * p + c] = albedo_orig[3 * (int64_t)tid + c];
    }
}

__global__ void gbuffer_kernel(BvhView b, const double* __restrict__ normals_orig,
                               const float* __restrict__ albedo_orig, Cam cam, double half_w,
                               double half_h, int width, int height, double* __restrict__ out_pos,
                               double* __restrict__ out_nrm, float* __restrict__ out_alb,
                               uint8_t* __restrict__ out_cov) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= (int64_t)height * width) return;
    int py = (int)(p / width), px = (int)(p % width);
    double sy = 1.0 - 2.0 * ((double)py + 0.5) / height;
    double sx = 2.0 * ((double)px + 0.5) / width - 1.0;
    double dx = cam.fwd[0] + sx * half_w * cam.right[0] + sy * half_h * cam.up[0];
    double dy = cam.fwd[1] + sx * half_w * cam.right[1] + sy * half_h * cam.up[1];
    double dz = cam.fwd[2] + sx * half_w * cam.right[2] + sy * half_h * cam.up[2];
    double inv = 1.0 / sqrt(dx * dx + dy * dy + dz * dz);
    dx *= inv;
    dy *= inv;
    dz *= inv;
    int32_t tid;
    int facing;
    double t = bvh_ray(b, cam.pos[0], cam.pos[1], cam.pos[2], dx, dy, dz,
                       __longlong_as_double(0x7ff0000000000000ll), tid, facing);
    if (tid < 0) {  // render.py:97-98; other channels keep their zero init
        out_cov[p] = 0;
        return;
    }
    out_cov[p] = 1;
    out_pos[3 * p] = cam.pos[0] + t * dx;
    out_pos[3 * p + 1] = cam.pos[1] + t * dy;
    out_pos[3 * p + 2] = cam.pos[2] + t * dz;
    for (int c = 0; c < 3; ++c) {
        out_nrm[3 * p + c] = normals_orig[3 * (int64_t)tid + c];
        out_alb[3 * p + c] = albedo_orig[3 * (int64_t)tid + c];
    }
}

// render.py:186-192: lambert = clip(n . l, 0); img = albedo * lambert * (1 - occ)
__global__ void compose_kernel(const double* __restrict__ g_nrm, const float* __restrict__ g_alb,
                               const uint8_t* __restrict__ g_cov, const double* __restrict__ occ,
                               int64_t n, double lx, double ly, double lz, double b0, double b1,
                               double b2, float* __restrict__ out) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (!g_cov[p]) {
        out[3 * p] = (float)b0;
        out[3 * p + 1] = (float)b1;
        out[3 * p + 2] = (float)b2;
        return;
    }
    double lam = g_nrm[3 * p] * lx + g_nrm[3 * p + 1] * ly + g_nrm[3 * p + 2] * lz;
    lam = lam < 0.0 ? 0.0 : lam;
    double s = lam * (1.0 - occ[p]);
    for (int c = 0; c < 3; ++c) out[3 * p + c] = (float)((double)g_alb[3 * p + c] * s);
}

__global__ void apply_bias_kernel(const float* __restrict__ in, int64_t n, float bias,
                                  float* __restrict__ out) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n) out[q] = __fsub_rn(in[q], bias);
}

static inline FieldView fview(const float* field, int nx, int ny, int nz, const double* lo,
                              const double* h, float bias = 0.0f) {
    return FieldView{field, nx, ny, nz, lo[0], lo[1], lo[2], h[0], h[1], h[2], bias};
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" int rtsdf_occlusion(const float* field, int nx, int ny, int nz, const double* lo,
                               const double* h, const double* g_pos, const double* g_nrm,
                               const uint8_t* g_cov, int height, int width, int row0, int nrows,
                               const double* light, double eps, int max_iter, double max_step,
                               double t_max, double k, double jitter, double offset, int draws,
                               uint64_t seed, float sample_bias, double* out, void* stream) {
    if (draws < 1 || max_iter < 1 || row0 < 0 || nrows < 0 || row0 + nrows > height) {
        set_error("occlusion: draws and max_iter must be >= 1, rows inside the image");
        return RTSDF_ERR_INVALID;
    }
    int64_t n = (int64_t)nrows * width;
    if (n <= 0) return RTSDF_OK;
    MarchArgs a{eps, max_iter, max_step, t_max, k};
    occlusion_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        fview(field, nx, ny, nz, lo, h, sample_bias), g_pos, g_nrm, g_cov, height, width, row0, nrows,
        light[0], light[1], light[2], a, jitter, offset, draws, seed, out);
    count_launch();
    return check_launch("occlusion");
}

extern "C" int rtsdf_sphere_trace(const float* field, int nx, int ny, int nz, const double* lo,
                                  const double* h, const double* origins, const double* dirs,
                                  int64_t n, double eps, int max_iter, double max_step,
                                  double t_max, const double* t0, double k, int32_t* status,
                                  double* t, int32_t* iters, double* min_term, void* stream) {
    if (n <= 0) return RTSDF_OK;
    MarchArgs a{eps, max_iter, max_step, t_max, k};
    sphere_trace_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        fview(field, nx, ny, nz, lo, h), origins, dirs, n, a, t0, status, t, iters, min_term);
    count_launch();
    return check_launch("sphere_trace");
}

extern "C" int rtsdf_trilinear_many(const float* field, int nx, int ny, int nz, const double* lo,
                                    const double* h, const double* pts, int64_t n, double* out,
                                    void* stream) {
    if (n <= 0) return RTSDF_OK;
    trilinear_many_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        fview(field, nx, ny, nz, lo, h), pts, n, out);
    count_launch();
    return check_launch("trilinear_many");
}

extern "C" int rtsdf_gbuffer(const void* bvh_packed, int64_t n_nodes, int64_t n_tris, int fast,
                             const double* normals_orig,
                             const float* albedo_orig, const double* cam, double half_w,
                             double half_h, int width, int height, double* out_pos,
                             double* out_nrm, float* out_alb, uint8_t* out_cov, void* stream) {
    int64_t n = (int64_t)height * width;
    if (n <= 0) return RTSDF_OK;
    Cam c;
    for (int a = 0; a < 3; ++a) {
        c.pos[a] = cam[a];
        c.fwd[a] = cam[3 + a];
        c.right[a] = cam[6 + a];
        c.up[a] = cam[9 + a];
    }
    if (fast)
        gbuffer_fast_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            fast_bvh_view(bvh_packed, n_nodes, n_tris), normals_orig, albedo_orig, c, half_w,
            half_h, width, height, out_pos, out_nrm, out_alb, out_cov);
    else
        gbuffer_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            bvh_view(bvh_packed, n_nodes), normals_orig, albedo_orig, c, half_w, half_h, width,
            height, out_pos, out_nrm, out_alb, out_cov);
    count_launch();
    return check_launch("gbuffer");
}

extern "C" int rtsdf_compose(const double* g_nrm, const float* g_alb, const uint8_t* g_cov,
                             const double* occ, int height, int width, const double* light,
                             const double* background, float* out_rgb, void* stream) {
    int64_t n = (int64_t)height * width;
    if (n <= 0) return RTSDF_OK;
    compose_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        g_nrm, g_alb, g_cov, occ, n, light[0], light[1], light[2], background[0], background[1],
        background[2], out_rgb);
    count_launch();
    return check_launch("compose");
}

extern "C" int rtsdf_apply_bias(const float* data, int64_t n, float bias, float* out,
                                void* stream) {
    if (n <= 0) return RTSDF_OK;
    apply_bias_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(data, n, bias,
                                                                                    out);
    count_launch();
    return check_launch("apply_bias");
}
