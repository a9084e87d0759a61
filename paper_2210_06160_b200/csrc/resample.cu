// resample.cu -- K4: coarse -> fine trilinear resample, ray mask, band-exit
// reset, and the ordered masked-texel compaction.
//
// Restates raysample.py:91-119 (_coarse_at_fine_kernel / _resample_and_mask),
// raysample.py:288-295 (texels that left the band lose their state) and
// raysample.py:266 (np.flatnonzero).  One full-grid pass does all of the
// per-texel work (10 B/texel of HBM traffic at coarse == fine dims); the
// compaction re-reads only the 1 B mask.  Indices come out ascending, like
// flatnonzero, so the sampler's texel order (and a host direction table
// indexed by it) matches the reference.
#include "common.cuh"

#define RS_THREADS 256
#define RS_PER_THREAD 16
#define RS_CELLS_PER_BLOCK (RS_THREADS * RS_PER_THREAD)
#define RS_TAB_MAX 1365  // per-axis table entries: 3 axes x 12 B within the 48 KB default

namespace rtsdf {

struct RsParams {
    FieldView coarse;
    int fnx, fny, fnz;
    double fhx, fhy, fhz;
    double d;
    int64_t c0, n_cells;  // global cells [c0, c0 + n_cells); buffers global-indexed
    FastDiv div_ny, div_nz;
    int tab;  // per-axis weight table entries in dynamic shared memory (0: no tables)
};

// raysample.py:97-101: fine centres measured from the COARSE lo, then the
// trilinear axis weights (field.py:104-118) -- a function of one index only.
__device__ __forceinline__ AxisW fine_axis(double clo, double fh, double ch, int cn, int idx) {
    return axis_weight(clo + ((double)idx + 0.5) * fh, clo, ch, cn);
}

__device__ __forceinline__ void cell_ijk(const RsParams& P, uint32_t c, int& i, int& j, int& k) {
    const uint32_t q = fdiv(c, P.div_nz);
    k = (int)(c - q * P.div_nz.d);
    i = (int)fdiv(q, P.div_ny);
    j = (int)(q - (uint32_t)i * P.div_ny.d);
}

// Each block owns RS_CELLS_PER_BLOCK consecutive cells.  The axis weights of
// the planes / rows / columns the block touches are computed once into shared
// tables (3 fp64 divisions per table entry instead of per cell), so the cell
// loop is 8 gathers + 7 fp64 lerps; identical arithmetic, identical bits.
__global__ void __launch_bounds__(RS_THREADS) resample_mask_kernel(
    RsParams P, float* __restrict__ c_fine, float* __restrict__ out_unmasked,
    uint8_t* __restrict__ mask_new, int32_t* __restrict__ block_counts,
    const uint8_t* __restrict__ mask_old, float* __restrict__ run_min,
    int32_t* __restrict__ front, int32_t* __restrict__ back) {
    __shared__ int warp_sum[RS_THREADS / 32];
    extern __shared__ double rs_tab[];  // tf[3][P.tab] doubles, then ti[3][P.tab] ints
    const int T = P.tab;
    double* tfb = rs_tab;
    int* tib = (int*)(rs_tab + 3 * T);
    const int64_t base = P.c0 + (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    const int64_t last = min(base + RS_CELLS_PER_BLOCK, P.c0 + P.n_cells) - 1;
    int i0, j0, k0, i1, j1, k1;
    cell_ijk(P, (uint32_t)base, i0, j0, k0);
    cell_ijk(P, (uint32_t)last, i1, j1, k1);
    // index ranges touched by [base, last]
    const int xs = i0, xn = i1 - i0 + 1;
    const int ys = i0 == i1 ? j0 : 0, yn = i0 == i1 ? j1 - j0 + 1 : P.fny;
    const int zs = (i0 == i1 && j0 == j1) ? k0 : 0, zn = (i0 == i1 && j0 == j1) ? k1 - k0 + 1 : P.fnz;
    const bool tab = xn <= T && yn <= T && zn <= T;  // host: T >= fny, fnz when T > 0
    if (tab) {
        const FieldView& f = P.coarse;
        for (int t = threadIdx.x; t < xn + yn + zn; t += RS_THREADS) {
            AxisW w;
            int ax, e;
            if (t < xn) {
                ax = 0, e = t;
                w = fine_axis(f.lox, P.fhx, f.hx, f.nx, xs + e);
            } else if (t < xn + yn) {
                ax = 1, e = t - xn;
                w = fine_axis(f.loy, P.fhy, f.hy, f.ny, ys + e);
            } else {
                ax = 2, e = t - xn - yn;
                w = fine_axis(f.loz, P.fhz, f.hz, f.nz, zs + e);
            }
            tfb[ax * T + e] = w.f;
            tib[ax * T + e] = w.i;
        }
        __syncthreads();
    }
    int cnt = 0;
#pragma unroll 2
    for (int r = 0; r < RS_PER_THREAD; ++r) {
        const int64_t c = base + r * RS_THREADS + threadIdx.x;
        if (c > last) break;
        int i, j, k;
        cell_ijk(P, (uint32_t)c, i, j, k);
        AxisW wx, wy, wz;
        if (tab) {
            wx.i = tib[i - xs], wx.f = tfb[i - xs];
            wy.i = tib[T + j - ys], wy.f = tfb[T + j - ys];
            wz.i = tib[2 * T + k - zs], wz.f = tfb[2 * T + k - zs];
            wx.j = P.coarse.nx > 1 ? wx.i + 1 : wx.i;
            wy.j = P.coarse.ny > 1 ? wy.i + 1 : wy.i;
            wz.j = P.coarse.nz > 1 ? wz.i + 1 : wz.i;
        } else {
            wx = fine_axis(P.coarse.lox, P.fhx, P.coarse.hx, P.coarse.nx, i);
            wy = fine_axis(P.coarse.loy, P.fhy, P.coarse.hy, P.coarse.ny, j);
            wz = fine_axis(P.coarse.loz, P.fhz, P.coarse.hz, P.coarse.nz, k);
        }
        const double v = trilinear_w(P.coarse, wx, wy, wz);
        bool m = v <= P.d;  // compared in fp64 (raysample.py:105)
        float vf = (float)v;
        if (c_fine) c_fine[c] = vf;
        if (out_unmasked && !m) out_unmasked[c] = vf;
        if (mask_new) mask_new[c] = m;
        if (mask_old && !m && mask_old[c]) {  // left the band: stale state resets
            run_min[c] = __int_as_float(0x7f800000);
            front[c] = 0;
            back[c] = 0;
        }
        cnt += m;
    }
    if (block_counts) {
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int w = 0; w < RS_THREADS / 32; ++w) s += warp_sum[w];
            block_counts[blockIdx.x] = s;
        }
    }
}

// Same partition and arithmetic as resample_mask_kernel, for grids whose z
// extent is a multiple of 4: a thread owns 4 groups of 4 consecutive cells of
// one row, so the cell decode, the x / y weights and the four corner-row
// offsets are computed once per group, and c_fine / mask_new / mask_old move
// as 16 / 4-byte vectors.
__global__ void __launch_bounds__(RS_THREADS) resample_mask4_kernel(
    RsParams P, float* __restrict__ c_fine, float* __restrict__ out_unmasked,
    uint8_t* __restrict__ mask_new, int32_t* __restrict__ block_counts,
    const uint8_t* __restrict__ mask_old, float* __restrict__ run_min,
    int32_t* __restrict__ front, int32_t* __restrict__ back) {
    __shared__ int warp_sum[RS_THREADS / 32];
    extern __shared__ double rs_tab[];  // tf[3][P.tab] doubles, then ti[3][P.tab] ints (host: tables fit)
    const int T = P.tab;
    double* tfb = rs_tab;
    int* tib = (int*)(rs_tab + 3 * T);
    const int64_t base = P.c0 + (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    const int64_t last = min(base + RS_CELLS_PER_BLOCK, P.c0 + P.n_cells) - 1;
    int i0, j0, k0, i1, j1, k1;
    cell_ijk(P, (uint32_t)base, i0, j0, k0);
    cell_ijk(P, (uint32_t)last, i1, j1, k1);
    const int xs = i0, xn = i1 - i0 + 1;
    const int ys = i0 == i1 ? j0 : 0, yn = i0 == i1 ? j1 - j0 + 1 : P.fny;
    const int zs = (i0 == i1 && j0 == j1) ? k0 : 0, zn = (i0 == i1 && j0 == j1) ? k1 - k0 + 1 : P.fnz;
    const FieldView& f = P.coarse;
    for (int t = threadIdx.x; t < xn + yn + zn; t += RS_THREADS) {  // host: xn, yn, zn <= T
        AxisW w;
        int ax, e;
        if (t < xn) {
            ax = 0, e = t;
            w = fine_axis(f.lox, P.fhx, f.hx, f.nx, xs + e);
        } else if (t < xn + yn) {
            ax = 1, e = t - xn;
            w = fine_axis(f.loy, P.fhy, f.hy, f.ny, ys + e);
        } else {
            ax = 2, e = t - xn - yn;
            w = fine_axis(f.loz, P.fhz, f.hz, f.nz, zs + e);
        }
        tfb[ax * T + e] = w.f;
        tib[ax * T + e] = w.i;
    }
    __syncthreads();
    const int64_t sx = (int64_t)f.ny * f.nz, sy = f.nz;
    const int dj = f.nx > 1 ? 1 : 0, djy = f.ny > 1 ? 1 : 0, djz = f.nz > 1 ? 1 : 0;
    int cnt = 0;
#pragma unroll 1
    for (int g = 0; g < RS_PER_THREAD / 4; ++g) {
        const int64_t c = base + ((int64_t)g * RS_THREADS + threadIdx.x) * 4;
        if (c > last) break;
        int i, j, k;
        cell_ijk(P, (uint32_t)c, i, j, k);
        const int xi = tib[i - xs], yi = tib[T + j - ys];
        const double fx = tfb[i - xs], fy = tfb[T + j - ys];
        const double ofx = __dsub_rn(1.0, fx), ofy = __dsub_rn(1.0, fy);
        const float* r00 = f.data + xi * sx + yi * sy;           // (x.i, y.i)
        const float* r10 = f.data + (xi + dj) * sx + yi * sy;    // (x.j, y.i)
        const float* r01 = f.data + xi * sx + (yi + djy) * sy;   // (x.i, y.j)
        const float* r11 = f.data + (xi + dj) * sx + (yi + djy) * sy;
        float4 vo;
        uint32_t mpack = 0;
        const uint32_t mold = mask_old ? *(const uint32_t*)(mask_old + c) : 0u;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int zi = tib[2 * T + k + e - zs], zj = zi + djz;
            const double fz = tfb[2 * T + k + e - zs], ofz = __dsub_rn(1.0, fz);
            // trilinear_w's arithmetic, term for term (field.py:95-128)
            const double c000 = __ldg(r00 + zi), c100 = __ldg(r10 + zi), c010 = __ldg(r01 + zi),
                         c110 = __ldg(r11 + zi), c001 = __ldg(r00 + zj), c101 = __ldg(r10 + zj),
                         c011 = __ldg(r01 + zj), c111 = __ldg(r11 + zj);
            const double c00 = __dadd_rn(__dmul_rn(c000, ofx), __dmul_rn(c100, fx));
            const double c10 = __dadd_rn(__dmul_rn(c010, ofx), __dmul_rn(c110, fx));
            const double c01 = __dadd_rn(__dmul_rn(c001, ofx), __dmul_rn(c101, fx));
            const double c11 = __dadd_rn(__dmul_rn(c011, ofx), __dmul_rn(c111, fx));
            const double c0 = __dadd_rn(__dmul_rn(c00, ofy), __dmul_rn(c10, fy));
            const double c1 = __dadd_rn(__dmul_rn(c01, ofy), __dmul_rn(c11, fy));
            const double v = __dadd_rn(__dmul_rn(c0, ofz), __dmul_rn(c1, fz));
            const bool m = v <= P.d;  // compared in fp64 (raysample.py:105)
            const float vf = (float)v;
            (&vo.x)[e] = vf;
            mpack |= (m ? 1u : 0u) << (8 * e);
            if (out_unmasked && !m) out_unmasked[c + e] = vf;
            if (!m && ((mold >> (8 * e)) & 0xffu)) {  // left the band: stale state resets
                run_min[c + e] = __int_as_float(0x7f800000);
                front[c + e] = 0;
                back[c + e] = 0;
            }
            cnt += m;
        }
        if (c_fine) *(float4*)(c_fine + c) = vo;
        if (mask_new) *(uint32_t*)(mask_new + c) = mpack;
    }
    if (block_counts) {
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int w = 0; w < RS_THREADS / 32; ++w) s += warp_sum[w];
            block_counts[blockIdx.x] = s;
        }
    }
}

__global__ void __launch_bounds__(RS_THREADS) count_mask_kernel(const uint8_t* __restrict__ mask,
                                                               int64_t c0, int64_t n,
                                                               int32_t* __restrict__ block_counts) {
    __shared__ int warp_sum[RS_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    int cnt = 0;
    for (int r = 0; r < RS_PER_THREAD; ++r) {
        int64_t c = base + r * RS_THREADS + threadIdx.x;
        if (c < n) cnt += mask[c0 + c] != 0;
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < RS_THREADS / 32; ++w) s += warp_sum[w];
        block_counts[blockIdx.x] = s;
    }
}

// Single-CTA exclusive scan of the per-block counts (n_blocks ~ 16 k at C3).
__global__ void __launch_bounds__(1024) scan_blocks_kernel(const int32_t* __restrict__ counts,
                                                          int64_t nb, int64_t* __restrict__ offsets,
                                                          int64_t* __restrict__ total) {
    __shared__ int64_t part[1024];
    const int64_t per = (nb + 1023) / 1024;
    const int64_t b0 = threadIdx.x * per;
    int64_t s = 0;
    for (int64_t b = b0; b < b0 + per && b < nb; ++b) s += counts[b];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        int64_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
    for (int64_t b = b0; b < b0 + per && b < nb; ++b) {
        offsets[b] = run;
        run += counts[b];
    }
    if (threadIdx.x == 1023) *total = part[1023];
}

// One thread owns RS_PER_THREAD (16) consecutive cells: the mask bytes (0/1)
// are read as one 16-byte vector where aligned, turned into a 16-bit set
// ((w & 0x01010101) * 0x01020408 >> 24 gathers the four byte flags of a word),
// one block-wide exclusive scan of the per-thread counts places them, and
// each thread writes its indices in ascending order -- the same block
// partition as the resample kernel's block_counts.
__global__ void __launch_bounds__(RS_THREADS) compact_kernel(const uint8_t* __restrict__ mask,
                                                            int64_t c0, int64_t n,
                                                            const int64_t* __restrict__ offsets,
                                                            int64_t* __restrict__ idx) {
    __shared__ int warp_tot[RS_THREADS / 32];
    __shared__ uint16_t pos[RS_CELLS_PER_BLOCK];  // block-local offsets of the masked cells
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t bbase = (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    const int64_t base = bbase + (int64_t)threadIdx.x * RS_PER_THREAD;
    const uint8_t* m = mask + c0 + base;
    uint32_t bits = 0;
    if (base + RS_PER_THREAD <= n && ((uintptr_t)m & 15) == 0) {
        const uint4 v = __ldg((const uint4*)m);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) bits |= (((w[q] & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << (4 * q);
    } else {
        for (int r = 0; r < RS_PER_THREAD; ++r)
            if (base + r < n && m[r] != 0) bits |= 1u << r;
    }
    const int cnt = __popc(bits);
    int incl = cnt;  // warp inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) {
        before += w < wid ? warp_tot[w] : 0;
        total += warp_tot[w];
    }
    // stage the ascending block-local offsets, then write the int64 indices
    // coalesced (one thread's run of up to 16 indices would otherwise be a
    // strided store per lane)
    int out = before + incl - cnt;
    while (bits) {
        const int r = __ffs(bits) - 1;
        pos[out++] = (uint16_t)(threadIdx.x * RS_PER_THREAD + r);
        bits &= bits - 1;
    }
    __syncthreads();
    int64_t* dst = idx + offsets[blockIdx.x];
    const int64_t first = c0 + bbase;
    for (int p = threadIdx.x; p < total; p += RS_THREADS) dst[p] = first + pos[p];
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" int64_t rtsdf_mask_blocks(int64_t n_cells) {
    return (n_cells + RS_CELLS_PER_BLOCK - 1) / RS_CELLS_PER_BLOCK;
}

extern "C" int rtsdf_resample_mask_range(const float* coarse, int cnx, int cny, int cnz,
                                         const double* clo, const double* ch, int fnx, int fny,
                                         int fnz, const double* fh, double d, int64_t c0,
                                         int64_t n_range, float* c_fine, float* out_unmasked,
                                         uint8_t* mask_new, int32_t* block_counts,
                                         const uint8_t* mask_old, float* run_min, int32_t* front,
                                         int32_t* back, void* stream) {
    if (cnx < 1 || cny < 1 || cnz < 1 || fnx < 1 || fny < 1 || fnz < 1) {
        set_error("resample_mask: bad dims");
        return RTSDF_ERR_INVALID;
    }
    const int64_t n_fine = (int64_t)fnx * fny * fnz;
    if (c0 < 0 || n_range < 0 || c0 + n_range > n_fine || n_fine >= ((int64_t)1 << 31)) {
        set_error("resample_mask: cell range [%lld, %lld) outside the fine grid", (long long)c0,
                  (long long)(c0 + n_range));
        return RTSDF_ERR_INVALID;
    }
    if (mask_old && (!run_min || !front || !back)) {
        set_error("resample_mask: mask_old needs run_min/front/back");
        return RTSDF_ERR_INVALID;
    }
    if (n_range == 0) return RTSDF_OK;
    RsParams P;
    P.coarse = FieldView{coarse, cnx, cny, cnz, clo[0], clo[1], clo[2], ch[0], ch[1], ch[2], 0.0f};
    P.fnx = fnx;
    P.fny = fny;
    P.fnz = fnz;
    P.fhx = fh[0];
    P.fhy = fh[1];
    P.fhz = fh[2];
    P.d = d;
    P.c0 = c0;
    P.n_cells = n_range;
    P.div_ny = make_fastdiv((uint32_t)fny);
    P.div_nz = make_fastdiv((uint32_t)fnz);
    int64_t nb = rtsdf_mask_blocks(n_range);
    // per-axis weight tables sized for the planes / rows / columns one block of
    // RS_CELLS_PER_BLOCK consecutive cells can touch (C3: 400 entries, 14 KB
    // of shared memory instead of a fixed 36 KB -- more L1 for the gathers)
    const int64_t planes = RS_CELLS_PER_BLOCK / ((int64_t)fny * fnz) + 2;  // >= planes a block spans
    int64_t T = fnz > fny ? fnz : fny;
    const int64_t xmax = planes < fnx ? planes : fnx;
    if (xmax > T) T = xmax;
    P.tab = T <= RS_TAB_MAX ? (int)T : 0;
    const size_t smem = (size_t)P.tab * 3 * (sizeof(double) + sizeof(int));
    // vector form: rows split into whole 4-cell groups, 16 / 4-byte aligned
    // buffers, weight tables for every block
    auto al = [](const void* q, uintptr_t a) { return ((uintptr_t)q & (a - 1)) == 0; };
    const bool vec = P.tab > 0 && fnz % 4 == 0 && c0 % 4 == 0 && n_range % 4 == 0 &&
                     al(c_fine, 16) && al(mask_new, 4) && al(mask_old, 4);
    if (vec)
        resample_mask4_kernel<<<(unsigned)nb, RS_THREADS, smem, (cudaStream_t)stream>>>(
            P, c_fine, out_unmasked, mask_new, block_counts, mask_old, run_min, front, back);
    else
        resample_mask_kernel<<<(unsigned)nb, RS_THREADS, smem, (cudaStream_t)stream>>>(
            P, c_fine, out_unmasked, mask_new, block_counts, mask_old, run_min, front, back);
    count_launch();
    return check_launch("resample_mask");
}

extern "C" int rtsdf_resample_mask(const float* coarse, int cnx, int cny, int cnz,
                                   const double* clo, const double* ch, int fnx, int fny, int fnz,
                                   const double* fh, double d, float* c_fine, float* out_unmasked,
                                   uint8_t* mask_new, int32_t* block_counts,
                                   const uint8_t* mask_old, float* run_min, int32_t* front,
                                   int32_t* back, void* stream) {
    return rtsdf_resample_mask_range(coarse, cnx, cny, cnz, clo, ch, fnx, fny, fnz, fh, d, 0,
                                     (int64_t)fnx * fny * fnz, c_fine, out_unmasked, mask_new,
                                     block_counts, mask_old, run_min, front, back, stream);
}

extern "C" size_t rtsdf_compact_ws_bytes(int64_t n_cells) {
    int64_t nb = rtsdf_mask_blocks(n_cells);
    return (size_t)nb * (sizeof(int64_t) + sizeof(int32_t)) + 256;
}

extern "C" int rtsdf_compact_mask_range(const uint8_t* mask, int64_t c0, int64_t n,
                                        int32_t* block_counts, int64_t* idx, int64_t* count,
                                        void* ws, size_t ws_bytes, void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    int64_t nb = rtsdf_mask_blocks(n);
    if (ws_bytes < rtsdf_compact_ws_bytes(n)) {
        set_error("compact_mask: workspace too small");
        return RTSDF_ERR_WORKSPACE;
    }
    if (n <= 0) {
        cudaMemsetAsync(count, 0, sizeof(int64_t), stream);
        return check_launch("compact_mask");
    }
    int64_t* offsets = (int64_t*)ws;
    if (!block_counts) {
        block_counts = (int32_t*)((char*)ws + nb * sizeof(int64_t));
        count_mask_kernel<<<(unsigned)nb, RS_THREADS, 0, stream>>>(mask, c0, n, block_counts);
        count_launch();
    }
    scan_blocks_kernel<<<1, 1024, 0, stream>>>(block_counts, nb, offsets, count);
    compact_kernel<<<(unsigned)nb, RS_THREADS, 0, stream>>>(mask, c0, n, offsets, idx);
    count_launch(2);
    return check_launch("compact_mask");
}

extern "C" int rtsdf_compact_mask(const uint8_t* mask, int64_t n, int32_t* block_counts,
                                  int64_t* idx, int64_t* count, void* ws, size_t ws_bytes,
                                  void* stream_) {
    return rtsdf_compact_mask_range(mask, 0, n, block_counts, idx, count, ws, ws_bytes, stream_);
}
