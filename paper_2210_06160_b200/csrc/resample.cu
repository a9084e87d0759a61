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
#define RS_PER_THREAD 8
#define RS_CELLS_PER_BLOCK (RS_THREADS * RS_PER_THREAD)

namespace rtsdf {

struct RsParams {
    FieldView coarse;
    int fnx, fny, fnz;
    double fhx, fhy, fhz;
    double d;
    int64_t n_cells;
};

__device__ __forceinline__ double resample_at(const RsParams& P, int64_t c) {
    const int64_t nyz = (int64_t)P.fny * P.fnz;
    int i = (int)(c / nyz);
    int64_t r = c - (int64_t)i * nyz;
    int j = (int)(r / P.fnz);
    int k = (int)(r - (int64_t)j * P.fnz);
    // raysample.py:97-101: fine centres measured from the COARSE lo
    double px = P.coarse.lox + ((double)i + 0.5) * P.fhx;
    double py = P.coarse.loy + ((double)j + 0.5) * P.fhy;
    double pz = P.coarse.loz + ((double)k + 0.5) * P.fhz;
    return trilinear(P.coarse, px, py, pz);
}

__global__ void __launch_bounds__(RS_THREADS) resample_mask_kernel(
    RsParams P, float* __restrict__ c_fine, float* __restrict__ out_unmasked,
    uint8_t* __restrict__ mask_new, int32_t* __restrict__ block_counts,
    const uint8_t* __restrict__ mask_old, float* __restrict__ run_min,
    int32_t* __restrict__ front, int32_t* __restrict__ back) {
    __shared__ int warp_sum[RS_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    int cnt = 0;
#pragma unroll 2
    for (int r = 0; r < RS_PER_THREAD; ++r) {
        int64_t c = base + r * RS_THREADS + threadIdx.x;
        if (c >= P.n_cells) break;
        double v = resample_at(P, c);
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

__global__ void __launch_bounds__(RS_THREADS) count_mask_kernel(const uint8_t* __restrict__ mask,
                                                               int64_t n, int32_t* __restrict__ block_counts) {
    __shared__ int warp_sum[RS_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    int cnt = 0;
    for (int r = 0; r < RS_PER_THREAD; ++r) {
        int64_t c = base + r * RS_THREADS + threadIdx.x;
        if (c < n) cnt += mask[c] != 0;
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

__global__ void __launch_bounds__(RS_THREADS) compact_kernel(const uint8_t* __restrict__ mask,
                                                            int64_t n,
                                                            const int64_t* __restrict__ offsets,
                                                            int64_t* __restrict__ idx) {
    __shared__ int warp_cnt[RS_THREADS / 32];
    const int64_t base = (int64_t)blockIdx.x * RS_CELLS_PER_BLOCK;
    int64_t run = offsets[blockIdx.x];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int r = 0; r < RS_PER_THREAD; ++r) {
        int64_t c = base + r * RS_THREADS + threadIdx.x;
        bool m = c < n && mask[c] != 0;
        unsigned bal = __ballot_sync(0xffffffffu, m);
        if (lane == 0) warp_cnt[wid] = __popc(bal);
        __syncthreads();
        int before = 0, all = 0;
        for (int w = 0; w < RS_THREADS / 32; ++w) {
            int v = warp_cnt[w];
            before += w < wid ? v : 0;
            all += v;
        }
        if (m) idx[run + before + __popc(bal & ((1u << lane) - 1))] = c;
        run += all;
        __syncthreads();
    }
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" int64_t rtsdf_mask_blocks(int64_t n_cells) {
    return (n_cells + RS_CELLS_PER_BLOCK - 1) / RS_CELLS_PER_BLOCK;
}

extern "C" int rtsdf_resample_mask(const float* coarse, int cnx, int cny, int cnz,
                                   const double* clo, const double* ch, int fnx, int fny, int fnz,
                                   const double* fh, double d, float* c_fine, float* out_unmasked,
                                   uint8_t* mask_new, int32_t* block_counts,
                                   const uint8_t* mask_old, float* run_min, int32_t* front,
                                   int32_t* back, void* stream) {
    if (cnx < 1 || cny < 1 || cnz < 1 || fnx < 1 || fny < 1 || fnz < 1) {
        set_error("resample_mask: bad dims");
        return RTSDF_ERR_INVALID;
    }
    if (mask_old && (!run_min || !front || !back)) {
        set_error("resample_mask: mask_old needs run_min/front/back");
        return RTSDF_ERR_INVALID;
    }
    RsParams P;
    P.coarse = FieldView{coarse, cnx, cny, cnz, clo[0], clo[1], clo[2], ch[0], ch[1], ch[2], 0.0f};
    P.fnx = fnx;
    P.fny = fny;
    P.fnz = fnz;
    P.fhx = fh[0];
    P.fhy = fh[1];
    P.fhz = fh[2];
    P.d = d;
    P.n_cells = (int64_t)fnx * fny * fnz;
    int64_t nb = rtsdf_mask_blocks(P.n_cells);
    resample_mask_kernel<<<(unsigned)nb, RS_THREADS, 0, (cudaStream_t)stream>>>(
        P, c_fine, out_unmasked, mask_new, block_counts, mask_old, run_min, front, back);
    count_launch();
    return check_launch("resample_mask");
}

extern "C" size_t rtsdf_compact_ws_bytes(int64_t n_cells) {
    int64_t nb = rtsdf_mask_blocks(n_cells);
    return (size_t)nb * (sizeof(int64_t) + sizeof(int32_t)) + 256;
}

extern "C" int rtsdf_compact_mask(const uint8_t* mask, int64_t n, int32_t* block_counts,
                                  int64_t* idx, int64_t* count, void* ws, size_t ws_bytes,
                                  void* stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    int64_t nb = rtsdf_mask_blocks(n);
    if (ws_bytes < rtsdf_compact_ws_bytes(n)) {
        set_error("compact_mask: workspace too small");
        return RTSDF_ERR_WORKSPACE;
    }
    int64_t* offsets = (int64_t*)ws;
    if (!block_counts) {
        block_counts = (int32_t*)((char*)ws + nb * sizeof(int64_t));
        count_mask_kernel<<<(unsigned)nb, RS_THREADS, 0, stream>>>(mask, n, block_counts);
        count_launch();
    }
    scan_blocks_kernel<<<1, 1024, 0, stream>>>(block_counts, nb, offsets, count);
    compact_kernel<<<(unsigned)nb, RS_THREADS, 0, stream>>>(mask, n, offsets, idx);
    count_launch(2);
    return check_launch("compact_mask");
}
