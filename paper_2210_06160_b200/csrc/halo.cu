// halo.cu -- compressed JFA halo planes for the z-slab sharded schedule.
//
// The early passes' inputs are almost all EMPTY (k >= 64 at C3: 97.8-99.5 %,
// SURVEY §8(e)); sending their halo planes raw dominates the NVLink volume
// (C5 on 8 GPUs: up to 3.5 GiB inbound per rank).  A plane range is sent as
// (1) a bitmap of its 32-cell segments that hold any seed and (2) those
// segments packed in order; the receiver expands it into the halo buffer,
// EMPTY elsewhere.  Exact by construction (every non-EMPTY value travels).
//
//   compress:   warp per bitmap word (32 segments): ballot of non-empty
//               segments -> word + popcount; exclusive scan of the popcounts
//               (cub); pack the marked segments; total count on the device
//   decompress: the same popcount scan over the received bitmap, then a warp
//               per word copies or EMPTY-fills its 32 segments
#include <cub/cub.cuh>

#include "common.cuh"

namespace rtsdf {

#define HALO_SEG 32

__device__ __forceinline__ bool seg_nonempty(const int32_t* __restrict__ src, int64_t n_el,
                                             int64_t seg) {
    const int64_t a = seg * HALO_SEG;
    bool any = false;
    if (a + HALO_SEG <= n_el && (((uintptr_t)(src + a)) & 15) == 0) {
        const int4* v = (const int4*)(src + a);
#pragma unroll
        for (int q = 0; q < HALO_SEG / 4; ++q) {
            const int4 x = __ldg(v + q);
            any |= (x.x & x.y & x.z & x.w) != RTSDF_EMPTY;
        }
    } else {
        for (int64_t e = a; e < a + HALO_SEG && e < n_el; ++e) any |= __ldg(src + e) != RTSDF_EMPTY;
    }
    return any;
}

__global__ void halo_mark_kernel(const int32_t* __restrict__ src, int64_t n_el, int64_t nw,
                                 uint32_t* __restrict__ bits, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nw) return;
    const int64_t nseg = (n_el + HALO_SEG - 1) / HALO_SEG;
    const int64_t seg = w * 32 + lane;
    const bool on = seg < nseg && seg_nonempty(src, n_el, seg);
    const unsigned m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) {
        if (bits) bits[w] = m;
        counts[w] = __popc(m);
    }
}

__global__ void halo_popc_kernel(const uint32_t* __restrict__ bits, int64_t nw,
                                 int32_t* __restrict__ counts) {
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w < nw) counts[w] = __popc(bits[w]);
}

// warp per word: lane l copies (pack) / expands (unpack) segment 32 w + l
template <bool PACK>
__global__ void halo_move_kernel(int32_t* __restrict__ plane_buf, const uint32_t* __restrict__ bits,
                                 const int32_t* __restrict__ offsets, int32_t* __restrict__ payload,
                                 int64_t n_el, int64_t nw, const int32_t* __restrict__ counts,
                                 int64_t* __restrict__ total) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nw) return;
    const uint32_t m = bits[w];
    if (PACK && total && w == nw - 1 && lane == 0) *total = (int64_t)offsets[w] + counts[w];
    // each segment moved by the whole warp, lane = element (coalesced)
    for (int l = 0; l < 32; ++l) {
        const int64_t seg = w * 32 + l;
        const int64_t e = seg * HALO_SEG + lane;
        if (seg * HALO_SEG >= n_el) break;
        const bool on = (m >> l) & 1u;
        const int64_t slot = (int64_t)(offsets[w] + __popc(m & ((1u << l) - 1u))) * HALO_SEG + lane;
        if (PACK) {
            if (on && e < n_el) payload[slot] = plane_buf[e];
        } else if (e < n_el) {
            plane_buf[e] = on ? payload[slot] : RTSDF_EMPTY;
        }
    }
}

static int64_t halo_words(int64_t n_el) { return ((n_el + HALO_SEG - 1) / HALO_SEG + 31) / 32; }

static size_t halo_scan_bytes(int64_t nw) {
    size_t t = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t, (const int32_t*)nullptr, (int32_t*)nullptr, (int)nw);
    return t;
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" int64_t rtsdf_halo_bitmap_words(int64_t n_el) { return n_el > 0 ? halo_words(n_el) : 0; }

extern "C" size_t rtsdf_halo_ws_bytes(int64_t n_el) {
    const int64_t nw = n_el > 0 ? halo_words(n_el) : 1;
    return (size_t)(2 * ((nw * sizeof(int32_t) + 255) / 256 * 256)) + halo_scan_bytes(nw) + 256;
}

extern "C" int rtsdf_halo_compress(const int32_t* src, int64_t n_el, uint32_t* bits, int32_t* payload,
                                   int64_t* total, void* ws, size_t ws_bytes, void* stream) {
    if (n_el <= 0) return RTSDF_OK;
    if (!src || !bits || !payload || !total || !ws || ws_bytes < rtsdf_halo_ws_bytes(n_el)) {
        set_error("halo_compress: bad arguments or workspace");
        return RTSDF_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nw = halo_words(n_el);
    int32_t* counts = (int32_t*)ws;
    int32_t* offsets = counts + (nw * sizeof(int32_t) + 255) / 256 * 256 / sizeof(int32_t);
    void* tmp = offsets + (nw * sizeof(int32_t) + 255) / 256 * 256 / sizeof(int32_t);
    size_t tb = halo_scan_bytes(nw);
    const unsigned g = (unsigned)((nw * 32 + 127) / 128);
    halo_mark_kernel<<<g, 128, 0, st>>>(src, n_el, nw, bits, counts);
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offsets, (int)nw, st);
    halo_move_kernel<true><<<g, 128, 0, st>>>(const_cast<int32_t*>(src), bits, offsets, payload, n_el,
                                              nw, counts, total);
    count_launch(3);
    return check_launch("halo_compress");
}

extern "C" int rtsdf_halo_decompress(const uint32_t* bits, const int32_t* payload, int64_t n_el,
                                     int32_t* dst, void* ws, size_t ws_bytes, void* stream) {
    if (n_el <= 0) return RTSDF_OK;
    if (!bits || !dst || !ws || ws_bytes < rtsdf_halo_ws_bytes(n_el)) {
        set_error("halo_decompress: bad arguments or workspace");
        return RTSDF_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nw = halo_words(n_el);
    int32_t* counts = (int32_t*)ws;
    int32_t* offsets = counts + (nw * sizeof(int32_t) + 255) / 256 * 256 / sizeof(int32_t);
    void* tmp = offsets + (nw * sizeof(int32_t) + 255) / 256 * 256 / sizeof(int32_t);
    size_t tb = halo_scan_bytes(nw);
    halo_popc_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(bits, nw, counts);
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offsets, (int)nw, st);
    halo_move_kernel<false><<<(unsigned)((nw * 32 + 127) / 128), 128, 0, st>>>(
        dst, bits, offsets, const_cast<int32_t*>(payload), n_el, nw, counts, nullptr);
    count_launch(3);
    return check_launch("halo_decompress");
}
