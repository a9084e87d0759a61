// raysample.cu -- K6 + K7: ray-sampled refinement fused with the Eq. 1
// combine/sign update.
//
// Restates raysample.py:132-176 (_sample_rays / _sample_masked_kernel),
// rng.py:30-53 and raysample.py:215-244 (_update_masked_kernel).  Default
// (wavefront) path: pass 1 traces every ray with a small BVH4 node budget and
// merges finished rays into per-texel accumulators; rays out of budget are
// queued, ordered by direction octant, and re-traced by pass 2; one thread
// per texel then applies the band reset + Eq. 1 + sign.  The accumulators
// combine with atomicMin on the fp64 bits of t (t >= 0: integer order is fp64
// order) and atomicAdd on packed vote counts: min and integer sums are exact
// and order-free, so the result does not depend on scheduling.  The
// warp-per-texel kernel (sample_update_kernel) owns each texel with one lane
// and uses no atomics; it serves texels beyond the wavefront workspace and
// runs without a workspace.
#include <cub/cub.cuh>

#include "common.cuh"
#include "trace.cuh"

namespace rtsdf {

struct SampleParams {
    FastBvh bvh;
    FastBvh4 bvh4;  // valid when n_nodes4 > 0
    const int64_t* idx;
    const int64_t* count;
    int64_t m_cap;
    int64_t n_begin;  // sample_update_kernel: first texel (the tail beyond the wavefront capacity)
    FieldView coarse;
    int fnx, fny, fnz;
    double fhx, fhy, fhz;
    int x;
    FastDiv div_x, div_ny, div_nz;  // wavefront ray-index decode
    uint64_t seed;
    int64_t frame;
    const int64_t* frame_dev;  // non-null: the frame number is read on the device (graph replays)
    double t_max;
    float tb;  // tmax_bound(t_max), computed once on the host
    const double* dirs;
    double* samp_min;
    int32_t* samp_front;
    int32_t* samp_back;
    const float* prev;
    const uint8_t* mask_old;
    float* run_min;
    int32_t* front;
    int32_t* back;
    double alpha;
    float* out;
};

#define SAMPLE_THREADS 128

__global__ void __launch_bounds__(SAMPLE_THREADS) sample_update_kernel(SampleParams P) {
    __shared__ int32_t stack_mem[RTSDF_FAST_STACK * SAMPLE_THREADS];
    int32_t* stack = stack_mem + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t M = min(*P.count, P.m_cap);
    const int x = P.x;
    const int tpw = x >= 32 || x == 0 ? 1 : 32 / x;  // texels per warp
    const int seg = x >= 32 || x == 0 ? 32 : x;      // lanes per texel
    const int rounds = x > 32 ? (x + 31) / 32 : 1;
    const int my_t = lane / seg, pos = lane - my_t * seg;
    const int64_t nyz = (int64_t)P.fny * P.fnz;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t wbase = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
         P.n_begin + wbase * tpw < M; wbase += warps) {
        const int64_t n = P.n_begin + wbase * tpw + my_t;
        const bool active = my_t < tpw && n < M;
        int64_t lin = active ? __ldg(P.idx + n) : 0;
        int i = (int)(lin / nyz), j = (int)((lin / P.fnz) % P.fny), k = (int)(lin % P.fnz);
        // raysample.py:167-169: texel centre from the coarse lo (same box)
        double px = P.coarse.lox + ((double)i + 0.5) * P.fhx;
        double py = P.coarse.loy + ((double)j + 0.5) * P.fhy;
        double pz = P.coarse.loz + ((double)k + 0.5) * P.fhz;
        uint64_t key = stream_key(P.seed, (uint64_t)lin,
                                  (uint64_t)(P.frame_dev ? *P.frame_dev : P.frame));
        double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        int fr = 0, bk = 0;
        for (int rd = 0; rd < rounds; ++rd) {
            int r = rd * 32 + pos;
            if (active && x > 0 && r < x && pos < seg) {
                double dx, dy, dz;
                if (P.dirs) {
                    const double* d = P.dirs + 3 * (n * x + r);
                    dx = d[0];
                    dy = d[1];
                    dz = d[2];
                } else {
                    unit_sphere_dir(key, (uint64_t)r, dx, dy, dz);
                }
                int32_t id;
                int facing;
                double t = trace_fast(P.bvh, px, py, pz, dx, dy, dz, P.t_max, stack,
                                      SAMPLE_THREADS, id, facing);
                if (id >= 0) {
                    if (t < best) best = t;
                    if (facing == 1) fr++;
                    else bk++;
                }
            }
        }
        // segmented tree reduction: position p combines p + o inside its texel
        for (int o = 16; o; o >>= 1) {
            double ob = __shfl_down_sync(0xffffffffu, best, o);
            int of = __shfl_down_sync(0xffffffffu, fr, o);
            int obk = __shfl_down_sync(0xffffffffu, bk, o);
            if (pos + o < seg && lane + o < 32) {
                best = ob < best ? ob : best;
                fr += of;
                bk += obk;
            }
        }
        if (!active || pos != 0) continue;
        if (P.samp_min) P.samp_min[n] = best;
        if (P.samp_front) P.samp_front[n] = fr;
        if (P.samp_back) P.samp_back[n] = bk;
        if (!P.prev) continue;
        // raysample.py:229-244
        float rm = P.run_min[lin];
        int32_t f = P.front[lin], b = P.back[lin];
        if (!P.mask_old[lin]) {
            rm = __int_as_float(0x7f800000);
            f = 0;
            b = 0;
        }
        double m = best;
        if (m < (double)rm) rm = (float)m;
        f += fr;
        b += bk;
        P.run_min[lin] = rm;
        P.front[lin] = f;
        P.back[lin] = b;
        double c = (double)(float)trilinear(P.coarse, px, py, pz);  // c_fine[i, j, k] (f32)
        double blend = P.alpha * fabs((double)P.prev[lin]) + (1.0 - P.alpha) * c;
        double mag = blend < m ? blend : m;
        P.out[lin] = b > f ? (float)(-mag) : (float)mag;
    }
}

// ----------------------------------------------------------------------------
// Wavefront sampler (default).  Most rays are short: in the C3 scene ~95 % of
// the masked texels hug the ground plane and their rays finish after 2-3 node
// visits, while the few rays heading into the sphere need ~13 levels -- in the
// warp-per-texel kernel every warp then waits for its longest lane (36 % SIMD
// efficiency).  Pass 1 traces every ray with a small node budget and writes
// the per-ray result; rays that run out of budget are appended to a queue
// (warp-aggregated) and pass 2 re-traces only those, densely packed.  A third
// kernel reduces each texel's x rays in ray order (one thread per texel) and
// applies the Eq. 1 update.  The queue order varies run to run but every ray's
// result is deterministic, and the per-texel reduction order is fixed.
#define WF_THREADS 128
#ifndef WF_MINB
#define WF_MINB 6  // resident blocks per SM the tracer kernels are compiled for
#endif
#define WF_BUDGET 4   // binary search tree: internal-node visits in pass 1
#ifndef WF_BUDGET4
#define WF_BUDGET4 2  // BVH4: root only (ground-plane leaves finish in pass 1); C3 pass 1 + 2:
#endif                // budget 2 5.16 ms, 3 5.31, 4 5.35, 6 5.80 (measured)
#ifndef WF_B2_PER_SM
#define WF_B2_PER_SM 12  // pass-2 blocks per SM (grid-stride over the long-ray queue)
#endif

// Per-texel accumulators instead of per-ray results: the closest hit t as its
// fp64 bit pattern (t >= 0, so unsigned integer order is fp64 order; ~0 = no
// hit) merged with atomicMin, and the front / back votes packed in one word
// (front | back << 16, x <= 65535) merged with atomicAdd.  min and integer sums
// are exact and order-free, so the result does not depend on which pass or lane
// delivers a ray -- deterministic without a per-ray buffer.
struct WfBuffers {
    unsigned long long* tkey;  // [m_cap]
    uint32_t* votes;           // [m_cap]
    int32_t* queue;            // [R] rays needing the full search
    int64_t* qcount;
    unsigned long long* qhead;  // pass 2: next queue chunk to claim
    const int64_t* texels;      // the masked-texel count (device): chunks of rays beyond
    int64_t m_cap;              // min(count, m_cap) * x were not written by this call's pass 1
    int x;
    bool aligned;              // x divides 32: a warp of pass 1 holds whole texels
    double4* tex;              // [m_cap] per texel: origin xyz + RNG stream key (bits)
    // Pass-2 order: the long rays sorted by (direction octant, ray id).  Pass 1
    // records, per chunk of 32 consecutive rays, the long-ray mask and the
    // three octant bit planes (ballots, no atomics); wf_oct_count / _scan /
    // _scatter turn them into the ordered queue.  Long rays of one octant from
    // neighbouring texels then share warps: measured 2.96 -> 2.59 ms for pass 2
    // at C3 (10.2 -> 11.7 active threads per instruction) vs the order in
    // which pass-1 warps happened to append.
    uint4* chunk;              // [R / 32] (long mask, octant x / y / z sign planes)
    int32_t* oct_blk;          // [n_oct_blocks * 8] per block octant counts
    int32_t* oct_pos;          // [n_oct_blocks * 8] their per-octant exclusive scan
    void* scan_tmp;            // cub temp storage
    size_t scan_tmp_bytes;
};

#define WF_OCT_THREADS 256  // chunks per block of the octant compaction

#define WF_NO_HIT 0xffffffffffffffffull

__device__ __forceinline__ void wf_commit(const WfBuffers& B, uint32_t n, double t, int facing) {
    atomicMin(&B.tkey[n], (unsigned long long)__double_as_longlong(t));
    atomicAdd(&B.votes[n], facing == 1 ? 1u : 0x10000u);
}

__global__ void wf_init_kernel(SampleParams P, WfBuffers B) {
    const int64_t M = min(*P.count, P.m_cap);
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
         n += (int64_t)gridDim.x * blockDim.x) {
        B.tkey[n] = WF_NO_HIT;
        B.votes[n] = 0;
    }
}

// Per-texel ray setup, once per texel instead of once per ray: the fine-cell
// centre (raysample.py:167-169) and the texel's SplitMix64 stream key
// (raysample.py:170, rng.py:30-35).
__global__ void __launch_bounds__(WF_THREADS) wf_setup_kernel(SampleParams P, WfBuffers B) {
    const int64_t M = min(*P.count, P.m_cap);
    const uint64_t frame = (uint64_t)(P.frame_dev ? *P.frame_dev : P.frame);
    for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < M;
         n += (int64_t)gridDim.x * blockDim.x) {
        // 32-bit index math: cells <= 1024^3
        const unsigned lin = (unsigned)__ldg(P.idx + n);
        const unsigned q = fdiv(lin, P.div_nz);
        const unsigned i = fdiv(q, P.div_ny);
        const int k = (int)(lin - q * P.div_nz.d), j = (int)(q - i * P.div_ny.d);
        double4 t;
        t.x = P.coarse.lox + ((double)i + 0.5) * P.fhx;
        t.y = P.coarse.loy + ((double)j + 0.5) * P.fhy;
        t.z = P.coarse.loz + ((double)k + 0.5) * P.fhz;
        t.w = __longlong_as_double((long long)stream_key(P.seed, (uint64_t)lin, frame));
        B.tex[n] = t;
    }
}

__device__ __forceinline__ void wf_ray(const SampleParams& P, const WfBuffers& B, int64_t r,
                                       double& ox, double& oy, double& oz, double& dx, double& dy,
                                       double& dz) {
    // rays < 2^31 (host-checked)
    const unsigned n = fdiv((unsigned)r, P.div_x);
    const int ray = (int)((unsigned)r - n * P.div_x.d);
    const double2* tp = (const double2*)(B.tex + n);
    const double2 a = __ldg(tp), b = __ldg(tp + 1);
    ox = a.x;
    oy = a.y;
    oz = b.x;
    if (P.dirs) {
        const double* d = P.dirs + 3 * r;  // dirs[(n * x + ray) * 3 + c]
        dx = d[0];
        dy = d[1];
        dz = d[2];
    } else {
        unit_sphere_dir((uint64_t)__double_as_longlong(b.y), (uint64_t)ray, dx, dy, dz);
    }
}

// Pass 1 on a BVH4 with budget 2 (root only), without trace_fast4's stack,
// pops and budget bookkeeping: the root's four child boxes, then its children
// in near-first order while within reach (entry <= the best hit so far): a
// leaf is tested, an inner child ends pass 1 for the ray (pass 2 traces it
// from the root) -- trace_fast4's order and outcome with node budget 2.  A box
// entry is a lower bound on every hit inside it, so the unreached children
// cannot hold a closer hit than the one found.
#ifndef WF1_SROOT
#define WF1_SROOT 1
#endif
#define WF1_ROOT_STRIDE 36  // floats per staged root copy: 144 B, the 8 copies on disjoint banks
__device__ __forceinline__ double wf_trace4_root(const SampleParams& P, double ox, double oy, double oz,
                                                 double dx, double dy, double dz, int32_t& out_id,
                                                 int& out_facing, bool* done, const float* sroot) {
    RayF r;
    r.ix = clamp_inv(dx);
    r.iy = clamp_inv(dy);
    r.iz = clamp_inv(dz);
    r.oix = (float)ox * r.ix;
    r.oiy = (float)oy * r.iy;
    r.oiz = (float)oz * r.iz;
    const float fdx = (float)dx, fdy = (float)dy, fdz = (float)dz;
    double best_t = P.t_max;
    int32_t best_id = -1;
    int best_facing = 0;
    float tb = P.tb;
    // the root's copy 0 (unswapped planes) with box_entry's min / max pairs: one
    // address for the whole warp (pass-1 rays mix all eight octants, and
    // per-lane octant copies measured 2.50 -> 2.72 ms in L1 wavefronts)
    float4 lx, ly, lz, hx, hy, hz;
    int4 ch;
    float t[4];
#if WF1_SROOT
    // the ray's octant copy of the root, staged in shared memory by the block
    // (the global copies would cost 8 L1 wavefronts per load: pass-1 warps mix
    // all octants): near planes in the lo slots, no pair min / max
    {
        const float* q = sroot + WF1_ROOT_STRIDE * ray_octant(r.ix, r.iy, r.iz);
        lx = *(const float4*)(q);
        ly = *(const float4*)(q + 4);
        lz = *(const float4*)(q + 8);
        hx = *(const float4*)(q + 12);
        hy = *(const float4*)(q + 16);
        hz = *(const float4*)(q + 20);
        ch = *(const int4*)(q + 24);
    }
    t[0] = box_entry_nf(lx.x, ly.x, lz.x, hx.x, hy.x, hz.x, r, tb);
    t[1] = box_entry_nf(lx.y, ly.y, lz.y, hx.y, hy.y, hz.y, r, tb);
    t[2] = box_entry_nf(lx.z, ly.z, lz.z, hx.z, hy.z, hz.z, r, tb);
    t[3] = box_entry_nf(lx.w, ly.w, lz.w, hx.w, hy.w, hz.w, r, tb);
#else
    (void)sroot;
    load_node4(P.bvh4.nodes, lx, ly, lz, hx, hy, hz, ch);
    t[0] = box_entry(lx.x, ly.x, lz.x, hx.x, hy.x, hz.x, r, tb);
    t[1] = box_entry(lx.y, ly.y, lz.y, hx.y, hy.y, hz.y, r, tb);
    t[2] = box_entry(lx.z, ly.z, lz.z, hx.z, hy.z, hz.z, r, tb);
    t[3] = box_entry(lx.w, ly.w, lz.w, hx.w, hy.w, hz.w, r, tb);
#endif
    const int32_t c[4] = {ch.x, ch.y, ch.z, ch.w};
    // near-first over the reachable children: an inner child first in line ends
    // pass 1 for this ray (pass 2 traces it from the root); a leaf is tested
    bool need = false;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        int qn = -1;
        float tn = RTSDF_FINF;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (t[q] < tn) {
                tn = t[q];
                qn = q;
            }
        if (qn < 0 || !(tn <= tb)) break;
        int32_t cn = c[0];
#pragma unroll
        for (int q = 1; q < 4; ++q) cn = qn == q ? c[q] : cn;
        if (cn >= 0) {
            need = true;
            break;
        }
        leaf_tris(P.bvh4.tris, P.bvh4.exact, cn, ox, oy, oz, dx, dy, dz, fdx, fdy, fdz, best_t, best_id,
                  best_facing, tb);
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = qn == q ? RTSDF_FINF : t[q];
    }
    *done = !need;
    out_id = best_id;
    out_facing = best_facing;
    return best_id < 0 ? -1.0 : best_t;
}

template <bool WIDE>
__device__ __forceinline__ double wf_trace(const SampleParams& P, double ox, double oy, double oz,
                                           double dx, double dy, double dz, int32_t* stack,
                                           __half* tstack, int32_t& id, int& facing, int budget,
                                           bool* done, const float* sroot = nullptr) {
#ifndef WF1_ROOT
#define WF1_ROOT 1
#endif
    if (WIDE && WF1_ROOT && budget == 2)
        return wf_trace4_root(P, ox, oy, oz, dx, dy, dz, id, facing, done, sroot);
    if (WIDE)
        return trace_fast4(P.bvh4, ox, oy, oz, dx, dy, dz, P.t_max, stack, tstack, WF_THREADS, id,
                           facing, P.tb, budget, done);
    return trace_fast(P.bvh, ox, oy, oz, dx, dy, dz, P.t_max, stack, WF_THREADS, id, facing,
                      budget, done);
}

// Pass 1's node budget bounds its stack: a binary-tree inner visit pushes <= 1
// entry, a BVH4 visit <= 3, and at most budget - 1 visits complete, so a small
// shared stack suffices (measured: no change at 6 / 7 / 8 resident blocks; a
// two-chunk form that generates both chunks' directions before tracing, for
// fp64 ILP, measured 2.55 -> 2.69 ms; loading the next grid-stride step's
// texel record one step ahead measured 2.47 -> 2.57 ms: 32 B of spills).
#define WF1_STACK (3 * (WF_BUDGET4 - 1) > WF_BUDGET - 1 ? 3 * (WF_BUDGET4 - 1) : WF_BUDGET - 1)
static_assert(WF1_STACK >= WF_BUDGET - 1 && WF1_STACK >= 3 * (WF_BUDGET4 - 1), "pass-1 stack");
template <bool WIDE>
#ifndef WF1_MINB
#define WF1_MINB WF_MINB  // pass-1 resident blocks per SM (7 / 8 spill: 2.33 -> 2.39 / 2.40 ms)
#endif
__global__ void __launch_bounds__(WF_THREADS, WF1_MINB) wf_pass1_kernel(SampleParams P, WfBuffers B, int budget) {
    __shared__ int32_t stack_mem[WF1_STACK * WF_THREADS];
    __shared__ __half tstack_mem[WIDE ? WF1_STACK * WF_THREADS : 1];
    __shared__ __align__(16) float sroot[WIDE && WF1_SROOT ? 8 * WF1_ROOT_STRIDE : 1];
    if (WIDE && WF1_SROOT) {  // the root's 8 octant records (boxes + child refs, 112 B each)
        for (int e = threadIdx.x; e < 8 * 28; e += blockDim.x)
            sroot[(e / 28) * WF1_ROOT_STRIDE + e % 28] = __ldg((const float*)(P.bvh4.nodes + e / 28) + e % 28);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int64_t R = min(*P.count, P.m_cap) * P.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); r0 < R; r0 += stride) {
        const int64_t r = r0 + lane;
        bool need = false;
        bool sx = false, sy = false, sz = false;  // direction octant of the ray
        unsigned long long key = WF_NO_HIT;
        uint32_t inc = 0;
        uint32_t n = 0xffffffffu;
        if (r < R) {
            double ox, oy, oz, dx, dy, dz;
            wf_ray(P, B, r, ox, oy, oz, dx, dy, dz);
            sx = dx < 0.0;
            sy = dy < 0.0;
            sz = dz < 0.0;
            n = fdiv((unsigned)r, P.div_x);
            int32_t id;
            int facing;
            bool done;
            double t = wf_trace<WIDE>(P, ox, oy, oz, dx, dy, dz, stack_mem + threadIdx.x,
                                      tstack_mem + threadIdx.x, id, facing, budget, &done, sroot);
            if (done && id >= 0) {
                key = (unsigned long long)__double_as_longlong(t);
                inc = facing == 1 ? 1u : 0x10000u;
            }
            need = !done;
        }
        // merge the finished rays per texel (lanes of one texel are a contiguous
        // run of consecutive ray ids)
        if (P.x == 32) {
            // one texel per warp: 64-bit min as two 32-bit warp reductions
            const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
            const uint32_t hmin = __reduce_min_sync(0xffffffffu, hi);
            const uint32_t lmin = __reduce_min_sync(0xffffffffu, hi == hmin ? lo : 0xffffffffu);
            const uint32_t isum = __reduce_add_sync(0xffffffffu, inc);
            if (lane == 0 && n != 0xffffffffu) {  // plain stores initialise the texel
                B.tkey[n] = ((unsigned long long)hmin << 32) | lmin;
                B.votes[n] = isum;
            }
        } else if (B.aligned) {
            // x | 32: aligned groups of x lanes, butterfly within the group
            for (int off = P.x >> 1; off; off >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, off);
                key = ok < key ? ok : key;
                inc += __shfl_xor_sync(0xffffffffu, inc, off);
            }
            if (n != 0xffffffffu && (lane & (P.x - 1)) == 0) {
                B.tkey[n] = key;
                B.votes[n] = inc;
            }
        } else {
            // general x: shuffle-down min / sum clipped to the run leaves the
            // run's total in its lowest lane; texels span warps -> atomics
            const unsigned grp = __match_any_sync(0xffffffffu, n);
            const int last = 31 - __clz(grp);
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const unsigned long long ok = __shfl_down_sync(0xffffffffu, key, off);
                const uint32_t oi = __shfl_down_sync(0xffffffffu, inc, off);
                if (lane + off <= last) {
                    key = ok < key ? ok : key;
                    inc += oi;
                }
            }
            if (n != 0xffffffffu && lane == __ffs(grp) - 1) {
                if (key != WF_NO_HIT) atomicMin(&B.tkey[n], key);
                if (inc) atomicAdd(&B.votes[n], inc);
            }
        }
        // r0 is a multiple of 32 (grid and block sizes are): chunk r0 / 32
        const unsigned m = __ballot_sync(0xffffffffu, need);
        const unsigned bx = __ballot_sync(0xffffffffu, sx), by = __ballot_sync(0xffffffffu, sy),
                       bz = __ballot_sync(0xffffffffu, sz);
        if (lane == 0) B.chunk[r0 >> 5] = make_uint4(m, bx, by, bz);
    }
}

// chunks this call's pass 1 wrote: the workspace is sized for the capacity,
// and records beyond the actual rays are stale (an earlier call's or never
// written) -- they must not enter the queue
__device__ __forceinline__ int64_t wf_live_chunks(const WfBuffers& B, int64_t n_chunks) {
    const int64_t R = min(*B.texels, B.m_cap) * B.x;
    return min(n_chunks, (R + 31) / 32);
}

// long rays of a chunk in octant o
__device__ __forceinline__ unsigned oct_mask(const uint4& c, int o) {
    return c.x & (o & 1 ? c.y : ~c.y) & (o & 2 ? c.z : ~c.z) & (o & 4 ? c.w : ~c.w);
}

// Block-wide exclusive scan (NT threads) of 8 per-thread octant counts;
// returns the block totals in tot[8] (shared; warp_tot holds 8 * NT / 32).
template <int NT>
__device__ __forceinline__ void oct_block_scan(int (&cnt)[8], int (&excl)[8], int* warp_tot,
                                               int* tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        int incl = cnt[o];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        excl[o] = incl - cnt[o];
        if (lane == 31) warp_tot[o * (NT / 32) + wid] = incl;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        int run = 0;
        for (int w = 0; w < NT / 32; ++w) {
            const int t = warp_tot[threadIdx.x * (NT / 32) + w];
            warp_tot[threadIdx.x * (NT / 32) + w] = run;
            run += t;
        }
        tot[threadIdx.x] = run;
    }
    __syncthreads();
#pragma unroll
    for (int o = 0; o < 8; ++o) excl[o] += warp_tot[o * (NT / 32) + wid];
}

__global__ void __launch_bounds__(WF_OCT_THREADS) wf_oct_count_kernel(int64_t n_chunks, WfBuffers B) {
    __shared__ int warp_tot[8 * (WF_OCT_THREADS / 32)];
    __shared__ int tot[8];
    const int64_t c = (int64_t)blockIdx.x * WF_OCT_THREADS + threadIdx.x;
    const uint4 ch = c < wf_live_chunks(B, n_chunks) ? B.chunk[c] : make_uint4(0, 0, 0, 0);
    int cnt[8], excl[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) cnt[o] = __popc(oct_mask(ch, o));
    oct_block_scan<WF_OCT_THREADS>(cnt, excl, warp_tot, tot);
    if (threadIdx.x < 8) B.oct_blk[(int64_t)blockIdx.x * 8 + threadIdx.x] = tot[threadIdx.x];
}

// Per-octant exclusive scan of the block counts: one cub device scan over
// 8-wide count vectors (decoupled look-back, many CTAs).
struct Oct8 {
    int v[8];
};
struct Oct8Sum {
    __host__ __device__ __forceinline__ Oct8 operator()(const Oct8& a, const Oct8& b) const {
        Oct8 r;
#pragma unroll
        for (int o = 0; o < 8; ++o) r.v[o] = a.v[o] + b.v[o];
        return r;
    }
};

static size_t oct_scan_temp_bytes(int64_t nb) {
    size_t t = 0;
    Oct8 zero{};
    cub::DeviceScan::ExclusiveScan(nullptr, t, (const Oct8*)nullptr, (Oct8*)nullptr, Oct8Sum(), zero,
                                   (int)nb);
    return t;
}

// The block's long rays, staged in shared memory octant by octant, then
// written as 8 contiguous runs (coalesced).
__global__ void __launch_bounds__(WF_OCT_THREADS) wf_oct_scatter_kernel(int64_t n_chunks, WfBuffers B) {
    __shared__ int warp_tot[8 * (WF_OCT_THREADS / 32)];
    __shared__ int tot[8];
    __shared__ int32_t stage[WF_OCT_THREADS * 32];
    const int64_t c = (int64_t)blockIdx.x * WF_OCT_THREADS + threadIdx.x;
    const uint4 ch = c < wf_live_chunks(B, n_chunks) ? B.chunk[c] : make_uint4(0, 0, 0, 0);
    int cnt[8], excl[8];
    unsigned om[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        om[o] = oct_mask(ch, o);
        cnt[o] = __popc(om[o]);
    }
    oct_block_scan<WF_OCT_THREADS>(cnt, excl, warp_tot, tot);
    int seg[9];
    seg[0] = 0;
#pragma unroll
    for (int o = 0; o < 8; ++o) seg[o + 1] = seg[o] + tot[o];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        unsigned mk = om[o];
        int p = seg[o] + excl[o];
        while (mk) {
            const int l = __ffs(mk) - 1;
            stage[p++] = (int32_t)((c << 5) + l);
            mk &= mk - 1;
        }
    }
    __syncthreads();
    // octant o's rays start after every ray of octants < o (totals = last
    // block's exclusive offset + its count)
    __shared__ int gpos[8];
    if (threadIdx.x < 8) {
        const int64_t last = (int64_t)(gridDim.x - 1) * 8;
        int base = 0;
        for (int o = 0; o < (int)threadIdx.x; ++o) base += B.oct_pos[last + o] + B.oct_blk[last + o];
        gpos[threadIdx.x] = base + B.oct_pos[(int64_t)blockIdx.x * 8 + threadIdx.x];
        if (blockIdx.x == 0 && threadIdx.x == 7)
            *B.qcount = base + B.oct_pos[last + 7] + B.oct_blk[last + 7];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < seg[8]; p += WF_OCT_THREADS) {
        int o = 0;
#pragma unroll
        for (int q = 1; q < 8; ++q) o += p >= seg[q];
        B.queue[gpos[o] + (p - seg[o])] = stage[p];
    }
}

// STK: traversal stack entries (RTSDF_FAST_STACK, or WF2_SMALL_STACK for BVH4s
// whose depth allows it: 18 KB less shared memory per block -- more L1 for the
// tree and one more resident block: C3 pass 2 2.22 -> 2.10 ms).
#define WF2_SMALL_STACK 24
template <bool WIDE, int STK>
#ifndef WF2_MINB
#define WF2_MINB (WF_MINB + 1)  // small-stack pass 2: resident blocks per SM
#endif
__global__ void __launch_bounds__(WF_THREADS, STK <= WF2_SMALL_STACK ? WF2_MINB : WF_MINB)
    wf_pass2_kernel(SampleParams P, WfBuffers B) {
    __shared__ int32_t stack_mem[STK * WF_THREADS];
    __shared__ __half tstack_mem[WIDE ? STK * WF_THREADS : 1];
    const int64_t Q = *B.qcount;
#ifndef WF2_DYN
#define WF2_DYN 1
#endif
#if WF2_DYN
    // warps claim 32-ray chunks of the queue dynamically (one atomic per chunk):
    // a warp that drew short rays takes the next chunk instead of idling at the
    // end of a static grid-stride share (claiming the next chunk one step
    // ahead, to overlap the atomic with the traversal, measured 1.92 -> 1.96 ms)
    const int lane = threadIdx.x & 31;
    while (true) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(B.qhead, 32ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)base >= Q) break;
        const int64_t q = (int64_t)base + lane;
        if (q >= Q) continue;
#else
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q;
         q += (int64_t)gridDim.x * blockDim.x) {
#endif
        const int64_t r = B.queue[q];
        double ox, oy, oz, dx, dy, dz;
        // regenerated, not handed over: pass 1 storing the long rays' fp64
        // directions ([R] x 32 B) for pass 2 to read back measured pass 2
        // 1.93 -> 1.92 ms but pass 1 2.42 -> 2.47 ms (register spill)
        wf_ray(P, B, r, ox, oy, oz, dx, dy, dz);
        int32_t id;
        int facing;
        // long rays: near-first traversal (with dynamic chunks the while-while
        // form measured slower: 2.30 vs 2.23 ms at C3)
        double t = WIDE ? trace_fast4(P.bvh4, ox, oy, oz, dx, dy, dz, P.t_max, stack_mem + threadIdx.x,
                                      tstack_mem + threadIdx.x, WF_THREADS, id, facing, P.tb)
                        : wf_trace<WIDE>(P, ox, oy, oz, dx, dy, dz, stack_mem + threadIdx.x,
                                         tstack_mem + threadIdx.x, id, facing, 0, nullptr);
        if (id >= 0) wf_commit(B, fdiv((unsigned)r, P.div_x), t, facing);
    }
}

// raysample.py:140-152 (per-texel min / votes, in ray order) + :229-244 (Eq. 1)
__global__ void __launch_bounds__(WF_THREADS) wf_reduce_update_kernel(SampleParams P, WfBuffers B) {
    const int64_t M = min(*P.count, P.m_cap);
    const int64_t nyz = (int64_t)P.fny * P.fnz;
    for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < M;
         n += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = B.tkey[n];
        const uint32_t votes = B.votes[n];
        const double best = key == WF_NO_HIT ? __longlong_as_double(0x7ff0000000000000ll)
                                             : __longlong_as_double((long long)key);
        const int fr = (int)(votes & 0xffffu), bk = (int)(votes >> 16);
        if (P.samp_min) P.samp_min[n] = best;
        if (P.samp_front) P.samp_front[n] = fr;
        if (P.samp_back) P.samp_back[n] = bk;
        if (!P.prev) continue;
        const int64_t lin = __ldg(P.idx + n);
        const int i = (int)(lin / nyz), j = (int)((lin / P.fnz) % P.fny), k = (int)(lin % P.fnz);
        const double px = P.coarse.lox + ((double)i + 0.5) * P.fhx;
        const double py = P.coarse.loy + ((double)j + 0.5) * P.fhy;
        const double pz = P.coarse.loz + ((double)k + 0.5) * P.fhz;
        float rm = P.run_min[lin];
        int32_t f = P.front[lin], b = P.back[lin];
        if (!P.mask_old[lin]) {
            rm = __int_as_float(0x7f800000);
            f = 0;
            b = 0;
        }
        const double m = best;
        if (m < (double)rm) rm = (float)m;
        f += fr;
        b += bk;
        P.run_min[lin] = rm;
        P.front[lin] = f;
        P.back[lin] = b;
        const double c = (double)(float)trilinear(P.coarse, px, py, pz);  // c_fine (f32)
        const double blend = P.alpha * fabs((double)P.prev[lin]) + (1.0 - P.alpha) * c;
        const double mag = blend < m ? blend : m;
        P.out[lin] = b > f ? (float)(-mag) : (float)mag;
    }
}

static int64_t wf_chunks(int64_t R) { return (R + 31) / 32; }
static int64_t wf_oct_blocks(int64_t R) { return (wf_chunks(R) + WF_OCT_THREADS - 1) / WF_OCT_THREADS; }

// qcount | per texel: tex, tkey, votes | per ray: queue | per 32 rays: chunk
// records | per octant-compaction block: 8 counters
static size_t wf_ws_bytes(int64_t m_cap, int x) {
    const int64_t R = m_cap * (x > 0 ? x : 1);
    return 256 + (size_t)m_cap * (sizeof(double4) + sizeof(unsigned long long) + sizeof(uint32_t)) +
           (size_t)R * sizeof(int32_t) + 256 + 256 + (size_t)wf_chunks(R) * sizeof(uint4) +
           2 * ((size_t)wf_oct_blocks(R) * 8 * sizeof(int32_t) + 256) +
           oct_scan_temp_bytes(wf_oct_blocks(R)) + 256;
}

static void launch_oct_queue(const WfBuffers& B, int64_t R, cudaStream_t st) {
    const int64_t nc = wf_chunks(R), nb = wf_oct_blocks(R);
    wf_oct_count_kernel<<<(unsigned)nb, WF_OCT_THREADS, 0, st>>>(nc, B);
    size_t tb = B.scan_tmp_bytes;
    cub::DeviceScan::ExclusiveScan(B.scan_tmp, tb, (const Oct8*)B.oct_blk, (Oct8*)B.oct_pos,
                                   Oct8Sum(), Oct8{}, (int)nb, st);
    wf_oct_scatter_kernel<<<(unsigned)nb, WF_OCT_THREADS, 0, st>>>(nc, B);
}

}  // namespace rtsdf

using namespace rtsdf;

extern "C" size_t rtsdf_sample_ws_bytes(int64_t m_cap, int x) { return wf_ws_bytes(m_cap, x); }

extern "C" int rtsdf_sample_update(const void* bvh_packed, int64_t n_nodes, int64_t n_tris,
                                   int64_t n_nodes4, int stack4,
                                   const int64_t* idx,
                                   const int64_t* count, int64_t m_cap,
                                   const rtsdf_resample_desc* rs, int x, uint64_t seed,
                                   int64_t frame, const int64_t* frame_dev, double t_max,
                                   const double* dirs,
                                   double* samp_min, int32_t* samp_front, int32_t* samp_back,
                                   const float* prev, const uint8_t* mask_old, float* run_min,
                                   int32_t* front, int32_t* back, double alpha, float* out,
                                   void* ws, size_t ws_bytes, void* stream) {
    if (x < 0 || !rs || !count || !idx) {
        set_error("sample_update: bad arguments");
        return RTSDF_ERR_INVALID;
    }
    if (prev && (!mask_old || !run_min || !front || !back || !out)) {
        set_error("sample_update: update needs mask_old/run_min/front/back/out");
        return RTSDF_ERR_INVALID;
    }
    if (m_cap <= 0) return RTSDF_OK;
    SampleParams P;
    P.bvh = fast_bvh_view(bvh_packed, n_nodes, n_tris);
    P.idx = idx;
    P.count = count;
    P.m_cap = m_cap;
    P.n_begin = 0;
    P.coarse = FieldView{rs->coarse, rs->cnx, rs->cny, rs->cnz, rs->clo[0], rs->clo[1],
                         rs->clo[2], rs->ch[0], rs->ch[1], rs->ch[2], 0.0f};
    P.fnx = rs->fnx;
    P.fny = rs->fny;
    P.fnz = rs->fnz;
    P.fhx = rs->fh[0];
    P.fhy = rs->fh[1];
    P.fhz = rs->fh[2];
    P.x = x;
    P.div_x = make_fastdiv((uint32_t)(x > 0 ? x : 1));
    P.div_ny = make_fastdiv((uint32_t)rs->fny);
    P.div_nz = make_fastdiv((uint32_t)rs->fnz);
    P.seed = seed;
    P.frame = frame;
    P.frame_dev = frame_dev;
    P.t_max = t_max;
    P.tb = tmax_bound(t_max);
    P.dirs = dirs;
    P.samp_min = samp_min;
    P.samp_front = samp_front;
    P.samp_back = samp_back;
    P.prev = prev;
    P.mask_old = mask_old;
    P.run_min = run_min;
    P.front = front;
    P.back = back;
    P.alpha = alpha;
    P.out = out;
    // wavefront sampler (needs the workspace); the warp-per-texel kernel when
    // there is none or x is beyond the packed-vote range
    const bool wf_ok = x >= 1 && x <= 65535 && ws && ws_bytes >= wf_ws_bytes(m_cap, x) &&
                       m_cap * (int64_t)x < ((int64_t)1 << 31);
    cudaStream_t st = (cudaStream_t)stream;
    if (wf_ok) {
        WfBuffers B;
        char* p = (char*)ws;
        B.qcount = (int64_t*)p;
        p += 256;
        const int64_t R = m_cap * x;
        B.tex = (double4*)p;
        p += m_cap * sizeof(double4);
        B.tkey = (unsigned long long*)p;
        p += m_cap * sizeof(unsigned long long);
        B.votes = (uint32_t*)p;
        p += m_cap * sizeof(uint32_t);
        B.queue = (int32_t*)p;
        p += R * sizeof(int32_t);
        p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
        B.chunk = (uint4*)p;
        p += wf_chunks(R) * sizeof(uint4);
        const int64_t nob = wf_oct_blocks(R);
        B.oct_blk = (int32_t*)p;
        p += (nob * 8 * sizeof(int32_t) + 255) / 256 * 256;
        B.oct_pos = (int32_t*)p;
        p += (nob * 8 * sizeof(int32_t) + 255) / 256 * 256;
        B.scan_tmp = p;
        B.scan_tmp_bytes = oct_scan_temp_bytes(nob);
        B.qhead = (unsigned long long*)((char*)B.qcount + 8);
        B.texels = count;
        B.m_cap = m_cap;
        B.x = x;
        B.aligned = 32 % x == 0;
        cudaMemsetAsync(B.qcount, 0, 2 * sizeof(int64_t), st);  // qcount, qhead
        int64_t blocks = (R + WF_THREADS - 1) / WF_THREADS;
        int64_t cap = (int64_t)num_sms() * 24;
        const bool wide = n_nodes4 > 0;
        // large BVH4s (C4: ~10^5 nodes): almost no ray finishes at the root, so pass 1
        // only generates, classifies and queues (budget 1: measured 110.5 -> 109.5
        // ms/frame at C4); small ones finish their ground-plane leaves in pass 1
        const int budget = wide ? (n_nodes4 > 8 * 4096 ? 1 : WF_BUDGET4) : WF_BUDGET;  // 8 octant records per node
        const unsigned b1 = (unsigned)(blocks < cap ? blocks : cap), b2 = (unsigned)(num_sms() * WF_B2_PER_SM);
        int launches = 4;  // setup, pass 1, pass 2, reduce + update
        wf_setup_kernel<<<(unsigned)cap, WF_THREADS, 0, st>>>(P, B);
        if (!B.aligned) {  // accumulators not initialised by pass 1
            wf_init_kernel<<<(unsigned)cap, WF_THREADS, 0, st>>>(P, B);
            ++launches;
        }
        if (wide) {
            P.bvh4 = fast_bvh4_view(bvh_packed, n_nodes, n_tris);
            wf_pass1_kernel<true><<<b1, WF_THREADS, 0, st>>>(P, B, budget);
            launch_oct_queue(B, R, st);
            launches += 2;  // count + scatter (+ cub's scan)
            if (stack4 > 0 && stack4 <= WF2_SMALL_STACK)
                wf_pass2_kernel<true, WF2_SMALL_STACK><<<b2, WF_THREADS, 0, st>>>(P, B);
            else
                wf_pass2_kernel<true, RTSDF_FAST_STACK><<<b2, WF_THREADS, 0, st>>>(P, B);
        } else {
            wf_pass1_kernel<false><<<b1, WF_THREADS, 0, st>>>(P, B, budget);
            launch_oct_queue(B, R, st);
            launches += 2;
            wf_pass2_kernel<false, RTSDF_FAST_STACK><<<b2, WF_THREADS, 0, st>>>(P, B);
        }
        int64_t ublocks = (m_cap + WF_THREADS - 1) / WF_THREADS;
        wf_reduce_update_kernel<<<(unsigned)(ublocks < cap ? ublocks : cap), WF_THREADS, 0, st>>>(P, B);
        // texels beyond the workspace capacity (the host sized it from an earlier
        // frame's count without a sync): traced and updated by the workspace-free
        // warp-per-texel kernel -- same per-ray results, same order-free
        // reduction, so the frame is exact whatever the capacity; a no-op when
        // *count <= m_cap
        SampleParams T = P;
        T.n_begin = m_cap;
        T.m_cap = INT64_MAX;
        sample_update_kernel<<<(unsigned)(num_sms() * 4), SAMPLE_THREADS, 0, st>>>(T);
        ++launches;
        count_launch(launches);
        return check_launch("sample_update");
    }
    int tpw = x >= 32 || x == 0 ? 1 : 32 / x;
    int64_t warps_needed = (m_cap + tpw - 1) / tpw;
    int64_t blocks = (warps_needed + SAMPLE_THREADS / 32 - 1) / (SAMPLE_THREADS / 32);
    int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    sample_update_kernel<<<(unsigned)blocks, SAMPLE_THREADS, 0, st>>>(P);
    count_launch();
    return check_launch("sample_update");
}

#ifdef RTSDF_TRACE_STATS
// experiment builds only: read and clear the traversal counters of this module
extern "C" void rtsdf_debug_trace_stats(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, rtsdf::g_trace_stats, sizeof(unsigned long long) * 12);
    static const unsigned long long zero[12] = {};
    cudaMemcpyToSymbol(rtsdf::g_trace_stats, zero, sizeof(zero));
}
#endif
