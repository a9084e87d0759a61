/*
 * rtsdf.h -- C ABI of the B200-native RTSDF hot path (librtsdf.so).
 *
 * The reference (`sdfshadow`, Python + numba, /root/reference/pkg/src/sdfshadow)
 * has no FFI: every public op is a Python validator around ONE numba kernel
 * called with raw arrays plus scalar dims/spacings.  Each entry point below
 * replaces exactly one of those kernel calls; the file:line it replaces is
 * cited on each declaration.  The Python host package
 * (paper_2210_06160_b200/) binds these with ctypes, keeping the reference's
 * function names, argument meaning and exception types.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers unless marked (host).  The caller
 *     owns every buffer; workspace sizes are queried with *_ws_bytes.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *     it, deterministic, and free of order-dependent atomics.
 *   - Grids are C-order (nx, ny, nz), z fastest, like the reference arrays.
 *   - Seeds inside the library are PACKED int32: (i << 20) | (j << 10) | k
 *     when every dim is <= 1024; for larger grids k takes the low bits(nz-1)
 *     bits, j the next bits(ny-1), i the top bits(nx-1) (their sum must be
 *     <= 31, and such grids run the per-cell JFA kernel).  EMPTY = -1.
 *     Numeric order == lexicographic (i, j, k) order.  The layout is a
 *     function of the dims; rtsdf_seeds_packed_to_linear converts to the
 *     reference's linear index (jfa.py:31,53).
 *   - Return value: 0 on success, else an RTSDF_ERR_* code; no exceptions or
 *     exits cross the ABI.  rtsdf_last_error() gives a message (thread-local).
 */
#ifndef RTSDF_H
#define RTSDF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RTSDF_OK = 0,
    RTSDF_ERR_INVALID = 1,   /* bad argument (maps to ValueError)            */
    RTSDF_ERR_CUDA = 2,      /* CUDA launch / runtime failure (RuntimeError) */
    RTSDF_ERR_DIMS = 3,      /* grid dims beyond packed int32 seeds: bits(nx-1) + bits(ny-1) + bits(nz-1) > 31 */
    RTSDF_ERR_WORKSPACE = 4  /* workspace too small                          */
};

const char* rtsdf_version(void);
const char* rtsdf_last_error(void);
/* number of kernel launches issued by this library since load (diagnostics) */
int64_t rtsdf_launch_count(void);
/* Adds n to the launch counter (a CUDA-graph replay of n counted launches). */
void rtsdf_count_launches(int64_t n);

/* ---------------------------------------------------------------- voxelize */
/* Replaces voxel.py:179 (_voxelize_kernel call) + the OOB check voxel.py:168-175
 * + jfa.py:54 (jfa_init's np.where).  Conservative closed-box 13-axis SAT in
 * fp64 without FMA.  occ (nullable) is zeroed then set to 1 per occupied cell;
 * seed_packed (nullable) is set to EMPTY then self-seeded per occupied cell.
 * counters (device, int64[2]) receive [0] = triangles outside [lo, hi],
 * [1] = occupied-cell writes (> 0 iff any cell occupied).  bad_flags (nullable,
 * uint8[n_tris]) receives 1 for each out-of-bounds triangle.               */
size_t rtsdf_voxelize_ws_bytes(int64_t n_tris);
int rtsdf_voxelize(const double* verts, int64_t n_verts, const int32_t* tris, int64_t n_tris,
                   const double* lo /*host[3]*/, const double* hi /*host[3]*/, int nx, int ny,
                   int nz, uint8_t* occ, int32_t* seed_packed, int64_t* counters,
                   uint8_t* bad_flags, void* ws, size_t ws_bytes, void* stream);

/* --------------------------------------------------------------------- JFA */
/* Replaces jfa.py:47-55 (jfa_init): seed = packed(c) if occ[c] else EMPTY;
 * count (device int64, nullable) += occupied cells.                         */
int rtsdf_jfa_init(const uint8_t* occ, int nx, int ny, int nz, int32_t* seed_packed,
                   int64_t* count, void* stream);

/* Replaces jfa.py:136 (_jfa_step_kernel call): one 27-tap pass at `offset`.
 * Adopt iff fp64 d2 (jfa.py:72-76, left to right, no FMA) is smaller, or equal
 * and the seed is lexicographically smaller (jfa.py:116-124).  (wx, wy, wz) > 0
 * asserts hx^2 : hy^2 : hz^2 == wx : wy : wz EXACTLY (host-checked with exact
 * rationals); the kernel then orders candidates by the integer
 * q = wx dx^2 + wy dy^2 + wz dz^2 and evaluates fp64 d2 only on integer ties.
 * (0, 0, 0) = general fp64 path.                                            */
int rtsdf_jfa_step(const int32_t* src, int32_t* dst, int nx, int ny, int nz, int offset,
                   double hx, double hy, double hz, int wx, int wy, int wz, void* ws,
                   size_t ws_bytes, void* stream);
/* Workspace of the JFA entry points: the integer-tie fix-up list (a device
 * counter + one int32 slot per cell of the grid / slab).                    */
size_t rtsdf_jfa_ws_bytes(int nx, int ny, int nz);

/* Slab form for z-slab (outer-axis) sharding across GPUs: this rank owns global
 * planes [x0, x0 + nxl) of an nx-plane grid in `local`; halo_lo holds global
 * planes [lo_first, lo_first + n_lo) and halo_hi [hi_first, hi_first + n_hi)
 * (received from other ranks).  Output planes [out_first, out_first +
 * out_count) (inside the owned range; dst points at plane out_first), so the
 * interior planes [x0 + k, x0 + nxl - k) -- which read only local planes -- can
 * run while the halo exchange is in flight and the boundary planes after it.
 * Every plane an output cell needs must be present; the host schedules the
 * exchange.                                                                 */
int rtsdf_jfa_step_slab(const int32_t* local, const int32_t* halo_lo, const int32_t* halo_hi,
                        int32_t* dst, int nx, int x0, int nxl, int lo_first, int n_lo,
                        int hi_first, int n_hi, int ny, int nz, int offset, double hx,
                        double hy, double hz, int wx, int wy, int wz, int out_first,
                        int out_count, void* ws, size_t ws_bytes, void* stream);
/* Compressed halo planes (sparse early passes of the slab schedule): n_el
 * int32 seeds as a bitmap of their non-EMPTY 32-cell segments
 * (rtsdf_halo_bitmap_words(n_el) words) + those segments packed in order
 * (payload capacity n_el; *total (device) = packed segments).  decompress
 * expands (bits, payload) into dst, EMPTY elsewhere.  ws:
 * rtsdf_halo_ws_bytes(n_el).  Exact: every non-EMPTY value is transmitted. */
int64_t rtsdf_halo_bitmap_words(int64_t n_el);
size_t rtsdf_halo_ws_bytes(int64_t n_el);
int rtsdf_halo_compress(const int32_t* src, int64_t n_el, uint32_t* bits, int32_t* payload,
                        int64_t* total, void* ws, size_t ws_bytes, void* stream);
int rtsdf_halo_decompress(const uint32_t* bits, const int32_t* payload, int64_t n_el, int32_t* dst,
                          void* ws, size_t ws_bytes, void* stream);

/* Replaces jfa.py:140-145 (jfa_run's pass loop): runs the whole schedule
 * n/2 .. 1 ping-ponging between buf_a (holding the init seeds) and buf_b.
 * *which (host) = 0 if the result is in buf_a, 1 if in buf_b.               */
int rtsdf_jfa_run(int32_t* buf_a, int32_t* buf_b, int nx, int ny, int nz, double hx, double hy,
                  double hz, int wx, int wy, int wz, int* which, void* ws, size_t ws_bytes,
                  void* stream);

/* Replaces pipeline.py:120-124 (run_jf = jfa_run + seeds_to_sdf): the full
 * schedule ping-ponging buf_a (init seeds) / buf_b, with the last (k = 1) pass
 * writing the f32 SDF straight into `out` (K3 fused: no seed grid round trip).
 * Both seed buffers are clobbered.  empty_count as in rtsdf_seeds_to_sdf.   */
int rtsdf_jfa_run_sdf(int32_t* buf_a, int32_t* buf_b, float* out, int nx, int ny, int nz,
                      double hx, double hy, double hz, int wx, int wy, int wz, double beta,
                      int64_t* empty_count, void* ws, size_t ws_bytes, void* stream);

/* Replaces jfa.py:180 (_seed_distance_kernel call): out = f32(sqrt(d2_fp64) - beta).
 * empty_count (device int64, nullable) += EMPTY cells (NoSeedsError check,
 * jfa.py:176-177).                                                          */
int rtsdf_seeds_to_sdf(const int32_t* seed_packed, float* out, int nx, int ny, int nz,
                       double hx, double hy, double hz, double beta, int64_t* empty_count,
                       void* stream);

/* ------------------------------------------------- slab (range) forms
 * For the z-slab sharded frame (paper_2210_06160_b200/shard.py).
 * These calls address every buffer by GLOBAL cell index: pass a base pointer
 * p such that p + c is the storage of global cell c for each cell the call
 * touches (slab-local storage that starts at global cell c0 -> storage - c0).
 * Only the range's cells are read or written -- plus, for the trilinear
 * resample, coarse planes x0 - 1 .. x0 + nxl (a one-plane halo).           */
int rtsdf_seeds_to_sdf_range(const int32_t* seed_packed, float* out, int nx, int ny, int nz,
                             int x0, int nxl, double hx, double hy, double hz, double beta,
                             int64_t* empty_count, void* stream);
int rtsdf_seeds_packed_to_linear(const int32_t* packed, int32_t* linear, int nx, int ny, int nz,
                                 void* stream);
int rtsdf_seeds_linear_to_packed(const int32_t* linear, int32_t* packed, int nx, int ny, int nz,
                                 void* stream);

/* ---------------------------------------------------- resample, mask, band */
/* Replaces raysample.py:114 (_coarse_at_fine_kernel) and the band-exit reset
 * raysample.py:288-295.  Per fine texel: v = fp64 trilinear of coarse at
 * clo + (i + 0.5) fh (field.py:95-128); mask = v <= d (fp64).
 *   c_fine (nullable): f32(v) for every texel;
 *   out_unmasked (nullable): f32(v) where !mask (raysample.py:290), untouched
 *                            where masked (the sampler writes those);
 *   mask_new (nullable) u8; block_counts (nullable, int32[n_blocks]) masked
 *   count per RS_CELLS_PER_BLOCK chunk for rtsdf_compact_mask;
 *   mask_old + run_min/front/back (nullable): reset where mask_old & !mask. */
int64_t rtsdf_mask_blocks(int64_t n_cells);
int rtsdf_resample_mask(const float* coarse, int cnx, int cny, int cnz,
                        const double* clo /*host[3]*/, const double* ch /*host[3]*/, int fnx,
                        int fny, int fnz, const double* fh /*host[3]*/, double d, float* c_fine,
                        float* out_unmasked, uint8_t* mask_new, int32_t* block_counts,
                        const uint8_t* mask_old, float* run_min, int32_t* front, int32_t* back,
                        void* stream);
/* Replaces raysample.py:266 (np.flatnonzero): ascending int64 indices of
 * mask != 0; *count (device int64) = M.  Needs block_counts from
 * rtsdf_resample_mask (or NULL to recount).                                 */
size_t rtsdf_compact_ws_bytes(int64_t n_cells);
int rtsdf_compact_mask(const uint8_t* mask, int64_t n_cells, int32_t* block_counts,
                       int64_t* idx, int64_t* count, void* ws, size_t ws_bytes, void* stream);
/* Range forms (global cell addressing, see the slab section above): cells
 * [c0, c0 + n_range) of the fine grid; block_counts / the compaction
 * workspace are sized for n_range; idx holds global indices.               */
int rtsdf_resample_mask_range(const float* coarse, int cnx, int cny, int cnz,
                              const double* clo /*host[3]*/, const double* ch /*host[3]*/,
                              int fnx, int fny, int fnz, const double* fh /*host[3]*/, double d,
                              int64_t c0, int64_t n_range, float* c_fine, float* out_unmasked,
                              uint8_t* mask_new, int32_t* block_counts, const uint8_t* mask_old,
                              float* run_min, int32_t* front, int32_t* back, void* stream);
int rtsdf_compact_mask_range(const uint8_t* mask, int64_t c0, int64_t n_range,
                             int32_t* block_counts, int64_t* idx, int64_t* count, void* ws,
                             size_t ws_bytes, void* stream);

/* --------------------------------------------------------------------- BVH */
/* Replaces geometry.py:202-267 (build_bvh), on the host (plain C++, same
 * median split on the longest node-bbox axis, stable order, leaf <= 4) so the
 * tree -- and therefore traversal order and pruning -- is the reference's.
 * All pointers HOST.  node arrays sized >= 2*T-1.  Returns node count (< 0 on
 * error).                                                                   */
int64_t rtsdf_bvh_build_host(const double* tri_lo, const double* tri_hi, int64_t n_tris,
                             double* node_lo, double* node_hi, int32_t* node_left,
                             int32_t* node_right, int32_t* order);
/* Binned-SAH build (host) in the same flat format, for the K6 search only:
 * that search returns the brute-force closest hit whatever the tree, so it may
 * use a tree built for speed (replaces nothing in the reference; the
 * reference-order traversal keeps using rtsdf_bvh_build_host's tree).
 * max_leaf in 1..7.                                                         */
int64_t rtsdf_bvh_build_sah_host(const double* tri_lo, const double* tri_hi, int64_t n_tris,
                                 int max_leaf, double* node_lo, double* node_hi,
                                 int32_t* node_left, int32_t* node_right, int32_t* order);
/* Collapse a flat binary tree into 4-wide nodes (128 B: padded fp32 child
 * boxes + child refs) for the K6 search; host in/out.  Each node is written
 * as 8 interleaved octant copies (record 8 i + o: the x / y / z lo and hi
 * planes swapped where bit 0 / 1 / 2 of o is set; inner child refs = 8 i), so
 * a ray reads its near planes from the lo slots.  cap and the return value
 * count 128-B records (8 per node); < 0: capacity.                          */
int64_t rtsdf_bvh4_collapse_host(const double* node_lo, const double* node_hi,
                                 const int32_t* node_left, const int32_t* node_right,
                                 int64_t n_nodes, void* out_nodes4, int64_t cap);
/* Pack the flat BVH (device SoA as in BvhIndex, geometry.py:186-195) into the
 * device traversal layout: nodes (64 B each) and triangles (128 B each); the
 * size is rounded up to 128 B (a BVH4 collapse appended there is aligned). */
size_t rtsdf_bvh_packed_bytes(int64_t n_nodes, int64_t n_tris);
int rtsdf_bvh_pack(const double* node_lo, const double* node_hi, const int32_t* node_left,
                   const int32_t* node_right, const int32_t* order, const double* tri_a,
                   const double* tri_e1, const double* tri_e2, const double* tri_n,
                   int64_t n_nodes, int64_t n_tris, void* packed, void* stream);

/* Replaces geometry.py:395-410 (ray_query) for a batch of rays.  fast = 0:
 * the reference's own traversal order in fp64 (_bvh_ray verbatim); fast = 1:
 * the K6 search (fp32 conservative boxes + fp32 pre-test, exact fp64 confirm)
 * that returns the brute-force closest hit the reference's contract names
 * (geometry.py:3-6).                                                        */
int rtsdf_ray_query(const void* bvh_packed, int64_t n_nodes, int64_t n_tris, int fast,
                    const double* origins, const double* dirs, int64_t n, double t_max,
                    double* out_t, int32_t* out_id, int32_t* out_facing, void* stream);

/* ---------------------------------------------- ray-sampled refine + Eq. 1 */
/* Replaces raysample.py:277-299 (_sample_masked_kernel + band reset +
 * _update_masked_kernel).  Default (workspace given): wavefront -- every ray
 * traced with a small node budget (its texel's finished rays merged by a warp
 * reduction), budget-exhausted rays re-traced from a compacted queue and
 * merged into per-texel accumulators (atomicMin on the fp64 bits of t, t >= 0;
 * atomicAdd of packed front/back votes) -- min and integer sums are exact and
 * order-free, so results are deterministic and independent of the queue
 * order; then one thread per texel applies Eq. 1.  Without a workspace: one
 * warp per texel, one lane per ray, warp-reduced.  Closest hits are the
 * brute-force ones the reference's BVH contract names (geometry.py:3-6;
 * trace.cuh).  Buffers indexed by texel (prev, out, mask_old, run_min,
 * front, back) use the global fine cell index idx[n].  M is read from
 * device memory (*count from rtsdf_compact_mask) so no host sync is needed;
 * m_cap bounds the grid.
 *   dirs (nullable): host-supplied table dirs[(n*x + r)*3 + c] (parity mode);
 *                    NULL = on-device SplitMix64 stream (rng.py:30-53).
 *   samp_min/front/back (nullable): per-texel frame results.
 *   update (prev != NULL): Eq. 1 combine + sign into out for masked texels,
 *     with c recomputed by the same trilinear as rtsdf_resample_mask; prev
 *     and out may alias (in-place).                                        */
typedef struct {
    const float* coarse;
    int cnx, cny, cnz;
    double clo[3], ch[3];
    int fnx, fny, fnz;
    double fh[3];
} rtsdf_resample_desc;

/* Workspace of the wavefront sampler for m_cap texels x rays: per-texel ray
 * setup (origin + stream key) and closest-hit / vote accumulators, and the
 * long-ray queue.  With ws == NULL the sampler falls back to the
 * warp-per-texel kernel (same results).                                     */
size_t rtsdf_sample_ws_bytes(int64_t m_cap, int x);
/* n_nodes4 > 0: the BVH4 collapse of the search tree (rtsdf_bvh4_collapse_host)
 * is appended to bvh_packed at offset rtsdf_bvh_packed_bytes(n_nodes, n_tris);
 * stack4: traversal stack entries that BVH4 can need (3 per level; 0 =
 * unknown): <= 24 lets the long-ray pass run with a smaller shared stack. */
int rtsdf_sample_update(const void* bvh_packed, int64_t n_nodes, int64_t n_tris, int64_t n_nodes4,
                        int stack4,
                        const int64_t* idx,
                        const int64_t* count, int64_t m_cap, const rtsdf_resample_desc* rs,
                        int x, uint64_t seed, int64_t frame, const int64_t* frame_dev /*nullable*/,
                        double t_max, const double* dirs,
                        double* samp_min, int32_t* samp_front, int32_t* samp_back,
                        const float* prev, const uint8_t* mask_old, float* run_min,
                        int32_t* front, int32_t* back, double alpha, float* out, void* ws,
                        size_t ws_bytes, void* stream);

/* ---------------------------------------------------- K5 on the device    */
/* Replaces geometry.py:202-267 (build_bvh) for the K6 search tree of dynamic
 * scenes (scenes.py:56-93 rebuilds it every animated frame): a linear BVH
 * (Karras radix tree over 30-bit Morton codes of the triangle-box centroids,
 * one triangle per leaf) built on the device from device vertices (V, 3) f64,
 * triangles (T, 3) i32 and unit normals (T, 3) f64 into the packed search
 * layout (rtsdf_bvh_packed_bytes(rtsdf_lbvh_nodes(T), T) bytes).  refit = 1
 * keeps the order and topology of the previous build in `ws` and recomputes
 * the boxes and triangle records from new vertices (same triangle list).
 * depth_out (device int32, nullable) receives max(depth) with atomicMax.
 * Any tree gives the reference's closest hits (geometry.py:3-6).           */
size_t rtsdf_lbvh_ws_bytes(int64_t n_tris);
int64_t rtsdf_lbvh_nodes(int64_t n_tris);
int rtsdf_lbvh_build(const double* verts, const int32_t* tris, const double* normals,
                     int64_t n_tris, int refit, void* packed, size_t packed_bytes, void* ws,
                     size_t ws_bytes, int32_t* depth_out, void* stream);

/* ------------------------------------------------------ validation oracles */
/* Replaces geometry.py:592 (_closest_many): exact unsigned point-to-mesh
 * distance per point (fp64 (n, 3) -> fp64 (n,)), over the reference-order
 * BVH (rtsdf_bvh_pack layout) in the reference's traversal order and pruning
 * (geometry.py:521-565), so results are bit-exact.                          */
int rtsdf_exact_distance(const void* bvh_packed, int64_t n_nodes, const double* points,
                         int64_t n, double* out, void* stream);
/* Replaces render.py:246 (_reference_kernel): per covered pixel the fraction
 * of spp cone-sampled shadow rays (origin pos + 1e-4 nrm, stream
 * (seed, pixel, 1)) with no hit; 1.0 where uncovered.  light / t1 / t2 are
 * the unit light direction and the cone basis (host[3] each, render.py:237-
 * 241); tan_r = tan(angular radius).  cos / sin are the bit-exact
 * restatement of the host glibc's (glibc_sincos.cuh), as below.            */
int rtsdf_reference_visibility(const void* bvh_packed, int64_t n_nodes, const double* g_pos,
                               const double* g_nrm, const uint8_t* g_cov, int height, int width,
                               const double* light /*host[3]*/, const double* t1 /*host[3]*/,
                               const double* t2 /*host[3]*/, double tan_r, int spp,
                               uint64_t seed, double* out_vis, void* stream);

/* Replaces rng.py:46-53 (unit_sphere_dir) for n stream keys x x counters:
 * dirs[(t * x + r) * 3 + c], the reference's uniform sphere directions with
 * the host libm's cos / sin restated bit for bit (glibc 2.39 FMA build,
 * glibc_sincos.cuh) -- the same device code the sampler uses.              */
int rtsdf_unit_sphere_dirs(const uint64_t* keys, int64_t n, int x, double* dirs, void* stream);
/* glibc sin / cos (|x| < 105414350, NaN beyond) of n device doubles: the
 * restatement's own check against the host libm (tests).                   */
int rtsdf_glibc_sincos(const double* x, int64_t n, double* s, double* c, void* stream);

/* ------------------------------------------------------------- soft shadow */
/* Replaces render.py:167 (_occlusion_kernel): per covered pixel fp64 sphere
 * trace with the triangulated cone term (raymarch.py:83-147).  sample_bias:
 * apply_bias (field.py:155-161) fused into every trilinear sample as an f32
 * subtraction, so shading needs no biased copy of the field (0 = none).
 * Only rows [row0, row0 + nrows) are shaded (pixel-sharded DL; the RNG stream
 * stays the global pixel index py * W + px, render.py:145).                 */
int rtsdf_occlusion(const float* field, int nx, int ny, int nz, const double* lo /*host[3]*/,
                    const double* h /*host[3]*/, const double* g_pos, const double* g_nrm,
                    const uint8_t* g_cov, int height, int width, int row0, int nrows,
                    const double* light /*host[3]*/,
                    double eps, int max_iter, double max_step, double t_max, double k,
                    double jitter, double offset, int draws, uint64_t seed, float sample_bias,
                    double* out, void* stream);
/* Replaces raymarch.py:128 (_march from sphere_trace) for a batch.          */
int rtsdf_sphere_trace(const float* field, int nx, int ny, int nz, const double* lo,
                       const double* h, const double* origins, const double* dirs, int64_t n,
                       double eps, int max_iter, double max_step, double t_max,
                       const double* t0 /*nullable*/, double k, int32_t* status, double* t,
                       int32_t* iters, double* min_term, void* stream);
/* Replaces field.py:141-148 (_sample_many).                                */
int rtsdf_trilinear_many(const float* field, int nx, int ny, int nz, const double* lo,
                         const double* h, const double* pts, int64_t n, double* out,
                         void* stream);
/* Replaces render.py:123 (_gbuffer_kernel).  cam (host[12]) = pos, fwd,
 * right, up.  fast = 0: the reference-order tree (_bvh_ray's traversal);
 * fast = 1: the K6 search tree (trace_fast; the same closest hit, used for
 * device-built trees of dynamic scenes).                                    */
int rtsdf_gbuffer(const void* bvh_packed, int64_t n_nodes, int64_t n_tris, int fast,
                  const double* normals_orig,
                  const float* albedo_orig, const double* cam, double half_w, double half_h,
                  int width, int height, double* out_pos, double* out_nrm, float* out_alb,
                  uint8_t* out_cov, void* stream);
/* Replaces render.py:186-192 (compose).                                    */
int rtsdf_compose(const double* g_nrm, const float* g_alb, const uint8_t* g_cov,
                  const double* occ, int height, int width, const double* light /*host[3]*/,
                  const double* background /*host[3]*/, float* out_rgb, void* stream);
/* Replaces field.py:155-161 (apply_bias): out = data - f32(bias) in f32.       */
int rtsdf_apply_bias(const float* data, int64_t n, float bias, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RTSDF_H */
