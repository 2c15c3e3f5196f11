/*
 * sph_b200.h -- C ABI of the B200-native SPH density / smoothing-length pass.
 *
 * One shared library (paper_1612_06090_b200/libsph_b200.so) behind the
 * reference's operator API.  Every entry point takes plain pointers and sizes;
 * no torch or CUDA types cross the boundary.  The reference is a Python
 * package (`sphlab`), so the reference-side binding is a ctypes stub
 * (INTEGRATION.md); the Python mirror in paper_1612_06090_b200/density.py is
 * that stub.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/sphlab):
 *   sph_density_pass      <- compute_density_pass(particles, config,
 *                            thread_count, max_iterations)   density.py:286-413
 *                            (smoothing_length / density / needs_recompute
 *                            written back into the caller's records,
 *                            PassStats todo trace in sph_stats)
 *   sph_sort_perm         <- build_octree(...).particle_perm   octree.py:306-348
 *   sph_neighbor_counts   <- range_query(tree, pos_i, h_i, exclude=i).size
 *                                                              octree.py:351-379
 *   sph_fnv1a64           <- snapshot.checksum64 / bench.density_checksum
 *                                                              snapshot.py:70-82,
 *                                                              bench.py:48-50
 *   sph_uniform_box_device <- workload.generate(UNIFORM_BOX) positions
 *                                                              workload.py:42-84
 *   sph_range_query       <- range_query(tree, pos_i, h_i, exclude=i) for all i
 *                                                              octree.py:179-227, 351-379
 *   sph_octree_build,     <- build_octree(positions) / range_query(tree, center,
 *   sph_octree_query         radius, workspace, exclude)     octree.py:306-379
 *   sph_nfw_positions_device: the clustered inputs of BASELINE configs 2-5
 *                           (the reference has no such generator; it follows
 *                           the UniformBox counter pattern, workload.py:42-84)
 *   sph_density_pass_multi <- compute_density_pass with the work split over
 *                            devices (SURVEY 8b n_gpus; items_per_worker per
 *                            device, density.py:407-409)
 *   sph_density_pass_device, sph_ctx_*, sph_last_error, sph_fp32_peak,
 *   sph_device_count      : device-resident form of the pass, context and
 *                           diagnostics (no reference counterpart)
 *   sph_morton_keys_device, sph_bbox_device, sph_decomp_*_device
 *                         : multi-GPU domain decomposition helpers
 *                           (paper_1612_06090_b200/distributed.py); the
 *                           reference runs in one shared-memory process
 *                           (scheduler.py), so they replace nothing
 * Status codes map to the reference's exceptions (density.py:69-74, 375-379,
 * 353-357; ValueError for invalid arguments, density.py:297-301).
 */
#ifndef SPH_B200_H
#define SPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPH_OK 0
#define SPH_NOT_CONVERGED 1 /* -> ConvergenceError(f"{unconverged} of {n} particles still flagged after {max_iterations} iterations") */
#define SPH_DEGENERATE 2    /* -> DegenerateWorkloadError (K-th neighbour at zero distance; bad_index) */
#define SPH_INVALID 3       /* -> ValueError */
#define SPH_CUDA_ERROR 4    /* -> RuntimeError(sph_last_error(ctx)) */
#define SPH_UNSUPPORTED 5   /* -> RuntimeError: input outside what this build handles (message in sph_last_error) */

#define SPH_PRECISION_F64 0 /* positions are float64 */
#define SPH_PRECISION_F32 1 /* positions are float32 (the fp32 configs); results stay bit-exact
                               against the fp64 reference on the widened values */
#define SPH_PRECISION_AUTO 2 /* positions are float64; the fp32 search kernels are used when every
                                coordinate is exactly fp32-representable (densities still summed in fp64) */

#define SPH_MAX_TODO 128

typedef struct sph_ctx sph_ctx;

typedef struct {
    int64_t n;              /* particle count (>= 1) */
    int32_t k;              /* k_neighbors (DesNumNgb), >= 1 */
    int32_t max_iterations; /* reference todo-loop budget (density.py:54) */
    int32_t precision;      /* SPH_PRECISION_* : element type of x/y/z */
    int32_t periodic;       /* 0: open boundaries (the reference); 1: periodic cube [0, box)^3 */
    double box;             /* periodic box side (ignored when periodic == 0) */
    int32_t kernel;         /* 0: Wendland C6 (the reference, kernel.py); 1: M4 cubic spline (extension) */
    int32_t reserved;
    int64_t n_targets;      /* 0: every particle is a target.  Otherwise particles [0, n_targets) are
                               targets and [n_targets, n) are ghosts (neighbour candidates only, e.g.
                               the halo layer of a domain-decomposed run); h / rho / flags then hold
                               n_targets entries */
} sph_params;

typedef struct {
    int32_t iterations;                 /* PassStats.iteration_count */
    int32_t n_todo;                     /* valid entries of todo_sizes */
    int64_t todo_sizes[SPH_MAX_TODO];   /* PassStats.todo_sizes (reference growth-only trace): the
                                           first min(iterations, SPH_MAX_TODO) rounds (h grows by 2^(1/3)
                                           per round, so round 128 is h0 * 2^42) */
    double t_stage_ms[8];               /* 0 h2d, 1 tree, 2 search, 3 select, 4 density, 5 finalize, 6 d2h, 7 total */
    int64_t pair_tests;                 /* target x candidate distance evaluations, all kernels */
    int64_t accepted_pairs;             /* pairs inside support in the density kernel */
    int64_t search_pair_tests;          /* pair tests of the search (histogram) kernel only */
    int64_t bad_index;                  /* first degenerate particle (original index) or -1 */
    int64_t unconverged;                /* particles still flagged after max_iterations */
    int32_t gpu_launches;               /* kernels launched by this call */
    int32_t search_rounds;              /* histogram rounds (1 + retries) */
    int32_t select_rounds;              /* band rounds */
    int32_t n_nodes;                    /* search-tree nodes */
    double t_kernel_ms[4];              /* device time of: 0 search, 1 select, 2 density, 3 tree build */
    double t_known_ms;                  /* device time of the known-radius kernel (inside t_kernel_ms[0]) */
    int64_t known_fallbacks;            /* targets it left to the general kernel (-1: it did not run) */
} sph_stats;

/* context: owns a CUDA stream and device buffers, grown on demand and
 * reused across calls (the analogue of density.py:264-283 _WorkerScratch) */
int sph_ctx_create(sph_ctx **out, int device);
void sph_ctx_destroy(sph_ctx *ctx);
const char *sph_last_error(const sph_ctx *ctx);
int sph_device_count(void);
/* the context's CUDA stream (a cudaStream_t as an opaque pointer), so a
 * caller can time the pass with its own events on the launching stream */
void *sph_ctx_stream(sph_ctx *ctx);

/*
 * Full pass on HOST buffers.  Each array is addressed as base + i * stride
 * (bytes), so the reference's packed records (stride 224) and plain SoA
 * arrays (stride = element size) are both accepted:
 *   x, y, z  : positions, element type per params->precision (read)
 *   mass     : float64 (read)
 *   h        : float64 smoothing_length: in = initial h (drives the todo
 *              trace only), out = converged h (K-th neighbour distance)
 *   rho      : float64 density out
 *   flags    : uint8 needs_recompute out (0 on success)
 * Synchronous; host pointers are not retained.
 */
int sph_density_pass(sph_ctx *ctx, const sph_params *params,
                     const void *x, const void *y, const void *z, int64_t pos_stride,
                     const double *mass, int64_t mass_stride,
                     double *h, int64_t h_stride,
                     double *rho, int64_t rho_stride,
                     uint8_t *flags, int64_t flags_stride,
                     sph_stats *stats);

/*
 * Multi-device pass (SURVEY 8b n_gpus / device mask; PassStats.items_per_worker
 * of shape (iterations, devices), density.py:407-409): the call of
 * sph_density_pass over n_ctx contexts, one per device slot (contexts from
 * sph_ctx_create; a device may appear more than once, each slot with its own
 * context).  Every device receives all positions, orders them and builds the
 * search tree; device d takes the targets of its slice [n d / n_ctx,
 * n (d + 1) / n_ctx) of the sorted (octree key) order -- contiguous key
 * ranges, so its targets are spatially compact -- and its results are
 * scattered into the caller's arrays by original index.  The devices run
 * concurrently (one host thread each); no collective is needed: the only
 * exchange is the host scatter of the results.  stats: n_ctx + 1 entries (one
 * per slot, then the merged pass: todo_sizes summed, times the max).  Errors as
 * sph_density_pass, message in sph_last_error(ctxs[0]); n_targets must be 0.
 */
int sph_density_pass_multi(sph_ctx *const *ctxs, int32_t n_ctx, const sph_params *params,
                           const void *x, const void *y, const void *z, int64_t pos_stride,
                           const double *mass, int64_t mass_stride,
                           double *h, int64_t h_stride,
                           double *rho, int64_t rho_stride,
                           uint8_t *flags, int64_t flags_stride,
                           sph_stats *stats);

/* Same pass on DEVICE-resident contiguous arrays (inputs already in HBM). */
int sph_density_pass_device(sph_ctx *ctx, const sph_params *params,
                            const void *d_x, const void *d_y, const void *d_z,
                            const double *d_mass, double *d_h, double *d_rho,
                            uint8_t *d_flags, sph_stats *stats);

/* 63-bit x-major octant-path keys of device-resident positions from a given
 * root cube (centre[3], half): the key the ordering sorts by (octree.py:93-104
 * descent, 21 levels), here for the key-range domain decomposition
 * (distributed ownership; no reference counterpart: the reference is one
 * shared-memory process).  Enqueued on the context's stream (sph_ctx_stream). */
int sph_morton_keys_device(sph_ctx *ctx, int32_t precision, int64_t n, const void *d_x, const void *d_y,
                           const void *d_z, const double *centre, double half, uint64_t *d_keys);

/* Domain-decomposition helpers (device pointers, the context's stream):
 *  pack_rows    : rows[i] = (x, y, z, m, h0, gid bits, key >> 32, key & 0xffffffff)
 *                 (gid as its int64 bit pattern, exact for any id)
 *                 of particle order[i], 8 doubles per record (the all-to-all payload)
 *  gather_rows  : dst row i = src row idx[i], width doubles per row
 *  row_keys     : keys of packed records (columns 6, 7) back to int64
 *  level_bounds : per particle (key-sorted) an upper bound of its K-th
 *                 neighbour distance: sqrt(3) * side of the deepest key cube
 *                 holding it and >= K others (INFINITY when n <= K)
 *  window_bounds: tightens bound[p] (in place, min) by the farthest of the K
 *                 others in each of three windows of K+1 key-consecutive
 *                 records around p (any K others bound the K-th distance)
 *  ghost_mask   : mask[i] |= 1 << rank(f) for every particle i of my groups
 *                 (descriptors gdesc, records rows) within foreign group f's
 *                 margin of its box (min-image when periodic): the ghosts
 *  group_boxes  : per group [start, start + count) of records: tight box of
 *                 columns 0-2 and the largest bound -> 7 doubles */
int sph_decomp_pack_rows_device(sph_ctx *ctx, int32_t precision, int64_t n, const int64_t *d_order,
                                const void *d_x, const void *d_y, const void *d_z, const double *d_mass,
                                const double *d_h0, const int64_t *d_gid, const int64_t *d_keys, double *d_rows);
int sph_decomp_gather_rows_device(sph_ctx *ctx, int64_t n, int32_t width, const int64_t *d_idx,
                                  const double *d_src, double *d_dst);
int sph_decomp_row_keys_device(sph_ctx *ctx, int64_t n, const double *d_rows, int64_t *d_keys);
int sph_decomp_level_bounds_device(sph_ctx *ctx, int64_t n, int32_t k, const int64_t *d_keys_sorted, double half,
                                   double *d_bound);
int sph_decomp_window_bounds_device(sph_ctx *ctx, int64_t n, int32_t k, int32_t width, const double *d_rows,
                                    double max_abs_coord, double *d_bound);
/* per-axis min / max of device-resident positions -> d_out[0..2] = lo,
 * d_out[3..5] = hi (fp64, device pointer), on the context's stream */
int sph_bbox_device(sph_ctx *ctx, int32_t precision, int64_t n, const void *d_x, const void *d_y, const void *d_z,
                    double *d_out);
int sph_decomp_ghost_mask_device(sph_ctx *ctx, int64_t n_groups, const double *d_gdesc, const int64_t *d_gstart,
                                 const int64_t *d_gcount, int32_t width, const double *d_rows, int64_t n_foreign,
                                 const double *d_fdesc, const int32_t *d_frank, int32_t periodic, double box,
                                 uint32_t *d_mask);
int sph_decomp_group_boxes_device(sph_ctx *ctx, int64_t n_groups, const int64_t *d_starts, const int64_t *d_counts,
                                  int32_t width, const double *d_rows, const double *d_bound, double *d_out);

/* The reference's tree object and its query around an arbitrary centre
 * (build_octree + range_query, octree.py:306-379).  sph_octree_build orders
 * the positions (host pointers, per precision) and builds the search tree,
 * kept in the context until its next build or pass.  sph_octree_query answers
 * m queries: for query q every particle j (original index) with
 * (dx*dx + dy*dy) + dz*dz <= radii[q]^2 in unfused fp64, dx = x_j - c_x
 * (octree.py:211-214), except exclude[q] (exclude may be NULL; -1 = none);
 * CSR offsets_out[m + 1], idx_out / d2_out sorted by index within a query.
 * When the total exceeds cap, *total_out is set, nothing else is written and
 * SPH_INVALID is returned (call again with a larger buffer: the reference's
 * QueryWorkspace.grow). */
int sph_octree_build(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z);
int sph_octree_query(sph_ctx *ctx, int64_t m, const double *centers, const double *radii, const int64_t *exclude,
                     int64_t cap, int64_t *offsets_out, int64_t *idx_out, double *d2_out, int64_t *total_out);

/* Octree particle_perm (leaf capacity 8), bit-exact with the reference,
 * depth up to 48 (runs of identical 63-bit keys are subdivided further).
 * Host pointers; positions per precision (contiguous). */
int sph_sort_perm(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y,
                  const void *z, int64_t *perm_out);
/* The same for any leaf capacity in [1, 32] (build_octree(positions,
 * leaf_capacity).particle_perm, octree.py:306-317); trees deeper than the 21
 * levels of the key are followed to MAX_TREE_DEPTH = 48 (octree.py:31). */
int sph_sort_perm_ex(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y,
                     const void *z, int32_t leaf_capacity, int64_t *perm_out);

/* Fixed-h neighbour counts #{j != i : (dx*dx + dy*dy) + dz*dz <= h_i*h_i}
 * in unfused fp64, bit-exact.  periodic/box as in sph_params. */
int sph_neighbor_counts(sph_ctx *ctx, int32_t precision, int32_t periodic, double box,
                        int64_t n, const void *x, const void *y, const void *z,
                        const double *h, int32_t *counts_out, sph_stats *stats);

/* The reference's range_query(tree, pos_i, h_i, exclude=i) (octree.py:179-227,
 * 351-379) for every particle i at once, open boundary: the other particles
 * with (dx*dx + dy*dy) + dz*dz <= h_i*h_i in unfused fp64, as CSR in the
 * caller's particle order.  offsets (n + 1, host) = the exclusive prefix sum
 * of sph_neighbor_counts for the same h; idx_out / d2_out (offsets[n] each,
 * host) receive each list sorted by index (the reference lists candidates in
 * tree order: the same sets).  SPH_INVALID if the offsets do not match. */
int sph_range_query(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z,
                    const double *h, const int64_t *offsets, int64_t *idx_out, double *d2_out);

/* measured FP32-pipe FFMA issue rate of the context's device (FFMA/s): the
 * roofline denominator of the neighbour kernels */
double sph_fp32_peak(sph_ctx *ctx);

/* FNV-1a-64 over a byte buffer (host; the reference checksum64) */
uint64_t sph_fnv1a64(const uint8_t *data, size_t len);

/* On-device input path: the reference's UniformBox positions
 * generated straight into device SoA arrays (fp64), bit-exact with
 * generate(WorkloadSpec(UNIFORM_BOX, n, seed)) (workload.py:77-84, splitmix64
 * draws workload.py:42-60): draw t = 3i + axis of particle i is
 * mix(seed + (t+1) * 0x9E3779B97F4A7C15) >> 11, times 2^-53, times box
 * (values at box clamp to nextafter(box, 0)).  Runs on the context's stream. */
int sph_uniform_box_device(sph_ctx *ctx, int64_t n, uint64_t seed, double box, double *d_x, double *d_y,
                           double *d_z);

/* On-device clustered generator (BASELINE configs 2-5):
 * particles [halo_start[h], halo_start[h+1]) of halo h follow an NFW profile
 * (concentration c, truncated at x_max = r / r_s) around its centre, the rest
 * [halo_start[n_halos], n) are uniform in the box.  d_halo holds 5 doubles
 * per halo: centre x, y, z, r_vir, velocity sigma.  Every draw is the
 * splitmix64 counter stream of sph_uniform_box_device (draw 8i + j for
 * particle i), so the set is a pure function of the seed and the halo table.
 * Positions wrap into [0, box) and are written as fp32; d_vel (3 floats per
 * particle, may be NULL) receives Gaussian velocities (never read by the
 * pass).  Device pointers, the context's stream. */
int sph_nfw_positions_device(sph_ctx *ctx, int64_t n, int64_t n_halos, const int64_t *d_halo_start,
                             const double *d_halo, double concentration, double x_max, uint64_t seed, double box,
                             float *d_x, float *d_y, float *d_z, float *d_vel);

#ifdef __cplusplus
}
#endif
#endif /* SPH_B200_H */
