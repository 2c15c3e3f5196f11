// sph_internal.cuh -- shared device helpers and host-side launch interfaces
// of the B200 SPH density pass.  See DESIGN.md for the data layout.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sph {

constexpr int kMaxLevel = 21;        // 63-bit Morton keys: 21 octree levels
constexpr int kLeafCap = 8;          // reference leaf capacity (octree.py:30)
constexpr int kMaxLeafCap = 32;      // largest leaf capacity particle_perm takes (the key-window halo)
#ifndef SPH_CELL_CAP
#define SPH_CELL_CAP 32
#endif
constexpr int kCellCap = SPH_CELL_CAP;  // search cell capacity (<= 32: one warp of candidates)
constexpr double kGrowth = 1.2599210498948732;  // 2.0 ** (1.0 / 3.0), density.py:53
constexpr double kWc6Norm = 1365.0 / (64.0 * 3.14159265358979323846);  // kernel.py:17
constexpr double kM4Norm = 8.0 / 3.14159265358979323846;              // M4 (extension)

// status bytes per target (sorted position)
enum : uint8_t { ST_NEED_HIST = 0, ST_NEED_BAND = 1, ST_DONE = 2, ST_UNREACHABLE = 3, ST_FAILED = 4, ST_GHOST = 5,
                 ST_LEGACY = 6, ST_FINAL = 8 };

// root cube of the reference octree (octree.py:324-336) + validation flags
struct RootInfo {
  double lo[3], hi[3];
  double c[3];
  double half;
  double pad;
  double max_abs;
  int nonfinite;
  int not_f32;   // some coordinate is not exactly representable in fp32
};

// ordered-int image of a double for atomicMin/atomicMax
__device__ __forceinline__ unsigned long long dbl_to_ord(double d) {
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_to_dbl(unsigned long long o) {
  unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
  return __longlong_as_double((long long)b);
}

// common prefix length (bits) of two 63-bit keys held in the low 63 bits
__device__ __forceinline__ int key_cpl(unsigned long long a, unsigned long long b) {
  return __clzll(a ^ b) - 1;  // 63 when equal
}
__host__ __device__ __forceinline__ unsigned long long key_prefix(unsigned long long key, int level) {
  return level == 0 ? 0ull : (key >> (63 - 3 * level));
}

// exact reference distance: ddx = x_j - q_x; d2 = (ddx*ddx + ddy*ddy) + ddz*ddz,
// every operation rounded on its own (octree.py:211-214, no contraction)
__device__ __forceinline__ double exact_d2(double dx, double dy, double dz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// Wendland C6 unit profile (kernel.py:30-36), fp64 op-for-op
__device__ __forceinline__ double wc6_profile(double q) {
  double u = __dsub_rn(1.0, q);
  double u2 = __dmul_rn(u, u);
  double u4 = __dmul_rn(u2, u2);
  double poly = __dadd_rn(1.0, __dmul_rn(q, __dadd_rn(8.0, __dmul_rn(q, __dadd_rn(25.0, __dmul_rn(32.0, q))))));
  return __dmul_rn(__dmul_rn(u4, u4), poly);
}
// _w_lowered(r, h) (kernel.py:39-45) given the precomputed C/(h*h*h)
__device__ __forceinline__ double wc6_lowered(double r, double h, double norm_h3) {
  double q = __ddiv_rn(r, h);
  return q < 1.0 ? __dmul_rn(norm_h3, wc6_profile(q)) : 0.0;
}
__device__ __forceinline__ float wc6_profile_f(float q) {
  float u = 1.0f - q;
  float u2 = u * u;
  float u4 = u2 * u2;
  return (u4 * u4) * fmaf(q, fmaf(q, fmaf(32.0f, q, 25.0f), 8.0f), 1.0f);
}
// M4 cubic spline with compact support h (extension; no reference oracle)
__device__ __forceinline__ double m4_profile(double q) {
  if (q < 0.5) return 1.0 - 6.0 * q * q + 6.0 * q * q * q;
  double t = 1.0 - q;
  return q < 1.0 ? 2.0 * t * t * t : 0.0;
}
__device__ __forceinline__ float m4_profile_f(float q) {
  if (q < 0.5f) return 1.0f - 6.0f * q * q + 6.0f * q * q * q;
  float t = 1.0f - q;
  return q < 1.0f ? 2.0f * t * t * t : 0.0f;
}

// search-tree node (pre-order, skip pointers).  lo.w = skip (int bits),
// hi.w = first sorted position (int bits).  A node is a cell iff skip == k+1.
struct TreeView {
  const float4 *nlo;
  const float4 *nhi;
  const int *nsize;   // particles in the node's subtree
  const float4 *crec;  // per-target traversal: 8 child records {box lo, code} {box hi, end} per node (+ virtual root)
  const int4 *anc4;    // first four ancestors of each node
  const int *cellof;   // cell holding each sorted particle
  int root_start;      // node whose children the unshifted-fallback / shifted walks expand (0, or the virtual node)
  int n_nodes;
};

// per-call device workspace handed to the kernels
struct PassArgs {
  int n;
  int k;
  int kernel_kind;
  const uint32_t *list;     // target list (sorted positions); nullptr = identity
  const int *list_count;    // device-side list length
  int static_count;         // used when list == nullptr
  TreeView tree;
  const void *pos;          // float4 (fp32 path) or double[4] (fp64 path) per sorted position
  const double *mass64;     // fp64 masses in sorted order (fp32 path with fp64 density sums)
  int dens64;               // fp32 path: evaluate accepted pairs in fp64 like the reference
  float *radius;            // per target search radius (histogram pass)
  double *t_lo, *t_hi;      // per target bracket of d2_K (band pass)
  double *d2k;              // result: K-th neighbour squared distance
  double *rho;              // result: density (sorted order)
  const double *hfix;       // fixed-h counting input (sorted order)
  int32_t *counts;          // fixed-h counting output (sorted order)
  uint8_t *state;           // per target status
  int *work_counter;        // persistent-kernel work cursor
  unsigned long long *stats;  // [0] pair tests, [1] accepted pairs
  int periodic;
  double box;
  float box_lo;             // box - (float)box: the fp32 image arithmetic's second word
  float rmax;               // largest meaningful search radius
  unsigned long long *dbg;  // optional per-bundle diagnostics (4 words per bundle) or nullptr
  float sub_d;              // task grouping: Chebyshev radius in units of the leader's radius
  int2 *tasks;              // (offset into members, count) per task
  uint32_t *members;        // task member targets (sorted positions)
  int *task_count;          // device task counter
  int *member_cursor;       // device member allocation cursor
  int shortcut;             // bit per mode: count whole cells from their box when possible
  int *ncount;              // per target: collect-instance marker (0x7fffffff: list overflowed in the main kernel)
  int tshrink;              // per-target kernel: shrink after every K >> tshrink new candidates
  int static_sched;         // per-target kernel: strided static assignment (0: the atomic counter; always 0)
  int tchunk;               // per-target kernel: consecutive targets per work grab (identity target order)
  const unsigned *clist;    // per-target kernel: neighbour-cell lists per cell (child-record indices into tree.crec), clcap each
  const int *clen;          // list length per cell (-1: none)
  const float *crad2;       // squared radius a cell's list covers
  const int *cellidx;       // cell index of each node (-1: internal)
  const int *cnear;         // records of each list within near_frac * D of the cell box (the rest at its back)
  float near_frac2;         // near_frac^2
  int clcap;
  uint32_t *fb_list;        // per-target kernel: targets left for the collect instance (+ counter)
  int *fb_count;
  const float4 *posj;       // sorted (x, y, z, sorted index bits) per position (fp32 path; k_lane stages it)
  int *kn_counters;         // k_lane hand-over reasons (see sph_lane.cu) or nullptr
};

// ---- launchers (sph_tree.cu) ----
struct TreeBuffers {
  // sort / ordering
  unsigned long long *keys_in, *keys;   // keys (unsorted / sorted)
  uint32_t *idx_in, *idx;               // original indices (unsorted / key-sorted)
  uint32_t *perm;                       // final order: sorted position -> original index
  uint8_t *lvl8, *lvl32;
  int *deep_count;
  uint32_t *deep_list;
  void *deep_segs;                      // k_deep's depth-first segment stacks (deep_segs_bytes())
  int leaf_cap;                         // reference leaf capacity of the ordering (8 for the pass)
  int *err_flag;
  // search tree
  int *noff;                            // n+1 node offsets per position
  int *n_nodes_dev;
  float4 *nlo, *nhi;
  int *nsize;                           // particles per node subtree
  float *r0;                            // per sorted position initial radius
  void *pos_sorted;                     // float4 or double[4] per position
  float4 *posj;                         // fp32 path: (x, y, z, sorted index bits) per position (or nullptr)
  double *mass_sorted;                  // fp64 masses per position
  void *cub_temp;
  size_t cub_temp_bytes;
  RootInfo *root;
  unsigned long long *bbox_ord;         // 6 ordered-int accumulators
  float r0_scale;                       // initial radius = r0_scale * density estimate
  float c0_scale;                       // ... capped by c0_scale * the cell's own tight-box estimate
  int emit_r0;                          // 0: R0 comes from k_r0 (per-target path) instead of k_node_emit
  int *node_p;                          // per node: its first sorted position (per-node emission, emit_r0 == 0)
  cudaEvent_t mass_ready;               // optional: wait for it before the masses are read
};

int tree_build(cudaStream_t s, TreeBuffers &tb, int n, int precision_in, int compute_f32,
               const void *x, const void *y, const void *z, const double *mass,
               int k, int *launches);
int tree_build_search(cudaStream_t s, TreeBuffers &tb, int n, int precision_in, int compute_f32,
                      const void *x, const void *y, const void *z, const double *mass, int k, float rmax,
                      int *launches);

void launch_bbox(cudaStream_t s, int n, int precision_in, const void *x, const void *y,
                 const void *z, unsigned long long *ord, RootInfo *root, int *launches);

size_t cub_temp_needed(int n);
// stable radix sort of the 63-bit keys with their indices (sph_sort.cu): a -> b
size_t radix_sort_temp_bytes(int n);
// single-pass exclusive scan / order-preserving select by state (sph_scan.cu)
size_t scan_temp_bytes(int n);
void scan_exclusive_i32(cudaStream_t s, const int *in, int *out, int n, void *temp);
void select_state(cudaStream_t s, const uint32_t *list_in, int n_in, const uint8_t *state, uint8_t want,
                  uint32_t *list_out, int *count_out, void *temp);
void radix_sort_pairs(cudaStream_t s, int n, unsigned long long *keys_a, uint32_t *vals_a, unsigned long long *keys_b,
                      uint32_t *vals_b, void *temp);
size_t deep_segs_bytes();
// batched range query lists (sph_range.cu)
int range_fill(cudaStream_t s, int f32, int n, const uint32_t *perm, const void *pos_sorted, const double *h_sorted,
               const TreeView &tree, const int64_t *offsets, int64_t total, int64_t *idx_out, double *d2_out,
               int *err, void *temp, size_t temp_bytes, int64_t *idx_tmp, double *d2_tmp, int num_sms);
size_t range_sort_temp(int n, int64_t total);
int range_points(cudaStream_t s, int f32, int count_only, int64_t m, const double *centers, const double *radii,
                 const int64_t *excl, const uint32_t *perm, const void *pos_sorted, const TreeView &tree,
                 const int64_t *offsets, int64_t *counts, int64_t *idx_tmp, double *d2_tmp, int *err, int num_sms);
int segmented_sort_pairs(cudaStream_t s, int64_t m, int64_t total, const int64_t *offsets, const int64_t *idx_in,
                         int64_t *idx_out, const double *d2_in, double *d2_out, void *temp, size_t temp_bytes);
// domain decomposition helpers (sph_decomp.cu)
void launch_pack_rows(cudaStream_t s, int64_t n, int precision_in, const int64_t *order, const void *x,
                      const void *y, const void *z, const double *m, const double *h0, const int64_t *gid,
                      const int64_t *keys, double *rows);
void launch_gather_rows(cudaStream_t s, int64_t n, int width, const int64_t *idx, const double *src, double *dst);
void launch_row_keys(cudaStream_t s, int64_t n, const double *rows, int64_t *keys);
void launch_level_bounds(cudaStream_t s, int64_t n, int k, const int64_t *keys, double side0, double *bound);
void launch_window_bounds(cudaStream_t s, int64_t n, int k, int width, const double *rows, double abs_slack,
                          double *bound);
void launch_ghost_mask(cudaStream_t s, int64_t ng, const double *gdesc, const int64_t *gstart, const int64_t *gcount,
                       int width, const double *rows, int64_t nf, const double *fdesc, const int32_t *frank,
                       int periodic, double box, uint32_t *mask, double *scratch);
void launch_group_boxes(cudaStream_t s, int64_t ng, const int64_t *starts, const int64_t *counts, int width,
                        const double *rows, const double *bound, double *out);
// 63-bit keys from a given root cube (domain decomposition)
void launch_keys_at(cudaStream_t s, int n, int precision_in, const void *x, const void *y, const void *z,
                    const double *centre, double half, unsigned long long *keys);

// ---- launchers (sph_pass.cu) ----
enum PassMode { MODE_HIST = 0, MODE_BAND = 1, MODE_DENS = 2, MODE_COUNT = 3 };
void launch_pass(cudaStream_t s, int mode, int f32, const PassArgs &a, int count, uint8_t want, int num_sms);
// one lane per target over bundles of 32 consecutive sorted targets (sph_lane.cu)
int lane_list_cap(int k);
bool lane_supported(int k);
void launch_lane(cudaStream_t s, const PassArgs &a, int lcap, float rscale, float exc, int max_stream, int num_sms,
                 const float *cal = nullptr, float calq = 0.85f);
// fused per-target search + select + density (sph_warp.cu)
int target_list_cap(int k);
void launch_target(cudaStream_t s, int f32, const PassArgs &a, int cap, int *fallbacks, int num_sms,
                   bool collect = false);
void launch_cell_index(cudaStream_t s, const float4 *nlo, int n_nodes, int *cellidx, int *cellnode, int *ncells);
void launch_cell_index_dev(cudaStream_t s, const float4 *nlo, const int *n_nodes_dev, int max_nodes, int *cellidx,
                           int *cellnode, int *ncells);
void launch_cell_lists(cudaStream_t s, const PassArgs &a, const int *cellnode, const int *ncells, int cap,
                       unsigned *clist, int *clen, float *crad2, int *cnear, float near_frac, float d_pct,
                       int num_sms, int ncell_host = -1);
void launch_kids(cudaStream_t s, const float4 *nlo, const float4 *nhi, int n_nodes, int n, float4 *crec, int *parent,
                 int4 *anc4, int *cellof);
// per-cell initial search radius from the node sizes and the parent chain
void launch_r0(cudaStream_t s, const float4 *nlo, const float4 *nhi, const int *nsize, const int *parent, int n_nodes,
               int n, int k, float r0_scale, float rmax, float root_side, float *r0);
void launch_select(cudaStream_t s, const uint32_t *list_in, int n_in, const uint8_t *state, uint8_t want,
                   uint32_t *list_out, int *count_out, void *temp, size_t temp_bytes);
size_t select_temp_needed(int n);
// clustered workload generator (sph_workload.cu)
void launch_nfw_positions(cudaStream_t s, int64_t n, int64_t n_halos, const int64_t *start, const double *halo,
                          double conc, double x_max, uint64_t seed, double box, float *x, float *y, float *z,
                          float *vel);

}  // namespace sph
