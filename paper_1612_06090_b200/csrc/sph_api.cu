// sph_api.cu -- the C ABI (include/sph_b200.h): context, buffers, and the
// orchestration of one density pass.
//
// Pass structure (all on one stream):
//   bbox -> [sync: validate] -> keys -> radix sort -> leaf levels -> perm ->
//   sorted SoA -> search tree -> [sync: node count]
//   HIST over all targets; while any target has < K candidates inside its
//   radius: compact those (order-preserving) and HIST again       (search)
//   BAND over all; while any bracket is overfull: compact, BAND again (select)
//   DENS over all                                                 (interact)
//   finalize: h = sqrt(d2_K), the reference's todo trace from h0 and d2_K,
//   scatter to original order                                    (write-back)
#include "sph_internal.cuh"
#include "../../include/sph_b200.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: host ranges around the pass stages (nsys / ncu --nvtx)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

using namespace sph;

namespace {

template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t count) {
    if (count <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t c = std::max<size_t>(count, 1);
    cudaError_t e = cudaMalloc(&p, c * sizeof(T));
    if (e == cudaSuccess) cap = c;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct sph_ctx {
  cudaEvent_t kev[2 * 64];
  int n_kev = 0;
  int kev_mode[64];
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;
  cudaEvent_t ev[12];
  // inputs / outputs for the host-pointer entry points
  DevBuf<double> in_x, in_y, in_z, in_m, io_h, out_rho;
  DevBuf<uint8_t> out_flags;
  // ordering
  DevBuf<unsigned long long> keys_in, keys, bbox_ord;
  DevBuf<uint32_t> idx_in, idx, perm, deep_list, iota, list;
  DevBuf<unsigned char> deep_segs;
  DevBuf<uint8_t> lvl8, lvl32, state;
  DevBuf<int> ints;  // [0] deep_count [1] err_flag [2] list_count [3] work_counter [4] task count [5] member cursor [6..] rounds hist
  DevBuf<int2> tasks;
  DevBuf<uint32_t> members;
  DevBuf<int> noff;
  DevBuf<int> node_p;
  DevBuf<float4> nlo, nhi;
  DevBuf<int> nsize;
  DevBuf<float> r0;
  DevBuf<unsigned char> pos_sorted, cub_temp;
  DevBuf<RootInfo> root;
  DevBuf<double> t_lo, t_hi, d2k, rho_s, hfix, mass_s;
  DevBuf<int32_t> counts_s, counts_o;
  DevBuf<unsigned long long> stats;  // [0] tests [1] accepted [2] bad index (ord)
  DevBuf<unsigned long long> dbg;    // SPH_DEBUG=1: per-bundle diagnostics
  bool debug = false;     // SPH_DEBUG=1: fallback counters on stderr
  int seed_stride = 12;   // SPH_SEED: seed stride of the per-target pass (12 beat 6/8/16 on C1-C5, r01l; 0/1 = off)
  float seed_margin = 1.1f;  // SPH_SEEDM: non-seed radius = margin x the neighbouring seeds' h
  int known = 5;          // SPH_KNOWN: 5 seeds + lane kernel + per-target kernel for what it leaves (default), 0 seeds + per-target kernel for every other target
  float lane_margin = 1.15f;  // SPH_LANEM: lane kernel radius = this x the neighbouring seeds' h
  float lane_noseed = 1.0f;   // SPH_LANE_NOSEED: > 0: no dense seeds, lane radius = this x the calibrated tree estimate (0: seeds every seed_stride-th target)
  int lane_cal_stride = 256;  // SPH_LANE_CAL: calibration sample = every this-th sorted target
  float lane_cal_q = 0.92f;   // SPH_LANE_CALQ: quantile of h / R0 (per class of R0) over the sample that scales the tree estimate
  int lane_stream = 2400;     // SPH_LANE_STREAM: bundles streaming more candidates than this go to the per-target kernel
  float lane_exc = 2.0f;      // SPH_LANEX: lanes reaching beyond this x the bundle's median reach are left out (0: none)
  bool known_ran = false;
  cudaEvent_t kev_known[2];
  DevBuf<uint32_t> kn_list;   // targets the known-radius kernel leaves to the general kernel
  DevBuf<float4> posj;        // fp32 path: (x, y, z, sorted index bits) per sorted position
  DevBuf<double> dscratch;  // decomposition helpers: super boxes of the ghost marking
  DevBuf<int> ncell_dev;    // cells of the search tree (counted with the tree, read with n_nodes)
  DevBuf<uint32_t> tlist;   // compacted target positions (ghost-aware seeding)
  int last_ncell = -1;
  // multi-device pass: this device's targets are the sorted positions
  // [slice_lo, slice_hi) (slice_hi < 0: every target); outputs compacted,
  // with the original index of each in slice_orig
  int64_t slice_lo = 0, slice_hi = -1;
  DevBuf<int64_t> slice_orig;
  // the tree of the last sph_octree_build (-1: none; any other tree build on
  // this context invalidates it)
  int64_t octree_n = -1;
  int leaf_cap = 8;  // reference leaf capacity of the ordering (sph_sort_perm_ex; the pass uses 8)
  int octree_f32 = 0;
  PassArgs octree_args{};
  DevBuf<uint32_t> seeds;
  DevBuf<float> calbuf;   // 64 histogram words of log(h / R0), then the sampled targets' R0
  int collect_cap = 1024;  // SPH_CCAP: list capacity of the collect instance
  cudaStream_t stream2 = nullptr;  // side stream for host-to-device copies the first kernels do not need
  cudaEvent_t ev_side_start = nullptr, ev_mass = nullptr, ev_h = nullptr;
  cudaEvent_t in_mass_ready = nullptr, in_h_ready = nullptr;  // set only during a host-API pass
  int cell_lists = 192;  // SPH_CLIST: neighbour-cell list capacity (0 = off)
  DevBuf<unsigned> clist;
  DevBuf<int> clen, cellidx, cellnode;
  DevBuf<float> crad2;
  DevBuf<int> cnear;
  float near_frac = 0.5f;   // SPH_NEARF: cell-list records beyond near_frac * D go to the list's back
  int tshrink = 1;       // SPH_TSHRINK (shrink after every K >> tshrink new candidates; 1 measured best on C2/C5)
  DevBuf<float4> crec;
  DevBuf<int4> anc4;
  DevBuf<int> parent, cellof;
  bool crec_ready = false;
  int tb_emit_r0 = 1;    // did the last tree build compute R0 (k_node_emit)?
  DevBuf<int> ncount;
  DevBuf<int> qints;
  float r0_scale = 1.15f;  // SPH_R0SCALE: tree-estimate radius scale (seeds)
  size_t cub_bytes = 0;
};

namespace {

constexpr int kIntsFixed = 6;
constexpr int kTB = 256;

int fail(sph_ctx *c, int code, const std::string &msg) {
  c->err = msg;
  return code;
}

int cuda_fail(sph_ctx *c, cudaError_t e, const char *where) {
  c->err = std::string(where) + ": " + cudaGetErrorString(e);
  cudaGetLastError();
  return SPH_CUDA_ERROR;
}

#define SPH_CK(call)                                   \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

// targets: original index < n_targets and sorted position in [lo, hi) (the
// slice of a multi-device pass); everything else is a ghost (candidate only)
__global__ void k_init_state(int n, int n_targets, const uint32_t *__restrict__ perm, uint8_t *__restrict__ state,
                             int lo, int hi) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) state[p] = ((int)perm[p] < n_targets && p >= lo && p < hi) ? ST_NEED_HIST : ST_GHOST;
}

__global__ void k_append_sgs(const int2 *tasks, const int *count, int4 *sgs, int base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *count) {
    const int2 t = tasks[i];
    sgs[base + i] = make_int4(t.x, t.y, -1, 0);
  }
}

__global__ void k_state_map(int n, uint8_t *state, uint8_t from, uint8_t to) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && state[i] == from) state[i] = to;
}

// calibration sample of the tree's radius estimate (the lane kernel without dense seeds): R0 of every
// sampled target saved before the per-target kernel overwrites it, then 64-bin histograms of log(h / R0)
// over [-1.5, 1.5), one per class of R0 (half octaves, 16 classes), in the first 1024 words
constexpr int kCalWords = 16 * 64;
__global__ void k_cal_save(int ns, const uint32_t *__restrict__ sample, const float *__restrict__ r0,
                           float *__restrict__ cal) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kCalWords) reinterpret_cast<int *>(cal)[i] = 0;
  if (i < ns) cal[kCalWords + i] = r0[sample[i]];
}
__global__ void k_cal_reduce(int ns, const uint32_t *__restrict__ sample, const uint8_t *__restrict__ state,
                             const double *__restrict__ d2k, float *__restrict__ cal) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const size_t p = sample[i];
  const double d = d2k[p];
  const float r = cal[kCalWords + i];
  if (state[p] == ST_FINAL && d > 0.0 && d < 1e300 && r > 0.f) {
    const float v = 0.5f * logf((float)d) - logf(r);
    const int b = min(max((int)((v + 1.5f) * (64.0f / 3.0f)), 0), 63);
    const int cls = (__float_as_int(r) >> 22) & 15;
    atomicAdd(reinterpret_cast<int *>(cal) + cls * 64 + b, 1);
  }
}

// seed targets for the per-target pass: every stride-th sorted position
__global__ void k_seed_list(int ns, int stride, uint32_t *seeds, int *count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *count = ns;
  if (i < ns) seeds[i] = (uint32_t)(i * stride);
}

// initial radius of the non-seed targets: margin x the larger converged h of
// the two seeds around them (their own estimate when neither seed converged)
// (only positions that are multiples of `only`: the next seed level)
__global__ void k_seed_radius(int n, int stride, int only, const uint8_t *__restrict__ state,
                              const double *__restrict__ d2k, float margin, float rmax, float *__restrict__ r0) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n || p % stride == 0 || p % only != 0 || state[p] != ST_NEED_HIST) return;
  const int s0 = p - p % stride, s1 = s0 + stride;
  double h = 0.0;
  if (state[s0] == ST_FINAL) h = d2k[s0];
  if (s1 < n && state[s1] == ST_FINAL) h = fmax(h, d2k[s1]);
  if (h > 0.0) r0[p] = fminf((float)sqrt(h) * margin, rmax);
}

// ghost-aware seeding (n_targets < n): seeds and radii along the compacted
// target order, so targets next to ghosts in sorted order still get seeds
__global__ void k_seed_list_from(int ns, int stride, const uint32_t *__restrict__ tlist, uint32_t *seeds,
                                 int *count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *count = ns;
  if (i < ns) seeds[i] = tlist[(size_t)i * stride];
}

__global__ void k_seed_radius_from(int nt, int stride, const uint32_t *__restrict__ tlist,
                                   const uint8_t *__restrict__ state, const double *__restrict__ d2k, float margin,
                                   float rmax, float *__restrict__ r0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nt || j % stride == 0) return;
  const int p = (int)tlist[j];
  if (state[p] != ST_NEED_HIST) return;
  const int j0 = j - j % stride, j1 = j0 + stride;
  const int s0 = (int)tlist[j0];
  double h = 0.0;
  if (state[s0] == ST_FINAL) h = d2k[s0];
  if (j1 < nt) {
    const int s1 = (int)tlist[j1];
    if (state[s1] == ST_FINAL) h = fmax(h, d2k[s1]);
  }
  if (h > 0.0) r0[p] = fminf((float)sqrt(h) * margin, rmax);
}

__global__ void k_iota(int n, uint32_t *a) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = (uint32_t)i;
}

// reference todo trace per particle: round j (1-based) searches with
// h_{j-1} = h0 * g^(j-1) (sequential fp64 products, density.py:227) and
// converges when count(h) >= K  <=>  d2_K <= h*h (octree.py:185, 215)
constexpr int kFinalizeSmemBins = 8192;  // 32 KB of round counters per block

__global__ void k_finalize(int n, int n_targets, const uint32_t *__restrict__ perm, const uint8_t *__restrict__ state,
                           const double *__restrict__ d2k, const double *__restrict__ rho_s,
                           const double *__restrict__ h0, int max_it, double *__restrict__ h_out,
                           double *__restrict__ rho_out, uint8_t *__restrict__ flags_out, int *rounds_hist,
                           unsigned long long *bad, int lo, int hi, int64_t *__restrict__ orig_out) {
  // per-block round histogram in shared memory when it fits (kFinalizeSmemBins),
  // otherwise straight into the global one
  extern __shared__ int sh_[];
  const bool local = max_it + 2 <= kFinalizeSmemBins;
  int *sh = local ? sh_ : rounds_hist;
  if (local) {
    for (int i = threadIdx.x; i < max_it + 2; i += blockDim.x) sh[i] = 0;
  }
  __syncthreads();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  // ghosts (original index >= n_targets, or outside the device's slice) are candidates only
  if (p < n && (int)perm[p] < n_targets && p >= lo && p < hi) {
    const uint32_t o = perm[p];
    // slice mode: outputs compacted by sorted position, with their original index
    const int64_t w = orig_out ? (int64_t)(p - lo) : (int64_t)o;
    if (orig_out) orig_out[w] = o;
    const uint8_t st = state[p];
    const bool fin = st == ST_DONE || st == ST_FINAL;
    const double d = fin ? d2k[p] : INFINITY;
    double hc = h0[o];
    int r = 1;
    bool conv = false;
    for (; r <= max_it; ++r) {
      if (d <= __dmul_rn(hc, hc)) { conv = true; break; }
      hc = __dmul_rn(hc, kGrowth);
    }
    const int bin = conv ? r : max_it + 1;
    atomicAdd(&sh[bin], 1);
    if (conv && d == 0.0) atomicMin(bad, (unsigned long long)o);
    h_out[w] = __dsqrt_rn(d);
    rho_out[w] = fin ? rho_s[p] : 0.0;
    flags_out[w] = conv ? 0 : 1;
  }
  __syncthreads();
  if (local) {
    for (int i = threadIdx.x; i < max_it + 2; i += blockDim.x)
      if (sh[i]) atomicAdd(&rounds_hist[i], sh[i]);
  }
}

template <typename T>
__global__ void k_gather_sorted(int n, const uint32_t *__restrict__ perm, const T *__restrict__ in, T *__restrict__ out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) out[p] = in[perm[p]];
}
template <typename T>
__global__ void k_scatter_orig(int n, const uint32_t *__restrict__ perm, const T *__restrict__ in, T *__restrict__ out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) out[perm[p]] = in[p];
}

inline int nblk(long long n, int t = kTB) { return (int)((n + t - 1) / t); }

// FP32-pipe throughput probe: 16 independent register-operand FFMA chains
// per thread (the roofline denominator for the neighbour kernels)
__global__ void __launch_bounds__(256) k_ffma_probe(float *out, int iters) {
  float a = 1.0f + threadIdx.x * 1e-7f, b = 1e-3f * (threadIdx.x & 7);
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

// scoped NVTX range (no-op unless a tool is attached)
struct Nvtx {
  explicit Nvtx(const char *name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx &) = delete;
  Nvtx &operator=(const Nvtx &) = delete;
};
// an NVTX range that may end before its scope does
struct NvtxSpan {
  bool on = true;
  explicit NvtxSpan(const char *name) { nvtxRangePushA(name); }
  void end() {
    if (on) nvtxRangePop();
    on = false;
  }
  ~NvtxSpan() { end(); }
};

struct Timer {
  sph_ctx *c;
  void mark(int i) { cudaEventRecord(c->ev[i], c->stream); }
  double ms(int a, int b) {
    float t = 0.f;
    cudaEventElapsedTime(&t, c->ev[a], c->ev[b]);
    return t;
  }
};

int ensure_common(sph_ctx *ctx, size_t n, int max_it) {
  SPH_CK(ctx->keys_in.ensure(n));
  SPH_CK(ctx->keys.ensure(n));
  SPH_CK(ctx->bbox_ord.ensure(6));
  SPH_CK(ctx->idx_in.ensure(n));
  SPH_CK(ctx->idx.ensure(n));
  SPH_CK(ctx->perm.ensure(n));
  SPH_CK(ctx->deep_list.ensure(n));
  SPH_CK(ctx->deep_segs.ensure(deep_segs_bytes()));
  SPH_CK(ctx->iota.ensure(n));
  SPH_CK(ctx->list.ensure(n));
  SPH_CK(ctx->lvl8.ensure(n));
  SPH_CK(ctx->lvl32.ensure(n));
  SPH_CK(ctx->state.ensure(n));
  SPH_CK(ctx->ints.ensure(kIntsFixed + (size_t)max_it + 2));
  SPH_CK(ctx->noff.ensure(n + 1));
  SPH_CK(ctx->nlo.ensure(2 * n + 64));
  SPH_CK(ctx->node_p.ensure(2 * n + 64));
  SPH_CK(ctx->nhi.ensure(2 * n + 64));
  SPH_CK(ctx->nsize.ensure(2 * n + 64));
  SPH_CK(ctx->r0.ensure(n));
  SPH_CK(ctx->pos_sorted.ensure(32 * n));
  SPH_CK(ctx->mass_s.ensure(n));
  SPH_CK(ctx->root.ensure(1));
  SPH_CK(ctx->stats.ensure(8));
  SPH_CK(ctx->tasks.ensure(n + 32));
  SPH_CK(ctx->members.ensure(n + 32));
  size_t need = std::max(cub_temp_needed((int)n), select_temp_needed((int)n));
  if (need > ctx->cub_temp.cap) SPH_CK(ctx->cub_temp.ensure(need));
  ctx->cub_bytes = ctx->cub_temp.cap;
  return SPH_OK;
}

TreeBuffers tree_buffers(sph_ctx *ctx) {
  TreeBuffers tb{};
  tb.leaf_cap = ctx->leaf_cap;
  tb.keys_in = ctx->keys_in.p;
  tb.keys = ctx->keys.p;
  tb.idx_in = ctx->idx_in.p;
  tb.idx = ctx->idx.p;
  tb.perm = ctx->perm.p;
  tb.lvl8 = ctx->lvl8.p;
  tb.lvl32 = ctx->lvl32.p;
  tb.deep_count = ctx->ints.p + 0;
  tb.deep_list = ctx->deep_list.p;
  tb.deep_segs = ctx->deep_segs.p;
  tb.err_flag = ctx->ints.p + 1;
  tb.noff = ctx->noff.p;
  tb.nlo = ctx->nlo.p;
  tb.nhi = ctx->nhi.p;
  tb.nsize = ctx->nsize.p;
  tb.r0 = ctx->r0.p;
  tb.pos_sorted = ctx->pos_sorted.p;
  tb.mass_sorted = ctx->mass_s.p;
  tb.cub_temp = ctx->cub_temp.p;
  tb.cub_temp_bytes = ctx->cub_bytes;
  tb.root = ctx->root.p;
  tb.bbox_ord = ctx->bbox_ord.p;
  tb.r0_scale = ctx->r0_scale;
  tb.c0_scale = 1e30f;
  tb.emit_r0 = 1;
  tb.node_p = ctx->node_p.p;
  return tb;
}

// bbox + validation; fills *root_h.  Synchronises once.
int stage_root(sph_ctx *ctx, int n, int precision, const void *x, const void *y, const void *z, RootInfo *root_h,
               int *launches) {
  launch_bbox(ctx->stream, n, precision == SPH_PRECISION_F32 ? 1 : 0, x, y, z, ctx->bbox_ord.p, ctx->root.p,
              launches);
  SPH_CK(cudaMemcpyAsync(root_h, ctx->root.p, sizeof(RootInfo), cudaMemcpyDeviceToHost, ctx->stream));
  SPH_CK(cudaStreamSynchronize(ctx->stream));
  SPH_CK(cudaGetLastError());
  if (root_h->nonfinite) return fail(ctx, SPH_INVALID, "positions must be finite");
  return SPH_OK;
}

// keys .. search tree; returns the node count through *n_nodes (one sync)
int stage_tree(sph_ctx *ctx, int n, int precision, int compute_f32, const void *x, const void *y, const void *z,
               const double *mass, int k, float rmax, int *n_nodes, int *launches, bool search_tree) {
  ctx->octree_n = -1;
  TreeBuffers tb = tree_buffers(ctx);
  tb.mass_ready = ctx->in_mass_ready;
  if (search_tree && compute_f32) {  // the known-radius kernel stages (x, y, z, index) records
    SPH_CK(ctx->posj.ensure(n));
    tb.posj = ctx->posj.p;
  }
  // the per-target path derives R0 from the node sizes (k_r0) instead
  tb.emit_r0 = 0;
  ctx->tb_emit_r0 = tb.emit_r0;
  const int in32 = precision == SPH_PRECISION_F32 ? 1 : 0;
  tree_build(ctx->stream, tb, n, in32, compute_f32, x, y, z, mass, k, launches);
  if (search_tree) tree_build_search(ctx->stream, tb, n, in32, compute_f32, x, y, z, mass, k, rmax, launches);
  int host[3] = {0, 0, -1};
  const bool index_cells = search_tree && ctx->cell_lists > 0;
  if (index_cells) {
    // cell index of every node, counted before the one sync of this stage
    // (the node count is still on the device: a grid over its upper bound)
    SPH_CK(ctx->cellidx.ensure(2 * (size_t)n + 64));
    SPH_CK(ctx->cellnode.ensure(2 * (size_t)n + 64));
    SPH_CK(ctx->ncell_dev.ensure(1));
    SPH_CK(cudaMemsetAsync(ctx->ncell_dev.p, 0, sizeof(int), ctx->stream));
    launch_cell_index_dev(ctx->stream, ctx->nlo.p, ctx->noff.p + n, 2 * n + 64, ctx->cellidx.p, ctx->cellnode.p,
                          ctx->ncell_dev.p);
    SPH_CK(cudaMemcpyAsync(&host[2], ctx->ncell_dev.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ++*launches;
  }
  SPH_CK(cudaMemcpyAsync(&host[0], ctx->ints.p + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if (search_tree)
    SPH_CK(cudaMemcpyAsync(&host[1], ctx->noff.p + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  SPH_CK(cudaStreamSynchronize(ctx->stream));
  ctx->last_ncell = host[2];
  SPH_CK(cudaGetLastError());
  *n_nodes = host[1];
  return SPH_OK;
}

float compute_rmax(const RootInfo &r, int periodic, double box) {
  if (periodic) return (float)(0.999 * box);
  double diag = 2.0 * r.half * 1.7320508075688772 * (1.0 + 1e-6) + 4.0 * r.pad;
  float f = (float)diag * 1.0001f;
  return f > 0.f ? f : 1e-30f;
}

PassArgs base_args(sph_ctx *ctx, int n, int k, int n_nodes, const sph_params *prm, float rmax) {
  PassArgs a{};
  a.n = n;
  a.k = k;
  a.kernel_kind = prm ? prm->kernel : 0;
  a.list = nullptr;
  a.list_count = ctx->ints.p + 2;
  a.static_count = n;
  a.tree.nlo = ctx->nlo.p;
  a.tree.nhi = ctx->nhi.p;
  a.tree.nsize = ctx->nsize.p;
  a.tree.n_nodes = n_nodes;
  a.pos = ctx->pos_sorted.p;
  a.mass64 = ctx->mass_s.p;
  // fp32 per-pair density sums stay within rel 1e-4 up to a few thousand terms; beyond that (K near n) the
  // terms are summed in fp64 like the fp64 / auto paths (tools/fuzz.py: K = 39,143 gave 1.2e-4 in fp32)
  a.dens64 = prm ? (prm->precision != SPH_PRECISION_F32 || k > 2048) : 0;
  a.radius = ctx->r0.p;
  a.t_lo = ctx->t_lo.p;
  a.t_hi = ctx->t_hi.p;
  a.d2k = ctx->d2k.p;
  a.rho = ctx->rho_s.p;
  a.hfix = ctx->hfix.p;
  a.counts = ctx->counts_s.p;
  a.state = ctx->state.p;
  a.work_counter = ctx->ints.p + 3;
  a.stats = ctx->stats.p;
  a.periodic = prm ? prm->periodic : 0;
  a.box = prm ? prm->box : 0.0;
  a.box_lo = (float)(a.box - (double)(float)a.box);  // second word of the fp32 image arithmetic
  a.rmax = rmax;
  a.dbg = nullptr;
  a.sub_d = 2.0f;  // walking fallback passes: task extent in units of the leader's radius
  a.tasks = ctx->tasks.p;
  a.members = ctx->members.p;
  a.task_count = ctx->ints.p + 4;
  a.member_cursor = ctx->ints.p + 5;
  a.shortcut = (1 << MODE_BAND) | (1 << MODE_COUNT);
  a.tshrink = ctx->tshrink;
  a.tchunk = 1;
  if (ctx->debug && ctx->dbg.ensure(8 * ((size_t)n + 32)) == cudaSuccess) a.dbg = ctx->dbg.p;
  return a;
}

// launch a pass kernel between two events (per-kernel device time)
void timed_pass(sph_ctx *ctx, int mode, int f32, const PassArgs &a, int count, uint8_t want) {
  const int i = ctx->n_kev;
  if (i < 64) {
    ctx->kev_mode[i] = mode;
    cudaEventRecord(ctx->kev[2 * i], ctx->stream);
  }
  launch_pass(ctx->stream, mode, f32, a, count, want, ctx->num_sms);
  if (i < 64) {
    cudaEventRecord(ctx->kev[2 * i + 1], ctx->stream);
    ctx->n_kev = i + 1;
  }
}

// SPH_DEBUG=1: print the most expensive bundles of the last launch
void debug_report(sph_ctx *ctx, int mode, int count) {
  if (!ctx->debug) return;
  int nb = 0;
  cudaStreamSynchronize(ctx->stream);
  cudaMemcpy(&nb, ctx->ints.p + 4, sizeof(int), cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> h(8 * (size_t)nb);
  cudaMemcpy(h.data(), ctx->dbg.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
  std::vector<int> idx(nb);
  for (int i = 0; i < nb; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return h[8 * x] > h[8 * y]; });
  unsigned long long tot = 0, tt = 0;
  double win = 0, cvis = 0, cneed = 0, fl = 0;
  for (int i = 0; i < nb; ++i) {
    tot += h[8 * i]; tt += h[8 * i + 1];
    win += h[8 * i + 4]; cvis += h[8 * i + 5]; cneed += h[8 * i + 6]; fl += h[8 * i + 7];
  }
  fprintf(stderr, "[sph dbg]   windows %.3g cells visited %.3g needed %.3g flushes %.3g\n", win, cvis, cneed, fl);
  if (const char *dump = getenv("SPH_DEBUG_DUMP")) {
    static int seq = 0;
    char path[512];
    snprintf(path, sizeof(path), "%s_%02d_mode%d.bin", dump, seq++, mode);
    if (FILE *f = fopen(path, "wb")) {
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      fclose(f);
    }
  }
  fprintf(stderr, "[sph dbg] mode %d: %d targets, %d bundles, sum cycles %.3g, tests %.3g\n", mode, count, nb,
          (double)tot, (double)tt);
  for (int i = 0; i < std::min(nb, 6); ++i) {
    const unsigned long long *d = &h[8 * idx[i]];
    float rb;
    unsigned bits = (unsigned)d[3];
    memcpy(&rb, &bits, 4);
    fprintf(stderr, "   bundle %d: cycles %.3g tests %.3g p0 %u targets %u subs %u Rb %g win %llu cvis %llu cneed %llu fl %llu\n",
            idx[i], (double)d[0], (double)d[1], (unsigned)(d[2] >> 32), (unsigned)((d[2] >> 8) & 0xff),
            (unsigned)(d[2] & 0xff), rb, d[4], d[5], d[6], d[7]);
  }
}

// sum of recorded kernel times per mode (call after a stream sync)
void collect_kernel_times(sph_ctx *ctx, sph_stats *st) {
  for (int i = 0; i < ctx->n_kev; ++i) {
    float t = 0.f;
    cudaEventElapsedTime(&t, ctx->kev[2 * i], ctx->kev[2 * i + 1]);
    const int m = ctx->kev_mode[i];
    if (st && m >= 0 && m < 3) st->t_kernel_ms[m] += t;
  }
  ctx->n_kev = 0;
}

// rounds of pass `mode` over targets whose state == want, compacting between
// rounds; returns the number of rounds run
int run_rounds(sph_ctx *ctx, int mode, int f32, PassArgs a, uint8_t want, int max_rounds, int *launches,
               int *rounds_out) {
  const int n = a.n;
  a.list = nullptr;
  a.static_count = n;
  timed_pass(ctx, mode, f32, a, n, want);
  debug_report(ctx, mode, n);
  ++*launches;
  int rounds = 1;
  for (;;) {
    launch_select(ctx->stream, ctx->iota.p, n, ctx->state.p, want, ctx->list.p, ctx->ints.p + 2, ctx->cub_temp.p,
                  ctx->cub_bytes);
    *launches += 2;
    int remaining = 0;
    SPH_CK(cudaMemcpyAsync(&remaining, ctx->ints.p + 2, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SPH_CK(cudaStreamSynchronize(ctx->stream));
    SPH_CK(cudaGetLastError());
    if (remaining == 0) break;
    if (rounds >= max_rounds) {
      *rounds_out = rounds;
      return fail(ctx, SPH_CUDA_ERROR, "neighbour search did not settle (internal round limit)");
    }
    a.list = ctx->list.p;
    timed_pass(ctx, mode, f32, a, remaining, want);
    debug_report(ctx, mode, remaining);
    ++*launches;
    ++rounds;
  }
  *rounds_out = rounds;
  return SPH_OK;
}

// child records / ancestors / cell map for the per-target kernel (sph_warp.cu)
int prepare_target_tree(sph_ctx *ctx, int n, int n_nodes, PassArgs &a) {
  SPH_CK(ctx->crec.ensure(16 * ((size_t)n_nodes + 1)));
  SPH_CK(ctx->anc4.ensure(n_nodes));
  SPH_CK(ctx->parent.ensure(n_nodes));
  SPH_CK(ctx->cellof.ensure(n));
  launch_kids(ctx->stream, ctx->nlo.p, ctx->nhi.p, n_nodes, n, ctx->crec.p, ctx->parent.p, ctx->anc4.p, ctx->cellof.p);
  if (!ctx->tb_emit_r0) {
    float root_side = 0.f;  // only used when the root is a single cell: its tight extent
    if (n_nodes == 1) {
      float4 l, h;
      cudaMemcpy(&l, ctx->nlo.p, sizeof(l), cudaMemcpyDeviceToHost);
      cudaMemcpy(&h, ctx->nhi.p, sizeof(h), cudaMemcpyDeviceToHost);
      root_side = std::max(h.x - l.x, std::max(h.y - l.y, h.z - l.z));
    }
    launch_r0(ctx->stream, ctx->nlo.p, ctx->nhi.p, ctx->nsize.p, ctx->parent.p, n_nodes, n, a.k, ctx->r0_scale,
              a.rmax, root_side, ctx->r0.p);
  }
  SPH_CK(cudaGetLastError());
  a.tree.crec = ctx->crec.p;
  a.tree.anc4 = ctx->anc4.p;
  a.tree.cellof = ctx->cellof.p;
  a.tree.root_start = n_nodes == 1 ? n_nodes : 0;  // a single-cell root: start from the virtual node
  ctx->crec_ready = true;
  return SPH_OK;
}

void use_target_tree(const sph_ctx *ctx, int n_nodes, PassArgs &a) {
  a.tree.crec = ctx->crec.p;
  a.tree.anc4 = ctx->anc4.p;
  a.tree.cellof = ctx->cellof.p;
  a.tree.root_start = n_nodes == 1 ? n_nodes : 0;
}

int density_pass_dev(sph_ctx *ctx, const sph_params *prm, const void *x, const void *y, const void *z,
                     const double *mass, const double *h0, double *h_out, double *rho_out, uint8_t *flags_out,
                     sph_stats *st, Timer &tm) {
  Nvtx range_pass("sph.pass");
  const int n = (int)prm->n;
  const int n_targets = prm->n_targets > 0 ? (int)prm->n_targets : n;
  const int k = prm->k;
  const int max_it = prm->max_iterations;
  int launches = 0;
  ctx->crec_ready = false;
  ctx->n_kev = 0;
  if (prm->n > (int64_t(1) << 27))
    return fail(ctx, SPH_UNSUPPORTED,
                "more than 2^27 particles on one device (list entries carry a 27-bit sorted index and a 5-bit "
                "image shift): split the set across devices (distributed.decomposed_pass)");
  { int rc0 = ensure_common(ctx, n, max_it); if (rc0) return rc0; }
  SPH_CK(ctx->t_lo.ensure(n));
  SPH_CK(ctx->t_hi.ensure(n));
  SPH_CK(ctx->d2k.ensure(n));
  SPH_CK(ctx->rho_s.ensure(n));
  tm.mark(1);
  RootInfo root{};
  int rc = SPH_OK;
  if (prm->periodic && !(prm->box > 0.0)) return fail(ctx, SPH_INVALID, "periodic box side must be > 0");
  // periodic with an explicit precision: nothing on the host depends on the
  // root box (rmax is 0.999 box), so its checks are read with the results
  // instead of costing a round trip here
  const bool defer_root = prm->periodic && prm->precision != SPH_PRECISION_AUTO;
  if (defer_root) {
    launch_bbox(ctx->stream, n, prm->precision == SPH_PRECISION_F32 ? 1 : 0, x, y, z, ctx->bbox_ord.p, ctx->root.p,
                &launches);
  } else {
    rc = stage_root(ctx, n, prm->precision, x, y, z, &root, &launches);
    if (rc) return rc;
    if (prm->periodic) {
      for (int a2 = 0; a2 < 3; ++a2)
        if (root.lo[a2] < 0.0 || root.hi[a2] >= prm->box)
          return fail(ctx, SPH_INVALID, "periodic mode needs every position inside [0, box)");
    }
  }
  const int compute_f32 = prm->precision == SPH_PRECISION_F32 || (prm->precision == 2 && !root.not_f32);
  const float rmax = compute_rmax(root, prm->periodic, prm->box);
  int n_nodes = 0;
  {
    Nvtx r("sph.tree");
    rc = stage_tree(ctx, n, prm->precision, compute_f32, x, y, z, mass, k, rmax, &n_nodes, &launches, true);
  }
  if (rc) return rc;
  tm.mark(2);
  int hist_rounds = 1, band_rounds = 0;
  // ---- search, exact select and density (per-target kernels) ----
  NvtxSpan range_search("sph.search");
  const bool sliced = ctx->slice_hi >= 0;
  const int slo = sliced ? (int)ctx->slice_lo : 0, shi = sliced ? (int)ctx->slice_hi : n;
  k_init_state<<<nblk(n), kTB, 0, ctx->stream>>>(n, n_targets, ctx->perm.p, ctx->state.p, slo, shi);
  k_iota<<<nblk(n), kTB, 0, ctx->stream>>>(n, ctx->iota.p);  // run_rounds compacts from it
  SPH_CK(cudaMemsetAsync(ctx->stats.p, 0, 8 * sizeof(unsigned long long), ctx->stream));
  SPH_CK(ctx->qints.ensure(32));
  SPH_CK(cudaMemsetAsync(ctx->qints.p, 0, 32 * sizeof(int), ctx->stream));
  PassArgs a = base_args(ctx, n, k, n_nodes, prm, rmax);
  rc = prepare_target_tree(ctx, n, n_nodes, a);
  if (rc) return rc;
  SPH_CK(ctx->ncount.ensure(n));
  a.ncount = ctx->ncount.p;
  a.fb_list = ctx->list.p;          // compacted targets for the collect instance
  a.fb_count = ctx->qints.p + 15;
  SPH_CK(cudaMemsetAsync(a.work_counter, 0, sizeof(int), ctx->stream));
  launches += 2;
  const int kv0 = ctx->n_kev;
  if (kv0 + 2 < 64) {
    ctx->kev_mode[kv0] = MODE_HIST;
    cudaEventRecord(ctx->kev[2 * kv0], ctx->stream);
  }
  bool known_run = false;
  const bool seeded = ctx->seed_stride > 1 && n >= 64 * ctx->seed_stride;
  if (seeded) {
    // a sparse calibration sample (or, SPH_LANE_NOSEED=0 / fp64 sets, seeds at every seed_stride-th sorted
    // position) through the general kernel from the tree's radius estimate; every other target then starts
    // from that estimate scaled by the sample's h / R0 quantile (or from its neighbouring seeds' converged h)
    const int ns = (n + ctx->seed_stride - 1) / ctx->seed_stride;
    const float noseed_m = ctx->lane_noseed;
    const int cal_stride = ctx->lane_cal_stride;
    const float cal_q = ctx->lane_cal_q;
    const bool noseed = noseed_m > 0.f && compute_f32 && ctx->known == 5 && lane_supported(k);
    SPH_CK(ctx->seeds.ensure(ns));
    PassArgs sa = a;
    sa.list = ctx->seeds.p;
    sa.list_count = ctx->qints.p + 14;
    if (n_targets < n || sliced) {
      // ghosts in the set: seed along the target order (compacted targets)
      SPH_CK(ctx->tlist.ensure(n));
      launch_select(ctx->stream, ctx->iota.p, n, ctx->state.p, ST_NEED_HIST, ctx->tlist.p, ctx->qints.p + 28,
                    ctx->cub_temp.p, ctx->cub_bytes);
      const int nt_eff = sliced ? shi - slo : n_targets;  // targets in the compacted list
      if (noseed) {
        // the calibration sample along the compacted target order
        const int ncal = (nt_eff + cal_stride - 1) / cal_stride;
        SPH_CK(ctx->calbuf.ensure(ncal + kCalWords + 64));
        k_seed_list_from<<<nblk(ncal), kTB, 0, ctx->stream>>>(ncal, cal_stride, ctx->tlist.p, ctx->seeds.p,
                                                              ctx->qints.p + 14);
        k_cal_save<<<nblk(std::max(ncal, kCalWords)), kTB, 0, ctx->stream>>>(ncal, ctx->seeds.p, ctx->r0.p, ctx->calbuf.p);
        launch_target(ctx->stream, compute_f32, sa, target_list_cap(k), ctx->qints.p + 5, ctx->num_sms);
        k_cal_reduce<<<nblk(ncal), kTB, 0, ctx->stream>>>(ncal, ctx->seeds.p, ctx->state.p, ctx->d2k.p, ctx->calbuf.p);
      } else {
        const int nst = (nt_eff + ctx->seed_stride - 1) / ctx->seed_stride;
        k_seed_list_from<<<nblk(nst), kTB, 0, ctx->stream>>>(nst, ctx->seed_stride, ctx->tlist.p, ctx->seeds.p,
                                                             ctx->qints.p + 14);
        launch_target(ctx->stream, compute_f32, sa, target_list_cap(k), ctx->qints.p + 5, ctx->num_sms);
        k_seed_radius_from<<<nblk(nt_eff), kTB, 0, ctx->stream>>>(nt_eff, ctx->seed_stride, ctx->tlist.p,
                                                                     ctx->state.p, ctx->d2k.p, ctx->seed_margin, rmax,
                                                                     ctx->r0.p);
      }
      launches += 5;
      a.list = ctx->tlist.p;  // walk the compacted targets, not every position
      a.list_count = ctx->qints.p + 28;
    } else if (noseed) {
      // no dense seeds: the lane kernel starts every target from the tree's radius estimate, scaled by the
      // geometric mean of h / R0 over a sparse sample (every cal_stride-th target through the per-target kernel)
      const int ncal = (n + cal_stride - 1) / cal_stride;
      SPH_CK(ctx->calbuf.ensure(ncal + kCalWords + 64));
      k_seed_list<<<nblk(ncal), kTB, 0, ctx->stream>>>(ncal, cal_stride, ctx->seeds.p, ctx->qints.p + 14);
      k_cal_save<<<nblk(std::max(ncal, kCalWords)), kTB, 0, ctx->stream>>>(ncal, ctx->seeds.p, ctx->r0.p, ctx->calbuf.p);
      launch_target(ctx->stream, compute_f32, sa, target_list_cap(k), ctx->qints.p + 5, ctx->num_sms);
      k_cal_reduce<<<nblk(ncal), kTB, 0, ctx->stream>>>(ncal, ctx->seeds.p, ctx->state.p, ctx->d2k.p, ctx->calbuf.p);
      launches += 4;
    } else {
      k_seed_list<<<nblk(ns), kTB, 0, ctx->stream>>>(ns, ctx->seed_stride, ctx->seeds.p, ctx->qints.p + 14);
      launch_target(ctx->stream, compute_f32, sa, target_list_cap(k), ctx->qints.p + 5, ctx->num_sms);
      k_seed_radius<<<nblk(n), kTB, 0, ctx->stream>>>(n, ctx->seed_stride, 1, ctx->state.p, ctx->d2k.p,
                                                      ctx->seed_margin, rmax, ctx->r0.p);
      launches += 3;
    }
    SPH_CK(cudaMemsetAsync(a.work_counter, 0, sizeof(int), ctx->stream));
    // neighbour-cell lists for the radii the seeds imply
    const int cap = ctx->cell_lists;
    const int ncell = ctx->last_ncell;  // counted with the tree (stage_tree)
    bool lane_ran = false;
    if (compute_f32 && ctx->known == 5 && lane_supported(k) && ctx->kn_list.ensure(n) == cudaSuccess) {
      // one lane per target over bundles of 32 sorted neighbours (sph_lane.cu);
      // what it leaves, the per-target kernel takes
      cudaEventRecord(ctx->kev_known[0], ctx->stream);
      PassArgs ka = a;
      ka.posj = ctx->posj.p;
      ka.fb_list = ctx->kn_list.p;
      ka.fb_count = ctx->qints.p + 21;
      ka.kn_counters = ctx->qints.p + 10;
      launch_lane(ctx->stream, ka, lane_list_cap(k), noseed ? noseed_m : ctx->lane_margin / ctx->seed_margin, ctx->lane_exc,
                  ctx->lane_stream, ctx->num_sms, noseed ? ctx->calbuf.p : nullptr, cal_q);
      cudaEventRecord(ctx->kev_known[1], ctx->stream);
      SPH_CK(cudaMemsetAsync(a.work_counter, 0, sizeof(int), ctx->stream));
      a.list = ctx->kn_list.p;
      a.list_count = ctx->qints.p + 21;
      launches += 2;
      known_run = true;
      lane_ran = true;
    }
    // neighbour-cell lists for the cells that still hold targets (all of them, or what the lane kernel left)
    if ((!known_run || lane_ran) && cap > 0 && ncell >= 0 && ctx->clist.ensure((size_t)ncell * cap) == cudaSuccess &&
        ctx->clen.ensure(ncell) == cudaSuccess && ctx->crad2.ensure(ncell) == cudaSuccess &&
        ctx->cnear.ensure(ncell) == cudaSuccess) {
      launch_cell_lists(ctx->stream, a, ctx->cellnode.p, ctx->ncell_dev.p, cap, ctx->clist.p, ctx->clen.p,
                        ctx->crad2.p, ctx->cnear.p, ctx->near_frac, 1.0f, ctx->num_sms, ncell);
      a.cnear = ctx->cnear.p;
      a.near_frac2 = ctx->near_frac * ctx->near_frac;
      a.clist = ctx->clist.p;
      a.clen = ctx->clen.p;
      a.crad2 = ctx->crad2.p;
      a.cellidx = ctx->cellidx.p;
      a.clcap = cap;
      launches += 1;
    }
    cudaGetLastError();  // an allocation failure above only skips the lists
  }
  ctx->known_ran = known_run;
  launch_target(ctx->stream, compute_f32, a, target_list_cap(k), ctx->qints.p + 5, ctx->num_sms);
  ++launches;
  a.list = nullptr;
  a.list_count = nullptr;
  if (ctx->debug) {
    int fbk[32];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpy(fbk, ctx->qints.p, sizeof(fbk), cudaMemcpyDeviceToHost);
    if (ctx->known == 5)
      fprintf(stderr, "[sph lane] %d targets to the per-target kernel: bundles bailed %d; lanes: few within R %d, "
              "list full %d, bracket %d, left out %d\n", fbk[21], fbk[10], fbk[11], fbk[12], fbk[13], fbk[23]);
    else
      fprintf(stderr, "[sph seeds] %d seeds to the general kernel\n", fbk[14]);
    fprintf(stderr, "[sph warp] fall back to the walking select: %d overflowed lists, %d bracket misses; %d walks\n",
            fbk[5], fbk[6], fbk[8]);
  }
  // the collect instance for overflowed lists is enqueued unconditionally: it
  // reads its target count on the device ([15], appended by the main kernel)
  // and exits at once when there is none, so no host round trip is needed
  // here.  The main kernel's other fallback counters ([6] bracket misses, [9]
  // stack overflows) and the collect instance's ([16..20]) are read with the
  // results; the walking passes for what is left then run before a second
  // finalize (never seen in the bench configs).
  {
    SPH_CK(cudaMemsetAsync(a.work_counter, 0, sizeof(int), ctx->stream));
    PassArgs c = a;
    c.list = ctx->list.p;
    c.list_count = ctx->qints.p + 15;
    c.fb_list = nullptr;
    launch_target(ctx->stream, compute_f32, c, ctx->collect_cap, ctx->qints.p + 16, ctx->num_sms, true);
    launches += 2;
  }
  if (kv0 + 2 < 64) {
    cudaEventRecord(ctx->kev[2 * kv0 + 1], ctx->stream);
    ctx->n_kev = kv0 + 1;
  }
  SPH_CK(cudaMemcpyAsync(ctx->stats.p + 3, ctx->stats.p, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                         ctx->stream));
  tm.mark(3);
  const bool warp_deferred = true;
  PassArgs warp_args = a;
  tm.mark(4);
  tm.mark(5);
  range_search.end();
  // ---- finalize ----
  Nvtx range_fin("sph.finalize");
  int *rounds_hist = ctx->ints.p + kIntsFixed;
  std::vector<int> hist(max_it + 2);
  unsigned long long stat_all[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int qd[32] = {0};
  for (int attempt = 0;; ++attempt) {
    SPH_CK(cudaMemsetAsync(rounds_hist, 0, sizeof(int) * (max_it + 2), ctx->stream));
    const unsigned long long bad_init = ~0ull;
    SPH_CK(cudaMemcpyAsync(ctx->stats.p + 2, &bad_init, sizeof(bad_init), cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->in_h_ready) cudaStreamWaitEvent(ctx->stream, ctx->in_h_ready, 0);  // h0 copied on the side stream
    k_finalize<<<nblk(n), kTB, max_it + 2 <= kFinalizeSmemBins ? sizeof(int) * (max_it + 2) : 0, ctx->stream>>>(
        n, n_targets, ctx->perm.p, ctx->state.p, ctx->d2k.p, ctx->rho_s.p, h0, max_it, h_out, rho_out, flags_out,
        rounds_hist, ctx->stats.p + 2, slo, shi, sliced ? ctx->slice_orig.p : nullptr);
    ++launches;
    tm.mark(6);
    SPH_CK(cudaMemcpyAsync(hist.data(), rounds_hist, sizeof(int) * (max_it + 2), cudaMemcpyDeviceToHost, ctx->stream));
    SPH_CK(cudaMemcpyAsync(stat_all, ctx->stats.p, sizeof(stat_all), cudaMemcpyDeviceToHost, ctx->stream));
    if (defer_root) SPH_CK(cudaMemcpyAsync(&root, ctx->root.p, sizeof(RootInfo), cudaMemcpyDeviceToHost, ctx->stream));
    if (warp_deferred) SPH_CK(cudaMemcpyAsync(qd, ctx->qints.p, sizeof(qd), cudaMemcpyDeviceToHost, ctx->stream));
    SPH_CK(cudaStreamSynchronize(ctx->stream));
    SPH_CK(cudaGetLastError());
    if (!warp_deferred || attempt > 0) break;
    // fallbacks of the per-target path: [9] stack overflows, [16] + [17] + [20]
    // what even the collect instance could not serve
    const int coll_left = qd[16] + qd[17] + qd[20];
    if (ctx->debug)
      fprintf(stderr, "[sph collect] %d targets; still to the walking select: %d overflowed, %d bracket misses, %d stack\n",
              qd[5] + qd[6], qd[16], qd[17], qd[20]);
    if (qd[9] == 0 && coll_left == 0) break;
    PassArgs wa = warp_args;
    if (qd[9] > 0) {
      // targets the stack could not serve: the bundle search passes
      int hr = 0;
      rc = run_rounds(ctx, MODE_HIST, compute_f32, wa, ST_NEED_HIST, 64, &launches, &hr);
      if (rc) return rc;
      hist_rounds += hr;
    }
    // targets no list could serve: walking select + density
    rc = run_rounds(ctx, MODE_BAND, compute_f32, wa, ST_NEED_BAND, 64, &launches, &band_rounds);
    if (rc) return rc;
    timed_pass(ctx, MODE_DENS, compute_f32, wa, n, ST_DONE);
    ++launches;
  }
  collect_kernel_times(ctx, st);
  if (defer_root) {  // the checks stage_root would have made, on the root read with the results
    if (root.nonfinite) return fail(ctx, SPH_INVALID, "positions must be finite");
    for (int a2 = 0; a2 < 3; ++a2)
      if (root.lo[a2] < 0.0 || root.hi[a2] >= prm->box)
        return fail(ctx, SPH_INVALID, "periodic mode needs every position inside [0, box)");
  }
  if (st) {
    st->t_kernel_ms[3] = tm.ms(1, 2);
    if (ctx->known_ran) {
      float t = 0.f;
      cudaEventElapsedTime(&t, ctx->kev_known[0], ctx->kev_known[1]);
      st->t_known_ms = t;
      st->known_fallbacks = qd[21];
    } else {
      st->known_fallbacks = -1;
    }
  }

  // ---- stats, reference todo trace, error mapping ----
  const long long unconv = hist[max_it + 1];
  int last = 0;
  for (int r = 1; r <= max_it; ++r)
    if (hist[r]) last = r;
  if (st) {
    st->iterations = unconv ? max_it : last;
    st->n_todo = std::min(st->iterations, SPH_MAX_TODO);
    long long acc = unconv;
    std::vector<long long> todo(last + 1, 0);
    for (int r = max_it; r >= 1; --r) {
      acc += hist[r];
      if (r <= last || unconv) {
        if (r - 1 < SPH_MAX_TODO) st->todo_sizes[r - 1] = acc;
      }
    }
    st->pair_tests = (int64_t)stat_all[0];
    st->accepted_pairs = (int64_t)stat_all[1];
    st->search_pair_tests = (int64_t)stat_all[3];
    st->unconverged = unconv;
    st->bad_index = stat_all[2] == ~0ull ? -1 : (int64_t)stat_all[2];
    st->gpu_launches = launches;
    st->search_rounds = hist_rounds;
    st->select_rounds = band_rounds;
    st->n_nodes = n_nodes;
  }
  if (stat_all[4])
    return fail(ctx, SPH_CUDA_ERROR, "exact K-th neighbour selection did not settle (internal round limit)");
  const bool degenerate = stat_all[2] != ~0ull;
  if (degenerate) {
    char buf[256];
    snprintf(buf, sizeof(buf), "particle %llu: %d-th nearest neighbour is at zero distance; >= %d coincident particles",
             (unsigned long long)stat_all[2], k, k + 1);
    return fail(ctx, SPH_DEGENERATE, buf);
  }
  if (unconv) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%lld of %d particles still flagged after %d iterations", unconv, n_targets, max_it);
    return fail(ctx, SPH_NOT_CONVERGED, buf);
  }
  return SPH_OK;
}

int validate(sph_ctx *ctx, const sph_params *p) {
  if (!ctx) return SPH_INVALID;
  if (!p) return fail(ctx, SPH_INVALID, "params is NULL");
  if (p->n < 1) return fail(ctx, SPH_INVALID, "workload must contain at least one particle");
  if (p->n >= (1ll << 31) - 64) return fail(ctx, SPH_INVALID, "n must be < 2^31 per device");
  if (p->k < 1) return fail(ctx, SPH_INVALID, "k_neighbors must be >= 1");
  if (p->max_iterations < 0) return fail(ctx, SPH_INVALID, "max_iterations must be >= 0");
  if (p->precision < 0 || p->precision > 2) return fail(ctx, SPH_INVALID, "unknown precision");
  if (p->kernel < 0 || p->kernel > 1) return fail(ctx, SPH_INVALID, "unknown kernel");
  if (p->n_targets < 0 || p->n_targets > p->n) return fail(ctx, SPH_INVALID, "n_targets must be in [0, n]");
  return SPH_OK;
}

size_t elem_size(int precision) { return precision == SPH_PRECISION_F32 ? 4 : 8; }

cudaError_t h2d_strided(void *dst, const void *src, size_t elem, int64_t stride, int64_t n, cudaStream_t s) {
  if (stride == (int64_t)elem) return cudaMemcpyAsync(dst, src, elem * n, cudaMemcpyHostToDevice, s);
  return cudaMemcpy2DAsync(dst, elem, src, (size_t)stride, elem, (size_t)n, cudaMemcpyHostToDevice, s);
}
cudaError_t d2h_strided(void *dst, const void *src, size_t elem, int64_t stride, int64_t n, cudaStream_t s) {
  if (stride == (int64_t)elem) return cudaMemcpyAsync(dst, src, elem * n, cudaMemcpyDeviceToHost, s);
  return cudaMemcpy2DAsync(dst, (size_t)stride, src, elem, elem, (size_t)n, cudaMemcpyDeviceToHost, s);
}

}  // namespace

extern "C" {

int sph_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int sph_ctx_create(sph_ctx **out, int device) {
  if (!out) return SPH_INVALID;
  *out = nullptr;
  int count = sph_device_count();
  if (count <= 0) return SPH_CUDA_ERROR;
  if (device < 0 || device >= count) return SPH_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return SPH_CUDA_ERROR;
  sph_ctx *c = new sph_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_side_start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_mass, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_h, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return SPH_CUDA_ERROR;
  }
  for (auto &e : c->ev) cudaEventCreate(&e);
  for (auto &e : c->kev) cudaEventCreate(&e);
  const char *dbg = getenv("SPH_DEBUG");
  c->debug = dbg && dbg[0] == '1';
  if (const char *v = getenv("SPH_SEED")) c->seed_stride = atoi(v);
  if (const char *v = getenv("SPH_SEEDM")) c->seed_margin = (float)atof(v);
  if (const char *v = getenv("SPH_KNOWN")) c->known = atoi(v);
  if (const char *v = getenv("SPH_LANEM")) c->lane_margin = (float)atof(v);
  if (const char *v = getenv("SPH_LANEX")) c->lane_exc = (float)atof(v);
  if (const char *v = getenv("SPH_LANE_STREAM")) c->lane_stream = atoi(v);
  if (const char *v = getenv("SPH_LANE_NOSEED")) c->lane_noseed = (float)atof(v);
  if (const char *v = getenv("SPH_LANE_CAL")) c->lane_cal_stride = std::max(16, atoi(v));
  if (const char *v = getenv("SPH_LANE_CALQ")) c->lane_cal_q = (float)atof(v);
  if (const char *v = getenv("SPH_CLIST")) c->cell_lists = atoi(v);
  if (const char *v = getenv("SPH_CCAP")) c->collect_cap = std::max(32, std::min(1024, atoi(v)));
  if (const char *v = getenv("SPH_TSHRINK")) c->tshrink = atoi(v);
  if (const char *v = getenv("SPH_NEARF")) c->near_frac = (float)atof(v);
  if (const char *v = getenv("SPH_R0SCALE")) c->r0_scale = (float)atof(v);
  cudaEventCreate(&c->kev_known[0]);
  cudaEventCreate(&c->kev_known[1]);
  *out = c;
  return SPH_OK;
}

void sph_ctx_destroy(sph_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->in_x.release(); c->in_y.release(); c->in_z.release(); c->in_m.release(); c->io_h.release();
  c->out_rho.release(); c->out_flags.release(); c->keys_in.release(); c->keys.release(); c->bbox_ord.release();
  c->idx_in.release(); c->idx.release(); c->perm.release(); c->deep_list.release(); c->deep_segs.release(); c->iota.release();
  c->list.release(); c->lvl8.release(); c->lvl32.release(); c->state.release(); c->ints.release();
  c->noff.release(); c->nlo.release(); c->nhi.release(); c->nsize.release(); c->r0.release(); c->pos_sorted.release();
  c->cub_temp.release(); c->tasks.release(); c->members.release(); c->seeds.release(); c->calbuf.release(); c->node_p.release();
  c->dscratch.release(); c->ncell_dev.release(); c->tlist.release(); c->clist.release(); c->clen.release();
  c->cellidx.release(); c->cellnode.release(); c->crad2.release(); c->cnear.release(); c->ncount.release();
  c->crec.release(); c->anc4.release(); c->parent.release(); c->cellof.release(); c->qints.release();
  c->root.release(); c->t_lo.release(); c->t_hi.release(); c->d2k.release(); c->kn_list.release(); c->posj.release();
  c->rho_s.release(); c->hfix.release(); c->mass_s.release(); c->counts_s.release(); c->counts_o.release(); c->stats.release();
  cudaEventDestroy(c->kev_known[0]);
  cudaEventDestroy(c->kev_known[1]);
  for (auto &e : c->ev) cudaEventDestroy(e);
  for (auto &e : c->kev) cudaEventDestroy(e);
  cudaStreamDestroy(c->stream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  for (cudaEvent_t e : {c->ev_side_start, c->ev_mass, c->ev_h})
    if (e) cudaEventDestroy(e);
  delete c;
}

void *sph_ctx_stream(sph_ctx *c) { return c ? (void *)c->stream : nullptr; }

const char *sph_last_error(const sph_ctx *c) { return c ? c->err.c_str() : "null context"; }

uint64_t sph_fnv1a64(const uint8_t *data, size_t len) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < len; ++i) h = (h ^ data[i]) * 0x100000001B3ull;
  return h;
}

namespace {
// splitmix64 UniformBox draws (reference workload.py:42-60, 77-84)
__global__ void k_uniform_box(int64_t n, uint64_t seed, double box, double *x, double *y, double *z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const uint64_t t = (uint64_t)(3 * i + a) + 1ull;
    uint64_t s = seed + t * 0x9E3779B97F4A7C15ull;
    s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ull;
    s = (s ^ (s >> 27)) * 0x94D049BB133111EBull;
    s = s ^ (s >> 31);
    const double u = __dmul_rn(__ull2double_rn(s >> 11), 0x1p-53);
    double w = __dmul_rn(u, box);
    if (w >= box) w = nextafter(box, 0.0);
    v[a] = w;
  }
  x[i] = v[0];
  y[i] = v[1];
  z[i] = v[2];
}
}  // namespace

int sph_uniform_box_device(sph_ctx *ctx, int64_t n, uint64_t seed, double box, double *d_x, double *d_y,
                           double *d_z) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || !(box > 0.0) || (n > 0 && (!d_x || !d_y || !d_z))) return fail(ctx, SPH_INVALID, "invalid uniform box request");
  if (n == 0) return SPH_OK;
  cudaSetDevice(ctx->device);
  k_uniform_box<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(n, seed, box, d_x, d_y, d_z);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, SPH_CUDA_ERROR, std::string("k_uniform_box: ") + cudaGetErrorString(e));
  return SPH_OK;
}

int sph_nfw_positions_device(sph_ctx *ctx, int64_t n, int64_t n_halos, const int64_t *d_halo_start,
                             const double *d_halo, double concentration, double x_max, uint64_t seed, double box,
                             float *d_x, float *d_y, float *d_z, float *d_vel) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || n_halos < 0 || !(box > 0.0) || !(concentration > 0.0) || !(x_max > 0.0) || !d_halo_start ||
      (n_halos > 0 && !d_halo) || (n > 0 && (!d_x || !d_y || !d_z)))
    return fail(ctx, SPH_INVALID, "invalid NFW generator request");
  if (n == 0) return SPH_OK;
  cudaSetDevice(ctx->device);
  launch_nfw_positions(ctx->stream, n, n_halos, d_halo_start, d_halo, concentration, x_max, seed, box, d_x, d_y, d_z,
                       d_vel);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, SPH_CUDA_ERROR, std::string("k_nfw_positions: ") + cudaGetErrorString(e));
  return SPH_OK;
}

double sph_fp32_peak(sph_ctx *ctx) {
  if (!ctx) return 0.0;
  cudaSetDevice(ctx->device);
  float *d = nullptr;
  if (cudaMalloc(&d, sizeof(float)) != cudaSuccess) return 0.0;
  const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
  k_ffma_probe<<<blocks, threads, 0, ctx->stream>>>(d, iters);  // warm-up
  cudaEventRecord(ctx->ev[10], ctx->stream);
  k_ffma_probe<<<blocks, threads, 0, ctx->stream>>>(d, iters);
  cudaEventRecord(ctx->ev[11], ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[10], ctx->ev[11]);
  cudaFree(d);
  return ms > 0.f ? (double)blocks * threads * iters * 16.0 / (ms * 1e-3) : 0.0;
}

int sph_density_pass_device(sph_ctx *ctx, const sph_params *prm, const void *d_x, const void *d_y,
                            const void *d_z, const double *d_mass, double *d_h, double *d_rho, uint8_t *d_flags,
                            sph_stats *st) {
  int rc = validate(ctx, prm);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (st) memset(st, 0, sizeof(*st));
  Timer tm{ctx};
  tm.mark(0);
  // the input h drives only the todo trace: keep a copy so d_h can be overwritten
  if (ctx->hfix.ensure(prm->n) != cudaSuccess) return fail(ctx, SPH_CUDA_ERROR, "out of device memory");
  SPH_CK(cudaMemcpyAsync(ctx->hfix.p, d_h, sizeof(double) * (prm->n_targets > 0 ? prm->n_targets : prm->n),
                         cudaMemcpyDeviceToDevice, ctx->stream));
  rc = density_pass_dev(ctx, prm, d_x, d_y, d_z, d_mass, ctx->hfix.p, d_h, d_rho, d_flags, st, tm);
  tm.mark(7);
  cudaStreamSynchronize(ctx->stream);
  if (st && (rc == SPH_OK || rc == SPH_DEGENERATE || rc == SPH_NOT_CONVERGED)) {
    st->t_stage_ms[0] = tm.ms(0, 1);
    st->t_stage_ms[1] = tm.ms(1, 2);
    st->t_stage_ms[2] = tm.ms(2, 3);
    st->t_stage_ms[3] = tm.ms(3, 4);
    st->t_stage_ms[4] = 0.0;
    st->t_stage_ms[5] = tm.ms(5, 6);
    st->t_stage_ms[6] = 0.0;
    st->t_stage_ms[7] = tm.ms(0, 7);
  }
  return rc;
}

int sph_density_pass(sph_ctx *ctx, const sph_params *prm, const void *x, const void *y, const void *z,
                     int64_t pos_stride, const double *mass, int64_t mass_stride, double *h, int64_t h_stride,
                     double *rho, int64_t rho_stride, uint8_t *flags, int64_t flags_stride, sph_stats *st) {
  int rc = validate(ctx, prm);
  if (rc) return rc;
  if (!x || !y || !z || !mass || !h || !rho || !flags) return fail(ctx, SPH_INVALID, "null array pointer");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (st) memset(st, 0, sizeof(*st));
  const int64_t n = prm->n;
  const size_t es = elem_size(prm->precision);
  SPH_CK(ctx->in_x.ensure(n));
  SPH_CK(ctx->in_y.ensure(n));
  SPH_CK(ctx->in_z.ensure(n));
  SPH_CK(ctx->in_m.ensure(n));
  SPH_CK(ctx->io_h.ensure(n));
  SPH_CK(ctx->hfix.ensure(n));
  SPH_CK(ctx->out_rho.ensure(n));
  SPH_CK(ctx->out_flags.ensure(n));
  Timer tm{ctx};
  tm.mark(0);
  cudaStream_t s = ctx->stream;
  SPH_CK(h2d_strided(ctx->in_x.p, x, es, pos_stride, n, s));
  SPH_CK(h2d_strided(ctx->in_y.p, y, es, pos_stride, n, s));
  SPH_CK(h2d_strided(ctx->in_z.p, z, es, pos_stride, n, s));
  // masses and initial h on the side stream: they overlap the key / sort /
  // tree kernels that only need positions (the pass waits on the events)
  const int64_t nt = prm->n_targets > 0 ? prm->n_targets : n;
  cudaStream_t s2 = ctx->stream2;
  SPH_CK(cudaEventRecord(ctx->ev_side_start, s));
  SPH_CK(cudaStreamWaitEvent(s2, ctx->ev_side_start, 0));  // reuse of the staging buffers is ordered
  SPH_CK(h2d_strided(ctx->in_m.p, mass, 8, mass_stride, n, s2));
  SPH_CK(cudaEventRecord(ctx->ev_mass, s2));
  SPH_CK(h2d_strided(ctx->hfix.p, h, 8, h_stride, nt, s2));
  SPH_CK(cudaEventRecord(ctx->ev_h, s2));
  ctx->in_mass_ready = ctx->ev_mass;
  ctx->in_h_ready = ctx->ev_h;
  rc = density_pass_dev(ctx, prm, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, ctx->in_m.p, ctx->hfix.p, ctx->io_h.p,
                        ctx->out_rho.p, ctx->out_flags.p, st, tm);
  ctx->in_mass_ready = nullptr;
  ctx->in_h_ready = nullptr;
  SPH_CK(cudaStreamWaitEvent(s, ctx->ev_h, 0));  // error paths: the side copies are done before returning
  if (rc == SPH_OK) {
    SPH_CK(d2h_strided(h, ctx->io_h.p, 8, h_stride, nt, s));
    SPH_CK(d2h_strided(rho, ctx->out_rho.p, 8, rho_stride, nt, s));
    SPH_CK(d2h_strided(flags, ctx->out_flags.p, 1, flags_stride, nt, s));
  }
  tm.mark(7);
  SPH_CK(cudaStreamSynchronize(s));
  if (st && (rc == SPH_OK || rc == SPH_DEGENERATE || rc == SPH_NOT_CONVERGED)) {
    st->t_stage_ms[0] = tm.ms(0, 1);
    st->t_stage_ms[1] = tm.ms(1, 2);
    st->t_stage_ms[2] = tm.ms(2, 3);
    st->t_stage_ms[3] = tm.ms(3, 4);
    st->t_stage_ms[4] = 0.0;
    st->t_stage_ms[5] = tm.ms(5, 6);
    st->t_stage_ms[6] = rc == SPH_OK ? tm.ms(6, 7) : 0.0;
    st->t_stage_ms[7] = tm.ms(0, 7);
  }
  return rc;
}

int sph_density_pass_multi(sph_ctx *const *ctxs, int32_t n_ctx, const sph_params *prm, const void *x,
                           const void *y, const void *z, int64_t pos_stride, const double *mass, int64_t mass_stride,
                           double *h, int64_t h_stride, double *rho, int64_t rho_stride, uint8_t *flags,
                           int64_t flags_stride, sph_stats *stats) {
  if (!ctxs || n_ctx < 1 || !ctxs[0]) return SPH_INVALID;
  sph_ctx *c0 = ctxs[0];
  for (int d = 0; d < n_ctx; ++d) {
    if (!ctxs[d]) return fail(c0, SPH_INVALID, "null context");
    for (int e = 0; e < d; ++e)
      if (ctxs[e] == ctxs[d]) return fail(c0, SPH_INVALID, "each slice needs its own context");
  }
  int rc = validate(c0, prm);
  if (rc) return rc;
  if (prm->n_targets != 0 && prm->n_targets != prm->n)
    return fail(c0, SPH_INVALID, "a multi-device pass takes every particle as a target (n_targets = 0)");
  if (!x || !y || !z || !mass || !h || !rho || !flags) return fail(c0, SPH_INVALID, "null array pointer");
  const int64_t n = prm->n;
  if (n_ctx > n) n_ctx = (int32_t)n;
  if (stats) memset(stats, 0, sizeof(sph_stats) * (n_ctx + 1));
  struct Part {
    int rc = SPH_OK;
    sph_stats st{};
    std::vector<int64_t> orig;
    std::vector<double> h, rho;
    std::vector<uint8_t> fl;
  };
  std::vector<Part> part(n_ctx);
  auto work = [&](int d) {
    Nvtx range_dev("sph.multi.device");
    sph_ctx *ctx = ctxs[d];
    Part &P = part[d];
    const int64_t lo = n * d / n_ctx, hi = n * (d + 1) / n_ctx, m = hi - lo;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    P.rc = [&]() -> int {
      // every device holds every position (the candidates) and takes the
      // targets of its slice of the sorted (key) order
      const size_t es = elem_size(prm->precision);
      SPH_CK(ctx->in_x.ensure(n));
      SPH_CK(ctx->in_y.ensure(n));
      SPH_CK(ctx->in_z.ensure(n));
      SPH_CK(ctx->in_m.ensure(n));
      SPH_CK(ctx->io_h.ensure(n));
      SPH_CK(ctx->hfix.ensure(n));
      SPH_CK(ctx->out_rho.ensure(n));
      SPH_CK(ctx->out_flags.ensure(n));
      SPH_CK(ctx->slice_orig.ensure(std::max<int64_t>(m, 1)));
      cudaStream_t s = ctx->stream;
      SPH_CK(h2d_strided(ctx->in_x.p, x, es, pos_stride, n, s));
      SPH_CK(h2d_strided(ctx->in_y.p, y, es, pos_stride, n, s));
      SPH_CK(h2d_strided(ctx->in_z.p, z, es, pos_stride, n, s));
      SPH_CK(h2d_strided(ctx->in_m.p, mass, 8, mass_stride, n, s));
      SPH_CK(h2d_strided(ctx->hfix.p, h, 8, h_stride, n, s));
      Timer tm{ctx};
      tm.mark(0);
      tm.mark(1);
      ctx->slice_lo = lo;
      ctx->slice_hi = hi;
      int r = density_pass_dev(ctx, prm, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, ctx->in_m.p, ctx->hfix.p,
                               ctx->io_h.p, ctx->out_rho.p, ctx->out_flags.p, &P.st, tm);
      ctx->slice_lo = 0;
      ctx->slice_hi = -1;
      if (r != SPH_OK && r != SPH_DEGENERATE && r != SPH_NOT_CONVERGED) return r;
      P.orig.resize(m);
      P.h.resize(m);
      P.rho.resize(m);
      P.fl.resize(m);
      SPH_CK(cudaMemcpyAsync(P.orig.data(), ctx->slice_orig.p, 8 * m, cudaMemcpyDeviceToHost, s));
      SPH_CK(cudaMemcpyAsync(P.h.data(), ctx->io_h.p, 8 * m, cudaMemcpyDeviceToHost, s));
      SPH_CK(cudaMemcpyAsync(P.rho.data(), ctx->out_rho.p, 8 * m, cudaMemcpyDeviceToHost, s));
      SPH_CK(cudaMemcpyAsync(P.fl.data(), ctx->out_flags.p, m, cudaMemcpyDeviceToHost, s));
      SPH_CK(cudaStreamSynchronize(s));
      return SPH_OK;
    }();
  };
  {
    std::vector<std::thread> th;
    for (int d = 1; d < n_ctx; ++d) th.emplace_back(work, d);
    work(0);
    for (auto &t : th) t.join();
  }
  for (int d = 0; d < n_ctx; ++d)
    if (part[d].rc != SPH_OK) {
      if (d) c0->err = ctxs[d]->err;
      return part[d].rc;
    }
  // merged statistics: the todo trace is the sum of the slices' traces
  sph_stats M{};
  int64_t bad = -1, unconv = 0;
  for (int d = 0; d < n_ctx; ++d) {
    const sph_stats &S = part[d].st;
    if (stats) stats[d] = S;
    M.iterations = std::max(M.iterations, S.iterations);
    for (int r = 0; r < SPH_MAX_TODO; ++r) M.todo_sizes[r] += S.todo_sizes[r];
    for (int i = 0; i < 8; ++i) M.t_stage_ms[i] = std::max(M.t_stage_ms[i], S.t_stage_ms[i]);
    for (int i = 0; i < 4; ++i) M.t_kernel_ms[i] = std::max(M.t_kernel_ms[i], S.t_kernel_ms[i]);
    M.pair_tests += S.pair_tests;
    M.accepted_pairs += S.accepted_pairs;
    M.search_pair_tests += S.search_pair_tests;
    M.gpu_launches += S.gpu_launches;
    M.search_rounds = std::max(M.search_rounds, S.search_rounds);
    M.select_rounds = std::max(M.select_rounds, S.select_rounds);
    M.n_nodes = S.n_nodes;
    if (S.bad_index >= 0 && (bad < 0 || S.bad_index < bad)) bad = S.bad_index;
    unconv += S.unconverged;
  }
  M.n_todo = std::min(M.iterations, SPH_MAX_TODO);
  M.bad_index = bad;
  M.unconverged = unconv;
  M.known_fallbacks = -1;
  if (stats) stats[n_ctx] = M;
  if (bad >= 0) {
    char buf[256];
    snprintf(buf, sizeof(buf), "particle %lld: %d-th nearest neighbour is at zero distance; >= %d coincident particles",
             (long long)bad, prm->k, prm->k + 1);
    return fail(c0, SPH_DEGENERATE, buf);
  }
  if (unconv) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%lld of %lld particles still flagged after %d iterations", (long long)unconv,
             (long long)n, prm->max_iterations);
    return fail(c0, SPH_NOT_CONVERGED, buf);
  }
  // results in the caller's (original) order
  for (int d = 0; d < n_ctx; ++d) {
    const Part &P = part[d];
    char *hb = reinterpret_cast<char *>(h), *rb = reinterpret_cast<char *>(rho), *fb = reinterpret_cast<char *>(flags);
    for (size_t i = 0; i < P.orig.size(); ++i) {
      const int64_t o = P.orig[i];
      *reinterpret_cast<double *>(hb + o * h_stride) = P.h[i];
      *reinterpret_cast<double *>(rb + o * rho_stride) = P.rho[i];
      *reinterpret_cast<uint8_t *>(fb + o * flags_stride) = P.fl[i];
    }
  }
  return SPH_OK;
}

int sph_range_query(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z,
                    const double *h, const int64_t *offsets, int64_t *idx_out, double *d2_out) {
  if (!ctx) return SPH_INVALID;
  if (n < 1) return fail(ctx, SPH_INVALID, "need at least one particle");
  if (n >= (1ll << 31) - 64) return fail(ctx, SPH_INVALID, "n must be < 2^31 per device");
  if (precision < 0 || precision > 2) return fail(ctx, SPH_INVALID, "unknown precision");
  if (!offsets || offsets[0] != 0) return fail(ctx, SPH_INVALID, "offsets must start at 0 (n + 1 entries)");
  const int64_t total = offsets[n];
  for (int64_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i]) return fail(ctx, SPH_INVALID, "offsets must be non-decreasing");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = ensure_common(ctx, n, 1);
  if (rc) return rc;
  const size_t es = elem_size(precision);
  SPH_CK(ctx->in_x.ensure(n));
  SPH_CK(ctx->in_y.ensure(n));
  SPH_CK(ctx->in_z.ensure(n));
  SPH_CK(ctx->in_m.ensure(n));
  SPH_CK(ctx->io_h.ensure(n));
  SPH_CK(ctx->hfix.ensure(n));
  cudaStream_t s = ctx->stream;
  SPH_CK(cudaMemcpyAsync(ctx->in_x.p, x, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_y.p, y, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_z.p, z, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->io_h.p, h, 8 * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemsetAsync(ctx->in_m.p, 0, 8 * n, s));
  int launches = 0;
  RootInfo root{};
  rc = stage_root(ctx, (int)n, precision, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, &root, &launches);
  if (rc) return rc;
  const int compute_f32 = precision == SPH_PRECISION_F32 || (precision == 2 && !root.not_f32);
  const float rmax = compute_rmax(root, 0, 0.0);
  int n_nodes = 0;
  rc = stage_tree(ctx, (int)n, precision, compute_f32, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, ctx->in_m.p, 1, rmax,
                  &n_nodes, &launches, true);
  if (rc) return rc;
  sph_params prm{};
  PassArgs a = base_args(ctx, (int)n, 1, n_nodes, &prm, rmax);
  rc = prepare_target_tree(ctx, (int)n, n_nodes, a);
  if (rc) return rc;
  k_gather_sorted<double><<<nblk(n), kTB, 0, s>>>((int)n, ctx->perm.p, ctx->io_h.p, ctx->hfix.p);
  struct Tmp {  // per-call workspace, freed on every return path
    DevBuf<int64_t> d_off, idx_a, idx_b;
    DevBuf<double> d2_a, d2_b;
    DevBuf<unsigned char> temp;
    DevBuf<int> err;
    ~Tmp() { d_off.release(); idx_a.release(); idx_b.release(); d2_a.release(); d2_b.release(); temp.release(); err.release(); }
  } tmp;
  auto &d_off = tmp.d_off, &idx_a = tmp.idx_a, &idx_b = tmp.idx_b;
  auto &d2_a = tmp.d2_a, &d2_b = tmp.d2_b;
  auto &temp = tmp.temp;
  auto &err = tmp.err;
  const size_t tneed = range_sort_temp((int)n, total);
  SPH_CK(d_off.ensure(n + 1));
  SPH_CK(idx_a.ensure(total + 1));
  SPH_CK(idx_b.ensure(total + 1));
  SPH_CK(d2_a.ensure(total + 1));
  SPH_CK(d2_b.ensure(total + 1));
  SPH_CK(temp.ensure(tneed + 1));
  SPH_CK(err.ensure(1));
  SPH_CK(cudaMemcpyAsync(d_off.p, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemsetAsync(err.p, 0, sizeof(int), s));
  if (range_fill(s, compute_f32, (int)n, ctx->perm.p, ctx->pos_sorted.p, ctx->hfix.p, a.tree, d_off.p, total,
                 idx_b.p, d2_b.p, err.p, temp.p, tneed + 1, idx_a.p, d2_a.p, ctx->num_sms) != 0)
    return fail(ctx, SPH_CUDA_ERROR, "range query: sort workspace too small");
  int herr = 0;
  SPH_CK(cudaMemcpyAsync(&herr, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  if (total > 0) {
    SPH_CK(cudaMemcpyAsync(idx_out, idx_b.p, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, s));
    SPH_CK(cudaMemcpyAsync(d2_out, d2_b.p, sizeof(double) * total, cudaMemcpyDeviceToHost, s));
  }
  SPH_CK(cudaStreamSynchronize(s));
  SPH_CK(cudaGetLastError());
  if (herr) return fail(ctx, SPH_INVALID, "range query: the offsets do not match the fixed-h neighbour counts");
  return SPH_OK;
}

int sph_octree_build(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z) {
  if (!ctx) return SPH_INVALID;
  if (n < 1) return fail(ctx, SPH_INVALID, "need at least one particle");
  if (n > (int64_t(1) << 27)) return fail(ctx, SPH_INVALID, "n must be <= 2^27 per device");
  if (precision < 0 || precision > 2) return fail(ctx, SPH_INVALID, "unknown precision");
  if (!x || !y || !z) return fail(ctx, SPH_INVALID, "null array pointer");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = ensure_common(ctx, n, 1);
  if (rc) return rc;
  const size_t es = elem_size(precision);
  SPH_CK(ctx->in_x.ensure(n));
  SPH_CK(ctx->in_y.ensure(n));
  SPH_CK(ctx->in_z.ensure(n));
  SPH_CK(ctx->in_m.ensure(n));
  cudaStream_t s = ctx->stream;
  SPH_CK(cudaMemcpyAsync(ctx->in_x.p, x, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_y.p, y, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_z.p, z, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemsetAsync(ctx->in_m.p, 0, 8 * n, s));
  int launches = 0;
  RootInfo root{};
  rc = stage_root(ctx, (int)n, precision, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, &root, &launches);
  if (rc) return rc;
  const int compute_f32 = precision == SPH_PRECISION_F32 || (precision == 2 && !root.not_f32);
  const float rmax = compute_rmax(root, 0, 0.0);
  int n_nodes = 0;
  rc = stage_tree(ctx, (int)n, precision, compute_f32, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, ctx->in_m.p, 1, rmax,
                  &n_nodes, &launches, true);
  if (rc) return rc;
  sph_params prm{};
  PassArgs a = base_args(ctx, (int)n, 1, n_nodes, &prm, rmax);
  rc = prepare_target_tree(ctx, (int)n, n_nodes, a);
  if (rc) return rc;
  SPH_CK(cudaStreamSynchronize(s));
  SPH_CK(cudaGetLastError());
  ctx->octree_args = a;
  ctx->octree_f32 = compute_f32;
  ctx->octree_n = n;
  return SPH_OK;
}

int sph_octree_query(sph_ctx *ctx, int64_t m, const double *centers, const double *radii, const int64_t *exclude,
                     int64_t cap, int64_t *offsets_out, int64_t *idx_out, double *d2_out, int64_t *total_out) {
  if (!ctx) return SPH_INVALID;
  if (ctx->octree_n < 0) return fail(ctx, SPH_INVALID, "no octree on this context (sph_octree_build first)");
  if (m < 0) return fail(ctx, SPH_INVALID, "query count must be >= 0");
  if (!offsets_out || (m > 0 && (!centers || !radii))) return fail(ctx, SPH_INVALID, "null array pointer");
  for (int64_t q = 0; q < m; ++q)
    if (!(radii[q] >= 0.0)) {
      char buf[128];
      snprintf(buf, sizeof(buf), "radius must be non-negative, got %g", radii[q]);
      return fail(ctx, SPH_INVALID, buf);
    }
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  offsets_out[0] = 0;
  if (total_out) *total_out = 0;
  if (m == 0) return SPH_OK;
  cudaStream_t s = ctx->stream;
  struct Tmp {  // per-call workspace, freed on every return path
    DevBuf<double> cen, rad, d2a, d2b;
    DevBuf<int64_t> exc, cnt, off, ia, ib;
    DevBuf<unsigned char> temp;
    DevBuf<int> err;
    ~Tmp() { cen.release(); rad.release(); d2a.release(); d2b.release(); exc.release(); cnt.release(); off.release();
             ia.release(); ib.release(); temp.release(); err.release(); }
  } t;
  SPH_CK(t.cen.ensure(3 * m));
  SPH_CK(t.rad.ensure(m));
  SPH_CK(t.cnt.ensure(m));
  SPH_CK(t.off.ensure(m + 1));
  SPH_CK(t.err.ensure(1));
  SPH_CK(cudaMemcpyAsync(t.cen.p, centers, 24 * m, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(t.rad.p, radii, 8 * m, cudaMemcpyHostToDevice, s));
  const int64_t *d_exc = nullptr;
  if (exclude) {
    SPH_CK(t.exc.ensure(m));
    SPH_CK(cudaMemcpyAsync(t.exc.p, exclude, 8 * m, cudaMemcpyHostToDevice, s));
    d_exc = t.exc.p;
  }
  SPH_CK(cudaMemsetAsync(t.err.p, 0, sizeof(int), s));
  const PassArgs &a = ctx->octree_args;
  range_points(s, ctx->octree_f32, 1, m, t.cen.p, t.rad.p, d_exc, ctx->perm.p, ctx->pos_sorted.p, a.tree, nullptr,
               t.cnt.p, nullptr, nullptr, t.err.p, ctx->num_sms);
  std::vector<int64_t> cnt(m);
  int herr = 0;
  SPH_CK(cudaMemcpyAsync(cnt.data(), t.cnt.p, 8 * m, cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaMemcpyAsync(&herr, t.err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaStreamSynchronize(s));
  if (herr) return fail(ctx, SPH_CUDA_ERROR, "range query: traversal stack overflow");
  for (int64_t q = 0; q < m; ++q) offsets_out[q + 1] = offsets_out[q] + cnt[q];
  const int64_t total = offsets_out[m];
  if (total_out) *total_out = total;
  if (total > cap) return fail(ctx, SPH_INVALID, "range query: results exceed the output capacity (see total)");
  if (total == 0) return SPH_OK;
  if (!idx_out || !d2_out) return fail(ctx, SPH_INVALID, "null output array");
  SPH_CK(t.ia.ensure(total));
  SPH_CK(t.ib.ensure(total));
  SPH_CK(t.d2a.ensure(total));
  SPH_CK(t.d2b.ensure(total));
  const size_t need = range_sort_temp((int)m, total);
  SPH_CK(t.temp.ensure(need + 1));
  SPH_CK(cudaMemcpyAsync(t.off.p, offsets_out, 8 * (m + 1), cudaMemcpyHostToDevice, s));
  range_points(s, ctx->octree_f32, 0, m, t.cen.p, t.rad.p, d_exc, ctx->perm.p, ctx->pos_sorted.p, a.tree, t.off.p,
               nullptr, t.ia.p, t.d2a.p, t.err.p, ctx->num_sms);
  if (segmented_sort_pairs(s, m, total, t.off.p, t.ia.p, t.ib.p, t.d2a.p, t.d2b.p, t.temp.p, need + 1) != 0)
    return fail(ctx, SPH_CUDA_ERROR, "range query: sort workspace too small");
  SPH_CK(cudaMemcpyAsync(idx_out, t.ib.p, 8 * total, cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaMemcpyAsync(d2_out, t.d2b.p, 8 * total, cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaMemcpyAsync(&herr, t.err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaStreamSynchronize(s));
  SPH_CK(cudaGetLastError());
  if (herr) return fail(ctx, SPH_CUDA_ERROR, "range query: list lengths changed between the count and fill passes");
  return SPH_OK;
}

int sph_morton_keys_device(sph_ctx *ctx, int32_t precision, int64_t n, const void *d_x, const void *d_y,
                           const void *d_z, const double *centre, double half, uint64_t *d_keys) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || n >= (1ll << 31)) return fail(ctx, SPH_INVALID, "n must be in [0, 2^31)");
  if (precision != SPH_PRECISION_F32 && precision != SPH_PRECISION_F64)
    return fail(ctx, SPH_INVALID, "precision must be f32 or f64");
  if (!centre || !(half >= 0.0)) return fail(ctx, SPH_INVALID, "need a root centre and half-extent >= 0");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_keys_at(ctx->stream, (int)n, precision == SPH_PRECISION_F32 ? 1 : 0, d_x, d_y, d_z, centre, half,
                 reinterpret_cast<unsigned long long *>(d_keys));
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_pack_rows_device(sph_ctx *ctx, int32_t precision, int64_t n, const int64_t *d_order,
                                const void *d_x, const void *d_y, const void *d_z, const double *d_mass,
                                const double *d_h0, const int64_t *d_gid, const int64_t *d_keys, double *d_rows) {
  if (!ctx) return SPH_INVALID;
  if (n < 0) return fail(ctx, SPH_INVALID, "n must be >= 0");
  if (precision != SPH_PRECISION_F32 && precision != SPH_PRECISION_F64)
    return fail(ctx, SPH_INVALID, "precision must be f32 or f64");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_pack_rows(ctx->stream, n, precision == SPH_PRECISION_F32 ? 1 : 0, d_order, d_x, d_y, d_z, d_mass, d_h0,
                   d_gid, d_keys, d_rows);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_gather_rows_device(sph_ctx *ctx, int64_t n, int32_t width, const int64_t *d_idx,
                                  const double *d_src, double *d_dst) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || width < 1) return fail(ctx, SPH_INVALID, "need n >= 0 and width >= 1");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_gather_rows(ctx->stream, n, width, d_idx, d_src, d_dst);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_row_keys_device(sph_ctx *ctx, int64_t n, const double *d_rows, int64_t *d_keys) {
  if (!ctx) return SPH_INVALID;
  if (n < 0) return fail(ctx, SPH_INVALID, "n must be >= 0");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_row_keys(ctx->stream, n, d_rows, d_keys);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_level_bounds_device(sph_ctx *ctx, int64_t n, int32_t k, const int64_t *d_keys_sorted, double half,
                                   double *d_bound) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || k < 1) return fail(ctx, SPH_INVALID, "need n >= 0 and k >= 1");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_level_bounds(ctx->stream, n, k, d_keys_sorted, 2.0 * half, d_bound);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_window_bounds_device(sph_ctx *ctx, int64_t n, int32_t k, int32_t width, const double *d_rows,
                                    double max_abs_coord, double *d_bound) {
  if (!ctx) return SPH_INVALID;
  if (n < 0 || k < 1 || k > 1024 || width < 3) return fail(ctx, SPH_INVALID, "need n >= 0, 1 <= k <= 1024, width >= 3");
  if (!(max_abs_coord >= 0.0)) return fail(ctx, SPH_INVALID, "max_abs_coord must be >= 0");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  // fp32 coordinates are within 2^-24 |x| of the records: 4 such errors per difference, with room
  launch_window_bounds(ctx->stream, n, k, width, d_rows, max_abs_coord * 1e-6 + 1e-30, d_bound);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_ghost_mask_device(sph_ctx *ctx, int64_t n_groups, const double *d_gdesc, const int64_t *d_gstart,
                                 const int64_t *d_gcount, int32_t width, const double *d_rows, int64_t n_foreign,
                                 const double *d_fdesc, const int32_t *d_frank, int32_t periodic, double box,
                                 uint32_t *d_mask) {
  if (!ctx) return SPH_INVALID;
  if (n_groups < 0 || n_foreign < 0 || width < 3) return fail(ctx, SPH_INVALID, "bad ghost-mask arguments");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  SPH_CK(ctx->dscratch.ensure(7 * ((n_foreign + 31) / 32) + 7 * ((n_foreign + 1023) / 1024) + 14));
  launch_ghost_mask(ctx->stream, n_groups, d_gdesc, d_gstart, d_gcount, width, d_rows, n_foreign, d_fdesc, d_frank,
                    periodic, box, d_mask, ctx->dscratch.p);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_decomp_group_boxes_device(sph_ctx *ctx, int64_t n_groups, const int64_t *d_starts, const int64_t *d_counts,
                                  int32_t width, const double *d_rows, const double *d_bound, double *d_out) {
  if (!ctx) return SPH_INVALID;
  if (n_groups < 0 || width < 3) return fail(ctx, SPH_INVALID, "need n_groups >= 0 and width >= 3");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  launch_group_boxes(ctx->stream, n_groups, d_starts, d_counts, width, d_rows, d_bound, d_out);
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_bbox_device(sph_ctx *ctx, int32_t precision, int64_t n, const void *d_x, const void *d_y, const void *d_z,
                    double *d_out) {
  if (!ctx) return SPH_INVALID;
  if (n < 1 || n >= (1ll << 31)) return fail(ctx, SPH_INVALID, "n must be in [1, 2^31)");
  if (precision != SPH_PRECISION_F32 && precision != SPH_PRECISION_F64)
    return fail(ctx, SPH_INVALID, "precision must be f32 or f64");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = ensure_common(ctx, n, 1);
  if (rc) return rc;
  int launches = 0;
  launch_bbox(ctx->stream, (int)n, precision == SPH_PRECISION_F32 ? 1 : 0, d_x, d_y, d_z, ctx->bbox_ord.p,
              ctx->root.p, &launches);
  SPH_CK(cudaMemcpyAsync(d_out, ctx->root.p->lo, 3 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  SPH_CK(cudaMemcpyAsync(d_out + 3, ctx->root.p->hi, 3 * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  SPH_CK(cudaGetLastError());
  return SPH_OK;
}

int sph_sort_perm(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z,
                  int64_t *perm_out) {
  return sph_sort_perm_ex(ctx, precision, n, x, y, z, 8, perm_out);
}

int sph_sort_perm_ex(sph_ctx *ctx, int32_t precision, int64_t n, const void *x, const void *y, const void *z,
                     int32_t leaf_capacity, int64_t *perm_out) {
  if (!ctx) return SPH_INVALID;
  if (leaf_capacity < 1) return fail(ctx, SPH_INVALID, "leaf_capacity must be >= 1");
  if (leaf_capacity > kMaxLeafCap) return fail(ctx, SPH_UNSUPPORTED, "leaf_capacity above 32 is not supported");
  if (n < 1) return fail(ctx, SPH_INVALID, "need at least one particle");
  if (n >= (1ll << 31) - 64) return fail(ctx, SPH_INVALID, "n must be < 2^31 per device");
  if (precision != SPH_PRECISION_F32 && precision != SPH_PRECISION_F64)
    return fail(ctx, SPH_INVALID, "precision must be f32 or f64");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  int rc = ensure_common(ctx, n, 1);
  if (rc) return rc;
  const size_t es = elem_size(precision);
  SPH_CK(ctx->in_x.ensure(n));
  SPH_CK(ctx->in_y.ensure(n));
  SPH_CK(ctx->in_z.ensure(n));
  cudaStream_t s = ctx->stream;
  SPH_CK(cudaMemcpyAsync(ctx->in_x.p, x, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_y.p, y, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_z.p, z, es * n, cudaMemcpyHostToDevice, s));
  int launches = 0;
  RootInfo root{};
  rc = stage_root(ctx, (int)n, precision, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, &root, &launches);
  if (rc) return rc;
  int n_nodes = 0;
  ctx->leaf_cap = leaf_capacity;
  rc = stage_tree(ctx, (int)n, precision, 0, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, nullptr, 1, 1.f, &n_nodes,
                  &launches, false);
  ctx->leaf_cap = 8;
  if (rc) return rc;
  std::vector<uint32_t> tmp(n);
  SPH_CK(cudaMemcpyAsync(tmp.data(), ctx->perm.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) perm_out[i] = (int64_t)tmp[i];
  return SPH_OK;
}

int sph_neighbor_counts(sph_ctx *ctx, int32_t precision, int32_t periodic, double box, int64_t n, const void *x,
                        const void *y, const void *z, const double *h, int32_t *counts_out, sph_stats *st) {
  if (!ctx) return SPH_INVALID;
  if (n < 1) return fail(ctx, SPH_INVALID, "need at least one particle");
  if (n >= (1ll << 31) - 64) return fail(ctx, SPH_INVALID, "n must be < 2^31 per device");
  if (precision < 0 || precision > 2) return fail(ctx, SPH_INVALID, "unknown precision");
  cudaSetDevice(ctx->device);
  ctx->err.clear();
  if (st) memset(st, 0, sizeof(*st));
  int rc = ensure_common(ctx, n, 1);
  if (rc) return rc;
  const size_t es = elem_size(precision);
  SPH_CK(ctx->in_x.ensure(n));
  SPH_CK(ctx->in_y.ensure(n));
  SPH_CK(ctx->in_z.ensure(n));
  SPH_CK(ctx->in_m.ensure(n));
  SPH_CK(ctx->io_h.ensure(n));
  SPH_CK(ctx->hfix.ensure(n));
  SPH_CK(ctx->counts_s.ensure(n));
  SPH_CK(ctx->counts_o.ensure(n));
  cudaStream_t s = ctx->stream;
  SPH_CK(cudaMemcpyAsync(ctx->in_x.p, x, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_y.p, y, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->in_z.p, z, es * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemcpyAsync(ctx->io_h.p, h, 8 * n, cudaMemcpyHostToDevice, s));
  SPH_CK(cudaMemsetAsync(ctx->in_m.p, 0, 8 * n, s));
  int launches = 0;
  RootInfo root{};
  rc = stage_root(ctx, (int)n, precision, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, &root, &launches);
  if (rc) return rc;
  if (periodic) {
    if (!(box > 0.0)) return fail(ctx, SPH_INVALID, "periodic box side must be > 0");
    for (int a2 = 0; a2 < 3; ++a2)
      if (root.lo[a2] < 0.0 || root.hi[a2] >= box)
        return fail(ctx, SPH_INVALID, "periodic mode needs every position inside [0, box)");
  }
  const int compute_f32 = precision == SPH_PRECISION_F32 || (precision == 2 && !root.not_f32);
  const float rmax = compute_rmax(root, periodic, box);
  int n_nodes = 0;
  rc = stage_tree(ctx, (int)n, precision, compute_f32, ctx->in_x.p, ctx->in_y.p, ctx->in_z.p, ctx->in_m.p, 1, rmax,
                  &n_nodes, &launches, true);
  if (rc) return rc;
  k_gather_sorted<double><<<nblk(n), kTB, 0, s>>>((int)n, ctx->perm.p, ctx->io_h.p, ctx->hfix.p);
  SPH_CK(cudaMemsetAsync(ctx->stats.p, 0, 4 * sizeof(unsigned long long), s));
  sph_params prm{};
  prm.periodic = periodic;
  prm.box = box;
  PassArgs a = base_args(ctx, (int)n, 1, n_nodes, &prm, rmax);
  launch_pass(s, MODE_COUNT, compute_f32, a, (int)n, 0, ctx->num_sms);
  k_scatter_orig<int32_t><<<nblk(n), kTB, 0, s>>>((int)n, ctx->perm.p, ctx->counts_s.p, ctx->counts_o.p);
  launches += 3;
  SPH_CK(cudaMemcpyAsync(counts_out, ctx->counts_o.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
  unsigned long long stat_all[2] = {0, 0};
  SPH_CK(cudaMemcpyAsync(stat_all, ctx->stats.p, sizeof(stat_all), cudaMemcpyDeviceToHost, s));
  SPH_CK(cudaStreamSynchronize(s));
  SPH_CK(cudaGetLastError());
  if (st) {
    st->pair_tests = (int64_t)stat_all[0];
    st->gpu_launches = launches;
    st->n_nodes = n_nodes;
  }
  return SPH_OK;
}

}  // extern "C"
