// sph_tree.cu -- particle ordering and search tree.
//
//  1. root cube + pad exactly as the reference (octree.py:324-336)
//  2. 63-bit x-major Morton keys descended with the reference's own fp64
//     centre arithmetic (octree.py:93-104, 143-149), so every octant
//     decision equals the reference's
//  3. LSD radix sort of (key, original index) -- stable, so ties keep
//     original-index order like the reference's stable counting sorts
//  4. leaf detection for leaf capacity 8 (and the coincident-point guard,
//     octree.py:75-86) and re-ordering inside each leaf by original index:
//     the result is Octree.particle_perm bit-for-bit
//  5. the search tree: cells = maximal octree nodes with <= 32 particles,
//     internal nodes above them, laid out in pre-order with skip pointers
//     (a stackless walk); cell boxes are tight, internal boxes are the
//     padded octree cubes
#include "sph_internal.cuh"


namespace sph {

namespace {

constexpr int kTB = 256;

__device__ __forceinline__ bool is_f32_exact(double v) { return (double)(float)v == v; }

template <typename PosT>
__global__ void k_bbox(int n, const PosT *__restrict__ x, const PosT *__restrict__ y,
                       const PosT *__restrict__ z, unsigned long long *ord, RootInfo *root) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int bad = 0, notf = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v[3] = {(double)x[i], (double)y[i], (double)z[i]};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (!isfinite(v[a])) { bad = 1; continue; }
      notf |= !is_f32_exact(v[a]);
      mn[a] = fmin(mn[a], v[a]);
      mx[a] = fmax(mx[a], v[a]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o; o >>= 1) {
      mn[a] = fmin(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = fmax(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  notf = __any_sync(0xffffffffu, notf);
  // block reduction first: one set of global atomics per block, not per warp
  __shared__ double s_mn[3][32], s_mx[3][32];
  __shared__ int s_bad, s_notf;
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) s_bad = s_notf = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s_mn[a][w] = mn[a];
      s_mx[a][w] = mx[a];
    }
    if (bad) atomicOr(&s_bad, 1);
    if (notf) atomicOr(&s_notf, 1);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int l = threadIdx.x;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double v = l < nw ? s_mn[a][l] : INFINITY, u = l < nw ? s_mx[a][l] : -INFINITY;
      for (int o = 16; o; o >>= 1) {
        v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
        u = fmax(u, __shfl_xor_sync(0xffffffffu, u, o));
      }
      if (l == 0) {
        atomicMin(&ord[a], dbl_to_ord(v));
        atomicMax(&ord[3 + a], dbl_to_ord(u));
      }
    }
    if (l == 0 && s_bad) atomicOr(&root->nonfinite, 1);
    if (l == 0 && s_notf) atomicOr(&root->not_f32, 1);
  }
}

// octree.py:324-336: lo/hi, centre = 0.5*(lo+hi), half = 0.5*max(hi-lo),
// pad = 8*eps*(max_abs + half)
__global__ void k_root(int n, const unsigned long long *ord, RootInfo *root) {
  if (threadIdx.x || blockIdx.x) return;
  double ext = 0.0, max_abs = 0.0;
  for (int a = 0; a < 3; ++a) {
    double lo = n ? ord_to_dbl(ord[a]) : 0.0, hi = n ? ord_to_dbl(ord[3 + a]) : 0.0;
    root->lo[a] = lo;
    root->hi[a] = hi;
    root->c[a] = __dmul_rn(0.5, __dadd_rn(lo, hi));
    double e = __dsub_rn(hi, lo);
    ext = (a == 0 || e > ext) ? e : ext;
    max_abs = fmax(max_abs, fmax(fabs(lo), fabs(hi)));
  }
  root->half = __dmul_rn(ext, 0.5);
  root->max_abs = max_abs;
  root->pad = __dmul_rn(__dmul_rn(8.0, 2.220446049250313e-16), __dadd_rn(max_abs, root->half));
}

template <typename PosT>
__global__ void k_keys(int n, const PosT *__restrict__ x, const PosT *__restrict__ y,
                       const PosT *__restrict__ z, const RootInfo *__restrict__ root,
                       unsigned long long *__restrict__ keys, uint32_t *__restrict__ idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = (double)x[i], py = (double)y[i], pz = (double)z[i];
  double cx = root->c[0], cy = root->c[1], cz = root->c[2], half = root->half;
  unsigned long long key = 0;
#pragma unroll
  for (int l = 0; l < kMaxLevel; ++l) {
    const int bx = px >= cx, by = py >= cy, bz = pz >= cz;
    key = (key << 3) | (unsigned long long)((bx << 2) | (by << 1) | bz);
    const double h2 = __dmul_rn(half, 0.5);
    cx = bx ? __dadd_rn(cx, h2) : __dsub_rn(cx, h2);
    cy = by ? __dadd_rn(cy, h2) : __dsub_rn(cy, h2);
    cz = bz ? __dadd_rn(cz, h2) : __dsub_rn(cz, h2);
    half = h2;
  }
  keys[i] = key;
  idx[i] = (uint32_t)i;
}

// Leaf level for capacity C: the group sharing the 3L-bit prefix has > C
// members iff some window of C+1 consecutive sorted keys containing p has
// common prefix >= 3L.  M(p) = max over those windows of cpl(key[s], key[s+C]);
// level = floor(M/3) + 1 (0 when no full window exists).
__global__ void k_levels(int n, const unsigned long long *__restrict__ keys, uint8_t *__restrict__ lvl8,
                         uint8_t *__restrict__ lvl32, int *deep_count, uint32_t *deep_list, int cap) {
  constexpr int H = kCellCap > 32 ? kCellCap : 32;  // window halo
  __shared__ unsigned long long sk[kTB + 2 * H];
  __shared__ int w8[kTB + H], w32[kTB + H];
  const int b0 = blockIdx.x * kTB;
  for (int t = threadIdx.x; t < kTB + 2 * H; t += kTB) {
    int q = b0 - H + t;
    sk[t] = (q >= 0 && q < n) ? keys[q] : 0ull;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kTB + H; t += kTB) {
    int s = b0 - H + t;  // window start
    w8[t] = (s >= 0 && s + cap <= n - 1) ? key_cpl(sk[t], sk[t + cap]) : -1;
    w32[t] = (s >= 0 && s + kCellCap <= n - 1) ? key_cpl(sk[t], sk[t + kCellCap]) : -1;
  }
  __syncthreads();
  const int p = b0 + threadIdx.x;
  if (p >= n) return;
  const int tp = threadIdx.x + H;  // index of window starting at p
  int m8 = -1, m32 = -1;
  for (int d = 0; d <= cap; ++d) m8 = max(m8, w8[tp - d]);
#pragma unroll 8
  for (int d = 0; d <= kCellCap; ++d) m32 = max(m32, w32[tp - d]);
  int l8 = m8 < 0 ? 0 : m8 / 3 + 1;
  int l32 = m32 < 0 ? 0 : m32 / 3 + 1;
  if (l8 > kMaxLevel) {
    l8 = kMaxLevel + 1;  // > cap identical 63-bit keys: resolved by k_deep
    int slot = atomicAdd(deep_count, 1);
    deep_list[slot] = (uint32_t)p;
  }
  lvl8[p] = (uint8_t)l8;
  lvl32[p] = (uint8_t)min(l32, kMaxLevel);
}

// Runs of > 8 identical 63-bit keys.  If every position in the run is the
// same point the reference keeps it as one non-separable leaf (octree.py:
// 75-86) at the first level where no other particle shares its prefix.
// Otherwise the reference tree goes below the 21 levels of the key: the run
// is subdivided here exactly as octree.py:36-176 does it (stable 8-way
// partitions by x-major octant with the reference's fp64 centre arithmetic,
// from the depth-21 cell down to MAX_TREE_DEPTH = 48, leaves at <= 8 members
// or non-separable), writing the run's slice of the particle order directly;
// its members keep lvl8 = kMaxLevel + 1 so k_leaf_order leaves them alone.
// Such a run stays one search cell (its particles share all 63 key bits); the
// search kernels take cells of any size.
constexpr int kMaxDepth = 48;  // octree.py:31
struct DeepSeg { int s, e, depth; double cx, cy, cz, half; };
constexpr int kDeepStack = 8 * (kMaxDepth - kMaxLevel) + 8;  // segments per thread (depth-first)
constexpr int kDeepThreads = 256;                             // k_deep grid (runs are rare)
template <typename PosT>
__global__ void k_deep(int n, const unsigned long long *__restrict__ keys, const uint32_t *__restrict__ idx,
                       const PosT *__restrict__ x, const PosT *__restrict__ y, const PosT *__restrict__ z,
                       const RootInfo *__restrict__ root, const int *deep_count, const uint32_t *deep_list,
                       uint8_t *lvl8, uint32_t *__restrict__ perm, uint32_t *__restrict__ scratch,
                       DeepSeg *__restrict__ segs, int *err_flag, int cap) {
  const int cnt = *deep_count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int p = (int)deep_list[t];
    const unsigned long long kp = keys[p];
    if (p > 0 && keys[p - 1] == kp) continue;  // only the run's first member works
    int e = p + 1;
    while (e < n && keys[e] == kp) ++e;
    const uint32_t j0 = idx[p];
    bool same = true;
    for (int q = p + 1; q < e && same; ++q) {
      const uint32_t j = idx[q];
      same = x[j] == x[j0] && y[j] == y[j0] && z[j] == z[j0];
    }
    if (same) {
      const int cl = p > 0 ? key_cpl(keys[p - 1], kp) : -1;
      const int cr = e < n ? key_cpl(keys[e - 1], keys[e]) : -1;
      const int m = max(cl, cr);
      const int L = m < 0 ? 0 : m / 3 + 1;
      for (int q = p; q < e; ++q) lvl8[q] = (uint8_t)L;
      continue;
    }
    // the depth-21 cell of the run: the key's own descent (k_keys arithmetic)
    double cx = root->c[0], cy = root->c[1], cz = root->c[2], half = root->half;
    for (int l = 0; l < kMaxLevel; ++l) {
      const unsigned o = (unsigned)(kp >> (60 - 3 * l)) & 7u;
      const double h2 = __dmul_rn(half, 0.5);
      cx = (o & 4u) ? __dadd_rn(cx, h2) : __dsub_rn(cx, h2);
      cy = (o & 2u) ? __dadd_rn(cy, h2) : __dsub_rn(cy, h2);
      cz = (o & 1u) ? __dadd_rn(cz, h2) : __dsub_rn(cz, h2);
      half = h2;
    }
    // inside a node the reference keeps the parent's stable order; at depth
    // 21 that is original-index order, which the stable key sort left in idx
    DeepSeg *stk = segs + (size_t)(blockIdx.x * blockDim.x + threadIdx.x) * kDeepStack;  // global, per thread
    int sp = 0;
    stk[sp++] = DeepSeg{p, e, kMaxLevel, cx, cy, cz, half};
    while (sp > 0) {
      const DeepSeg g = stk[--sp];
      if (g.e - g.s <= cap || g.depth >= kMaxDepth) continue;
      const uint32_t f = perm[g.s];
      bool sep = false;
      for (int q = g.s + 1; q < g.e && !sep; ++q) {
        const uint32_t j = perm[q];
        sep = x[j] != x[f] || y[j] != y[f] || z[j] != z[f];
      }
      if (!sep) continue;  // coincident-point guard (octree.py:75-86)
      int counts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int q = g.s; q < g.e; ++q) {
        const uint32_t j = perm[q];
        const int o = (((double)x[j] >= g.cx) << 2) | (((double)y[j] >= g.cy) << 1) | ((double)z[j] >= g.cz);
        ++counts[o];
      }
      int offs[9];
      offs[0] = 0;
      for (int o = 0; o < 8; ++o) offs[o + 1] = offs[o] + counts[o];
      int cur[8];
      for (int o = 0; o < 8; ++o) cur[o] = offs[o];
      for (int q = g.s; q < g.e; ++q) {
        const uint32_t j = perm[q];
        const int o = (((double)x[j] >= g.cx) << 2) | (((double)y[j] >= g.cy) << 1) | ((double)z[j] >= g.cz);
        scratch[g.s + cur[o]++] = j;
      }
      for (int q = g.s; q < g.e; ++q) perm[q] = scratch[q];
      const double h2 = __dmul_rn(g.half, 0.5);
      for (int o = 0; o < 8; ++o) {
        if (counts[o] <= cap) continue;
        stk[sp++] = DeepSeg{g.s + offs[o], g.s + offs[o + 1], g.depth + 1,
                        (o & 4) ? __dadd_rn(g.cx, h2) : __dsub_rn(g.cx, h2),
                        (o & 2) ? __dadd_rn(g.cy, h2) : __dsub_rn(g.cy, h2),
                        (o & 1) ? __dadd_rn(g.cz, h2) : __dsub_rn(g.cz, h2), h2};
      }
    }
  }
}

__device__ __forceinline__ bool same_leaf(const unsigned long long *keys, const uint8_t *lvl, int a, int b) {
  const int la = lvl[a];
  return la == lvl[b] && key_prefix(keys[a], la) == key_prefix(keys[b], la);
}

// inside each leaf the reference keeps original-index order (stable
// partitions from an identity perm); the key sort ordered them by key
__global__ void k_leaf_order(int n, const unsigned long long *__restrict__ keys, const uint8_t *__restrict__ lvl8,
                             const uint32_t *__restrict__ idx, uint32_t *__restrict__ perm, int cap) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (lvl8[p] > kMaxLevel) return;  // a run below depth 21: ordered by k_deep
  if (p > 0 && same_leaf(keys, lvl8, p - 1, p)) return;
  uint32_t v[kMaxLeafCap];
  int c = 0;
  while (p + c < n && c <= cap && (c == 0 || same_leaf(keys, lvl8, p, p + c))) {
    if (c < cap) v[c] = idx[p + c];
    ++c;
  }
  if (c > cap || c < 2) return;  // coincident runs are already in index order
  for (int i = 1; i < c; ++i) {
    uint32_t t = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > t) { v[j + 1] = v[j]; --j; }
    v[j + 1] = t;
  }
  for (int i = 0; i < c; ++i) perm[p + i] = v[i];
}

struct alignas(32) D4 { double x, y, z, m; };

template <typename PosT>
__global__ void k_gather_f32(int n, const uint32_t *__restrict__ perm, const PosT *__restrict__ x,
                             const PosT *__restrict__ y, const PosT *__restrict__ z,
                             const double *__restrict__ mass, float4 *__restrict__ out,
                             double *__restrict__ mass_out, float4 *__restrict__ posj) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t o = perm[p];
  const double m = mass[o];
  const float fx = (float)x[o], fy = (float)y[o], fz = (float)z[o];
  out[p] = make_float4(fx, fy, fz, (float)m);
  mass_out[p] = m;
  if (posj) posj[p] = make_float4(fx, fy, fz, __uint_as_float((unsigned)p));
}

template <typename PosT>
__global__ void k_gather_f64(int n, const uint32_t *__restrict__ perm, const PosT *__restrict__ x,
                             const PosT *__restrict__ y, const PosT *__restrict__ z,
                             const double *__restrict__ mass, D4 *__restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t o = perm[p];
  out[p] = D4{(double)x[o], (double)y[o], (double)z[o], mass[o]};
}

__device__ __forceinline__ int first_level(const unsigned long long *keys, int p) {
  if (p == 0) return 0;
  const int c = key_cpl(keys[p - 1], keys[p]);
  return c >= 63 ? kMaxLevel + 1 : c / 3 + 1;
}

__global__ void k_node_count(int n, const unsigned long long *__restrict__ keys,
                             const uint8_t *__restrict__ lvl32, int *__restrict__ nemit) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  if (p == n) { nemit[p] = 0; return; }
  nemit[p] = max(0, (int)lvl32[p] - first_level(keys, p) + 1);
}

// first q in [lo, n) whose key exceeds kmax (keys sorted)
__device__ __forceinline__ int upper_bound_key(const unsigned long long *keys, int lo, int n,
                                               unsigned long long kmax) {
  int hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (keys[mid] <= kmax) lo = mid + 1; else hi = mid;
  }
  return lo;
}
// first q in [0, hi) whose key is >= kmin
__device__ __forceinline__ int lower_bound_key(const unsigned long long *keys, int hi,
                                               unsigned long long kmin) {
  int lo = 0;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (keys[mid] < kmin) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ unsigned long long low_mask(int level) {
  return level == 0 ? 0x7fffffffffffffffull : ((1ull << (63 - 3 * level)) - 1ull);
}

__device__ __forceinline__ float f_rd(double v) { return __double2float_rd(v); }
__device__ __forceinline__ float f_ru(double v) { return __double2float_ru(v); }

template <bool F32>
__global__ void k_node_emit(int n, const unsigned long long *__restrict__ keys, const uint8_t *__restrict__ lvl32,
                            const int *__restrict__ noff, const RootInfo *__restrict__ root,
                            const void *__restrict__ pos_sorted, int k, float rmax, float r0_scale, float c0_scale, int emit_r0,
                            float4 *__restrict__ nlo, float4 *__restrict__ nhi, int *__restrict__ nsize,
                            float *__restrict__ r0) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int L0 = first_level(keys, p);
  const int Lc = lvl32[p];
  if (Lc < L0) return;
  const unsigned long long kp = keys[p];
  const double pad2 = 2.0 * root->pad;
  // descend centres to L0 with the reference arithmetic
  double c[3] = {root->c[0], root->c[1], root->c[2]};
  double half = root->half;
  for (int l = 1; l < L0; ++l) {
    const int o = (int)((kp >> (63 - 3 * l)) & 7ull);
    const double h2 = __dmul_rn(half, 0.5);
    c[0] = (o & 4) ? __dadd_rn(c[0], h2) : __dsub_rn(c[0], h2);
    c[1] = (o & 2) ? __dadd_rn(c[1], h2) : __dsub_rn(c[1], h2);
    c[2] = (o & 1) ? __dadd_rn(c[2], h2) : __dsub_rn(c[2], h2);
    half = h2;
  }
  int node = noff[p];
  for (int L = L0; L <= Lc; ++L, ++node) {
    if (L > 0) {
      const int o = (int)((kp >> (63 - 3 * L)) & 7ull);
      const double h2 = __dmul_rn(half, 0.5);
      c[0] = (o & 4) ? __dadd_rn(c[0], h2) : __dsub_rn(c[0], h2);
      c[1] = (o & 2) ? __dadd_rn(c[1], h2) : __dsub_rn(c[1], h2);
      c[2] = (o & 1) ? __dadd_rn(c[2], h2) : __dsub_rn(c[2], h2);
      half = h2;
    }
    const int end = (L == 0) ? n : upper_bound_key(keys, p + 1, n, kp | low_mask(L));
    const int skip = noff[end];
    float4 lo, hi;
    if (L < Lc) {
      const double e = half + pad2;
      lo = make_float4(f_rd(c[0] - e), f_rd(c[1] - e), f_rd(c[2] - e), __int_as_float(skip));
      hi = make_float4(f_ru(c[0] + e), f_ru(c[1] + e), f_ru(c[2] + e), __int_as_float(p));
    } else {
      // cell: tight box over its particles
      float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int q = p; q < end; ++q) {
        if (F32) {
          const float4 v = reinterpret_cast<const float4 *>(pos_sorted)[q];
          mn[0] = fminf(mn[0], v.x); mn[1] = fminf(mn[1], v.y); mn[2] = fminf(mn[2], v.z);
          mx[0] = fmaxf(mx[0], v.x); mx[1] = fmaxf(mx[1], v.y); mx[2] = fmaxf(mx[2], v.z);
        } else {
          const D4 v = reinterpret_cast<const D4 *>(pos_sorted)[q];
          mn[0] = fminf(mn[0], f_rd(v.x)); mn[1] = fminf(mn[1], f_rd(v.y)); mn[2] = fminf(mn[2], f_rd(v.z));
          mx[0] = fmaxf(mx[0], f_ru(v.x)); mx[1] = fmaxf(mx[1], f_ru(v.y)); mx[2] = fmaxf(mx[2], f_ru(v.z));
        }
      }
      lo = make_float4(mn[0], mn[1], mn[2], __int_as_float(skip));
      hi = make_float4(mx[0], mx[1], mx[2], __int_as_float(p));
      if (!emit_r0) {  // the per-target path computes R0 from the node sizes (k_r0)
        nlo[node] = lo;
        nhi[node] = hi;
        nsize[node] = end - p;
        continue;
      }
      // Initial search radius.  Density estimates from the smallest ancestors
      // holding >= K/2 and >= 2K particles; the smaller of the two (an
      // under-estimate costs one cheap retry, an over-estimate costs a large
      // candidate volume), capped by the guaranteed bound sqrt(3)*side of the
      // smallest ancestor holding >= K+1 particles.
      double est_a = 0.0, est_b = 0.0, bound = 0.0;
      for (int La = L; La >= 0; --La) {
        int cnt;
        if (La == 0) {
          cnt = n;
        } else {
          const unsigned long long kmin = kp & ~low_mask(La);
          const int s = lower_bound_key(keys, p + 1, kmin);
          const int e2 = upper_bound_key(keys, p + 1, n, kp | low_mask(La));
          cnt = e2 - s;
        }
        const double side = fmax(2.0 * ldexp(root->half, -La), 1e-300);
        const double est = side * cbrt(3.0 * k / (4.0 * 3.14159265358979323846 * (double)max(cnt, 1)));
        if (est_a == 0.0 && (cnt >= (k + 1) / 2 || La == 0)) est_a = est;
        if (bound == 0.0 && (cnt >= k + 1 || La == 0)) bound = 1.7320508075688772 * side * (1.0 + 1e-6);
        if (cnt >= 2 * k || La == 0) { est_b = est; break; }
      }
      // tight-box density of the cell itself: small dense clumps that sit in a
      // large, mostly empty ancestor are otherwise over-estimated by far
      double est_c = INFINITY;
      if (end - p >= 4) {
        const double side_c = 2.0 * ldexp(root->half, -L);
        const double fl = 0.05 * side_c;
        const double vol = fmax((double)mx[0] - mn[0], fl) * fmax((double)mx[1] - mn[1], fl) *
                           fmax((double)mx[2] - mn[2], fl);
        est_c = cbrt(3.0 * k * vol / (4.0 * 3.14159265358979323846 * (double)(end - p)));
      }
      float R = (float)fmin(fmin(r0_scale * fmin(est_a, est_b), c0_scale * est_c), bound);
      if (!(R > 0.f)) R = rmax;
      R = fminf(R, rmax);
      for (int q = p; q < end; ++q) r0[q] = R;
    }
    nlo[node] = lo;
    nhi[node] = hi;
    nsize[node] = end - p;
  }
}

// per-node form of k_node_emit for the per-target path (no R0 here: k_r0):
// k_node_owner records the first position p of every node, then one thread
// per node descends to its level and finds its end, so the long chains of
// the top nodes' binary searches run side by side instead of in one thread.
__global__ void k_node_owner(int n, const int *__restrict__ noff, int *__restrict__ node_p) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  for (int i = noff[p]; i < noff[p + 1]; ++i) node_p[i] = p;
}

template <bool F32>
__global__ void k_node_emit_nodes(int n, const unsigned long long *__restrict__ keys, const int *__restrict__ noff,
                                  const uint8_t *__restrict__ lvl32, const int *__restrict__ node_p,
                                  const RootInfo *__restrict__ root, const void *__restrict__ pos_sorted,
                                  float4 *__restrict__ nlo, float4 *__restrict__ nhi, int *__restrict__ nsize) {
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= noff[n]) return;
  const int p = node_p[node];
  const int L = first_level(keys, p) + (node - noff[p]);
  const int Lc = lvl32[p];
  const unsigned long long kp = keys[p];
  const double pad2 = 2.0 * root->pad;
  double c[3] = {root->c[0], root->c[1], root->c[2]};
  double half = root->half;
  for (int l = 1; l <= L; ++l) {  // the reference centre arithmetic down to L
    const int o = (int)((kp >> (63 - 3 * l)) & 7ull);
    const double h2 = __dmul_rn(half, 0.5);
    c[0] = (o & 4) ? __dadd_rn(c[0], h2) : __dsub_rn(c[0], h2);
    c[1] = (o & 2) ? __dadd_rn(c[1], h2) : __dsub_rn(c[1], h2);
    c[2] = (o & 1) ? __dadd_rn(c[2], h2) : __dsub_rn(c[2], h2);
    half = h2;
  }
  const int end = (L == 0) ? n : upper_bound_key(keys, p + 1, n, kp | low_mask(L));
  const int skip = noff[end];
  float4 lo, hi;
  if (L < Lc) {
    const double e = half + pad2;
    lo = make_float4(f_rd(c[0] - e), f_rd(c[1] - e), f_rd(c[2] - e), __int_as_float(skip));
    hi = make_float4(f_ru(c[0] + e), f_ru(c[1] + e), f_ru(c[2] + e), __int_as_float(p));
  } else {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int q = p; q < end; ++q) {
      if (F32) {
        const float4 v = reinterpret_cast<const float4 *>(pos_sorted)[q];
        mn[0] = fminf(mn[0], v.x); mn[1] = fminf(mn[1], v.y); mn[2] = fminf(mn[2], v.z);
        mx[0] = fmaxf(mx[0], v.x); mx[1] = fmaxf(mx[1], v.y); mx[2] = fmaxf(mx[2], v.z);
      } else {
        const D4 v = reinterpret_cast<const D4 *>(pos_sorted)[q];
        mn[0] = fminf(mn[0], f_rd(v.x)); mn[1] = fminf(mn[1], f_rd(v.y)); mn[2] = fminf(mn[2], f_rd(v.z));
        mx[0] = fmaxf(mx[0], f_ru(v.x)); mx[1] = fmaxf(mx[1], f_ru(v.y)); mx[2] = fmaxf(mx[2], f_ru(v.z));
      }
    }
    lo = make_float4(mn[0], mn[1], mn[2], __int_as_float(skip));
    hi = make_float4(mx[0], mx[1], mx[2], __int_as_float(p));
  }
  nlo[node] = lo;
  nhi[node] = hi;
  nsize[node] = end - p;
}

template <typename T>
__global__ void k_fill(int n, T *a, T v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

inline int nblk(long long n, int t = kTB) { return (int)((n + t - 1) / t); }

// keys of the domain decomposition (distributed/decomp.py): the same 21-level
// descent as k_keys, from a root cube given by value (the all-reduced one)
template <typename PosT>
__global__ void k_keys_at(int n, const PosT *__restrict__ x, const PosT *__restrict__ y,
                          const PosT *__restrict__ z, double c0x, double c0y, double c0z, double half0,
                          unsigned long long *__restrict__ keys) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double px = (double)x[i], py = (double)y[i], pz = (double)z[i];
  double cx = c0x, cy = c0y, cz = c0z, half = half0;
  unsigned long long key = 0;
#pragma unroll
  for (int l = 0; l < kMaxLevel; ++l) {
    const int bx = px >= cx, by = py >= cy, bz = pz >= cz;
    key = (key << 3) | (unsigned long long)((bx << 2) | (by << 1) | bz);
    const double h2 = __dmul_rn(half, 0.5);
    cx = bx ? __dadd_rn(cx, h2) : __dsub_rn(cx, h2);
    cy = by ? __dadd_rn(cy, h2) : __dsub_rn(cy, h2);
    cz = bz ? __dadd_rn(cz, h2) : __dsub_rn(cz, h2);
    half = h2;
  }
  keys[i] = key;
}

}  // namespace

size_t deep_segs_bytes() { return sizeof(DeepSeg) * (size_t)kDeepStack * kDeepThreads; }

size_t cub_temp_needed(int n) {  // the sort's and the scan's workspace (no library kernels)
  const size_t a = radix_sort_temp_bytes(n), b = scan_temp_bytes(n + 1);
  return a > b ? a : b;
}

void launch_keys_at(cudaStream_t s, int n, int precision_in, const void *x, const void *y, const void *z,
                    const double *centre, double half, unsigned long long *keys) {
  if (n <= 0) return;
  if (precision_in == 1)
    k_keys_at<float><<<(n + 255) / 256, 256, 0, s>>>(n, (const float *)x, (const float *)y, (const float *)z,
                                                     centre[0], centre[1], centre[2], half, keys);
  else
    k_keys_at<double><<<(n + 255) / 256, 256, 0, s>>>(n, (const double *)x, (const double *)y, (const double *)z,
                                                      centre[0], centre[1], centre[2], half, keys);
}

void launch_bbox(cudaStream_t s, int n, int precision_in, const void *x, const void *y, const void *z,
                 unsigned long long *ord, RootInfo *root, int *launches) {
  unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  cudaMemcpyAsync(ord, init, sizeof(init), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(root, 0, sizeof(RootInfo), s);
  const int grid = n > 0 ? std::min(nblk(n), 148 * 8) : 1;
  if (precision_in == 1)
    k_bbox<float><<<grid, kTB, 0, s>>>(n, (const float *)x, (const float *)y, (const float *)z, ord, root);
  else
    k_bbox<double><<<grid, kTB, 0, s>>>(n, (const double *)x, (const double *)y, (const double *)z, ord, root);
  k_root<<<1, 32, 0, s>>>(n, ord, root);
  *launches += 2;
}

// Everything after the bbox: keys, sort, perm, sorted SoA, search tree.
// Requires tb.root to hold the root info (launch_bbox) and the caller to
// have validated it.  Returns 0 or SPH_UNSUPPORTED-style error via err_flag.
int tree_build(cudaStream_t s, TreeBuffers &tb, int n, int precision_in, int compute_f32,
               const void *x, const void *y, const void *z, const double *mass, int k, int *launches) {
  const bool in32 = precision_in == 1;
  if (in32)
    k_keys<float><<<nblk(n), kTB, 0, s>>>(n, (const float *)x, (const float *)y, (const float *)z, tb.root,
                                          tb.keys_in, tb.idx_in);
  else
    k_keys<double><<<nblk(n), kTB, 0, s>>>(n, (const double *)x, (const double *)y, (const double *)z, tb.root,
                                           tb.keys_in, tb.idx_in);
  size_t tbytes = tb.cub_temp_bytes;
  // stable LSD radix sort of (key, original index), hand-written onesweep (sph_sort.cu)
  radix_sort_pairs(s, n, tb.keys_in, tb.idx_in, tb.keys, tb.idx, tb.cub_temp);
  (void)tbytes;
  cudaMemsetAsync(tb.deep_count, 0, sizeof(int), s);
  cudaMemsetAsync(tb.err_flag, 0, sizeof(int), s);
  const int cap = tb.leaf_cap > 0 ? tb.leaf_cap : kLeafCap;
  k_levels<<<nblk(n), kTB, 0, s>>>(n, tb.keys, tb.lvl8, tb.lvl32, tb.deep_count, tb.deep_list, cap);
  cudaMemcpyAsync(tb.perm, tb.idx, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s);
  // idx_in (the sort's input) is free again: k_deep's partition scratch
  if (in32)
    k_deep<float><<<kDeepThreads / 128, 128, 0, s>>>(n, tb.keys, tb.idx, (const float *)x, (const float *)y,
                                                     (const float *)z, tb.root, tb.deep_count, tb.deep_list, tb.lvl8,
                                                     tb.perm, tb.idx_in, (DeepSeg *)tb.deep_segs, tb.err_flag, cap);
  else
    k_deep<double><<<kDeepThreads / 128, 128, 0, s>>>(n, tb.keys, tb.idx, (const double *)x, (const double *)y,
                                                      (const double *)z, tb.root, tb.deep_count, tb.deep_list,
                                                      tb.lvl8, tb.perm, tb.idx_in, (DeepSeg *)tb.deep_segs,
                                                      tb.err_flag, cap);
  k_leaf_order<<<nblk(n), kTB, 0, s>>>(n, tb.keys, tb.lvl8, tb.idx, tb.perm, cap);
  *launches += 5;  // keys, levels, deep, leaf order (+ the radix sort's own kernels)
  return 0;
}

int tree_build_search(cudaStream_t s, TreeBuffers &tb, int n, int precision_in, int compute_f32,
                      const void *x, const void *y, const void *z, const double *mass, int k, float rmax,
                      int *launches) {
  const bool in32 = precision_in == 1;
  if (tb.mass_ready) cudaStreamWaitEvent(s, tb.mass_ready, 0);  // masses copied on a side stream
  if (compute_f32) {
    if (in32)
      k_gather_f32<float><<<nblk(n), kTB, 0, s>>>(n, tb.perm, (const float *)x, (const float *)y,
                                                  (const float *)z, mass, (float4 *)tb.pos_sorted, tb.mass_sorted,
                                                  tb.posj);
    else
      k_gather_f32<double><<<nblk(n), kTB, 0, s>>>(n, tb.perm, (const double *)x, (const double *)y,
                                                   (const double *)z, mass, (float4 *)tb.pos_sorted, tb.mass_sorted,
                                                   tb.posj);
  } else {
    if (in32)
      k_gather_f64<float><<<nblk(n), kTB, 0, s>>>(n, tb.perm, (const float *)x, (const float *)y,
                                                  (const float *)z, mass, (D4 *)tb.pos_sorted);
    else
      k_gather_f64<double><<<nblk(n), kTB, 0, s>>>(n, tb.perm, (const double *)x, (const double *)y,
                                                   (const double *)z, mass, (D4 *)tb.pos_sorted);
  }
  k_node_count<<<nblk(n + 1), kTB, 0, s>>>(n, tb.keys, tb.lvl32, tb.noff);
  scan_exclusive_i32(s, tb.noff, tb.noff, n + 1, tb.cub_temp);  // node offsets (sph_scan.cu)
  if (!tb.emit_r0 && tb.node_p) {
    k_node_owner<<<nblk(n), kTB, 0, s>>>(n, tb.noff, tb.node_p);
    const int max_nodes = 2 * n + 64;
    if (compute_f32)
      k_node_emit_nodes<true><<<nblk(max_nodes), kTB, 0, s>>>(n, tb.keys, tb.noff, tb.lvl32, tb.node_p, tb.root,
                                                              tb.pos_sorted, tb.nlo, tb.nhi, tb.nsize);
    else
      k_node_emit_nodes<false><<<nblk(max_nodes), kTB, 0, s>>>(n, tb.keys, tb.noff, tb.lvl32, tb.node_p, tb.root,
                                                               tb.pos_sorted, tb.nlo, tb.nhi, tb.nsize);
    *launches += 4;
    return 0;
  }
  if (compute_f32)
    k_node_emit<true><<<nblk(n), kTB, 0, s>>>(n, tb.keys, tb.lvl32, tb.noff, tb.root, tb.pos_sorted, k, rmax, tb.r0_scale, tb.c0_scale, tb.emit_r0,
                                              tb.nlo, tb.nhi, tb.nsize, tb.r0);
  else
    k_node_emit<false><<<nblk(n), kTB, 0, s>>>(n, tb.keys, tb.lvl32, tb.noff, tb.root, tb.pos_sorted, k, rmax, tb.r0_scale, tb.c0_scale, tb.emit_r0,
                                               tb.nlo, tb.nhi, tb.nsize, tb.r0);
  *launches += 3;
  return 0;
}

}  // namespace sph
