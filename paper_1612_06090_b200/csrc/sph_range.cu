// Batched range query: for every particle i the list of OTHER particles j with
// (dx*dx + dy*dy) + dz*dz <= h_i*h_i in unfused fp64 -- the reference's
// range_query(tree, pos_i, h_i, exclude=i) (octree.py:179-227, 351-379) for
// all particles at once, as CSR (offsets from the counts of
// sph_neighbor_counts).  One warp per query walks the search tree's child
// records (box tests in fp32 with slack), every candidate of a hit cell gets
// the exact fp64 distance, accepted pairs are written with a ballot prefix;
// each query's list is then sorted by index (CUB segmented sort).
#include "sph_internal.cuh"
#include <cub/cub.cuh>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kRW = 4;        // warps per block
constexpr int kRStack = 256;  // node ids per warp

struct alignas(32) D4 { double x, y, z, m; };

template <bool F32>
__global__ void __launch_bounds__(kRW * 32) k_range_fill(int n, const uint32_t *__restrict__ perm,
                                                         const void *__restrict__ pos_sorted,
                                                         const double *__restrict__ h_sorted, TreeView tree,
                                                         const int64_t *__restrict__ offsets,
                                                         int64_t *__restrict__ idx_out, double *__restrict__ d2_out,
                                                         int *__restrict__ err) {
  __shared__ int s_stk[kRW][kRStack];
  const int lane = threadIdx.x & 31;
  int *stk = s_stk[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1u;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < n; p += nw) {
    double tx, ty, tz;
    if constexpr (F32) {
      const float4 t = reinterpret_cast<const float4 *>(pos_sorted)[p];
      tx = t.x; ty = t.y; tz = t.z;
    } else {
      const D4 t = reinterpret_cast<const D4 *>(pos_sorted)[p];
      tx = t.x; ty = t.y; tz = t.z;
    }
    const double h = h_sorted[p];
    const double r2 = __dmul_rn(h, h);
    const int q = (int)perm[p];
    const int64_t base = offsets[q], want = offsets[q + 1] - base;
    // fp32 box test: conservative (radius and coordinates widened by a few ulps)
    const float fx = (float)tx, fy = (float)ty, fz = (float)tz;
    const float sl = fmaxf(fmaxf(fabsf(fx), fabsf(fy)), fabsf(fz)) * 4.8e-7f;
    const float rf = (float)h * (1.0f + 1e-5f) + sl;
    const float rf2 = rf * rf;
    int64_t w = 0;
    if (lane == 0) stk[0] = tree.root_start;
    int top = 1;
    bool over = false;
    __syncwarp();
    while (top > 0) {
      const int np = min(top, 4);
      top -= np;
      const int par = (lane >> 3) < np ? stk[top + (lane >> 3)] : -1;
      __syncwarp();
      bool hit = false, is_cell = false;
      int code = 0, end = 0;
      if (par >= 0) {
        const float4 *rec = tree.crec + 16 * (size_t)par + 2 * (lane & 7);
        const float4 l4 = rec[0], h4 = rec[1];
        code = __float_as_int(l4.w);
        end = __float_as_int(h4.w);
        is_cell = code < 0;
        const float gx = fmaxf(fmaxf(l4.x - fx, fx - h4.x), 0.f);
        const float gy = fmaxf(fmaxf(l4.y - fy, fy - h4.y), 0.f);
        const float gz = fmaxf(fmaxf(l4.z - fz, fz - h4.z), 0.f);
        hit = gx * gx + gy * gy + gz * gz <= rf2;
      }
      const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
      if (top + __popc(pm) > kRStack) { over = true; break; }
      if (hit && !is_cell) stk[top + __popc(pm & lt)] = code;
      top += __popc(pm);
      // the hit cells one after the other, 32 candidates at a time
      unsigned cm = __ballot_sync(FULL, hit && is_cell);
      while (cm) {
        const int src = __ffs(cm) - 1;
        cm &= cm - 1u;
        const int s0 = ~__shfl_sync(FULL, code, src), e0 = __shfl_sync(FULL, end, src);
        for (int j0 = s0; j0 < e0; j0 += 32) {
          const int j = j0 + lane;
          bool acc = false;
          double d2 = 0.0;
          if (j < e0 && j != p) {
            double cx, cy, cz;
            if constexpr (F32) {
              const float4 c = reinterpret_cast<const float4 *>(pos_sorted)[j];
              cx = c.x; cy = c.y; cz = c.z;
            } else {
              const D4 c = reinterpret_cast<const D4 *>(pos_sorted)[j];
              cx = c.x; cy = c.y; cz = c.z;
            }
            d2 = exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
            acc = d2 <= r2;
          }
          const unsigned am = __ballot_sync(FULL, acc);
          if (acc) {
            const int64_t slot = w + __popc(am & lt);
            if (slot < want) {
              idx_out[base + slot] = (int64_t)perm[j];
              d2_out[base + slot] = d2;
            }
          }
          w += __popc(am);
        }
      }
      __syncwarp();
    }
    if (lane == 0 && (over || w != want)) atomicAdd(err, 1);
  }
}

// Queries around arbitrary centres (the reference's range_query(tree, center,
// radius, exclude), octree.py:351-379): COUNT writes the list length of each
// query, otherwise the lists are written at offsets[q] (unsorted).  A
// candidate j is accepted when (dx*dx + dy*dy) + dz*dz <= r*r in unfused
// fp64 with dx = x_j - c_x (octree.py:211-214) and its original index is not
// exclude[q].
template <bool F32, bool COUNT>
__global__ void __launch_bounds__(kRW * 32) k_range_points(int64_t m, const double *__restrict__ centers,
                                                           const double *__restrict__ radii,
                                                           const int64_t *__restrict__ excl,
                                                           const uint32_t *__restrict__ perm,
                                                           const void *__restrict__ pos_sorted, TreeView tree,
                                                           const int64_t *__restrict__ offsets,
                                                           int64_t *__restrict__ counts, int64_t *__restrict__ idx_out,
                                                           double *__restrict__ d2_out, int *__restrict__ err) {
  __shared__ int s_stk[kRW][kRStack];
  const int lane = threadIdx.x & 31;
  int *stk = s_stk[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1u;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t q = gw; q < m; q += nw) {
    const double tx = centers[3 * q], ty = centers[3 * q + 1], tz = centers[3 * q + 2];
    const double r = radii[q];
    const double r2 = __dmul_rn(r, r);
    const int64_t ex = excl ? excl[q] : -1;
    const int64_t base = COUNT ? 0 : offsets[q], want = COUNT ? 0 : offsets[q + 1] - base;
    // fp32 box test: conservative (radius and coordinates widened by a few ulps)
    const float fx = (float)tx, fy = (float)ty, fz = (float)tz;
    const float sl = fmaxf(fmaxf(fabsf(fx), fabsf(fy)), fabsf(fz)) * 4.8e-7f;
    const float rf = (float)r * (1.0f + 1e-5f) + sl;
    const float rf2 = rf * rf;
    int64_t w = 0;
    if (lane == 0) stk[0] = tree.root_start;
    int top = 1;
    bool over = false;
    __syncwarp();
    while (top > 0) {
      const int np = min(top, 4);
      top -= np;
      const int par = (lane >> 3) < np ? stk[top + (lane >> 3)] : -1;
      __syncwarp();
      bool hit = false, is_cell = false;
      int code = 0, end = 0;
      if (par >= 0) {
        const float4 *rec = tree.crec + 16 * (size_t)par + 2 * (lane & 7);
        const float4 l4 = rec[0], h4 = rec[1];
        code = __float_as_int(l4.w);
        end = __float_as_int(h4.w);
        is_cell = code < 0;
        const float gx = fmaxf(fmaxf(l4.x - fx, fx - h4.x), 0.f);
        const float gy = fmaxf(fmaxf(l4.y - fy, fy - h4.y), 0.f);
        const float gz = fmaxf(fmaxf(l4.z - fz, fz - h4.z), 0.f);
        hit = gx * gx + gy * gy + gz * gz <= rf2;
      }
      const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
      if (top + __popc(pm) > kRStack) { over = true; break; }
      if (hit && !is_cell) stk[top + __popc(pm & lt)] = code;
      top += __popc(pm);
      unsigned cm = __ballot_sync(FULL, hit && is_cell);
      while (cm) {
        const int src = __ffs(cm) - 1;
        cm &= cm - 1u;
        const int s0 = ~__shfl_sync(FULL, code, src), e0 = __shfl_sync(FULL, end, src);
        for (int j0 = s0; j0 < e0; j0 += 32) {
          const int j = j0 + lane;
          bool acc = false;
          double d2 = 0.0;
          int64_t o = -1;
          if (j < e0) {
            double cx, cy, cz;
            if constexpr (F32) {
              const float4 c = reinterpret_cast<const float4 *>(pos_sorted)[j];
              cx = c.x; cy = c.y; cz = c.z;
            } else {
              const D4 c = reinterpret_cast<const D4 *>(pos_sorted)[j];
              cx = c.x; cy = c.y; cz = c.z;
            }
            o = (int64_t)perm[j];
            d2 = exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
            acc = d2 <= r2 && o != ex;
          }
          const unsigned am = __ballot_sync(FULL, acc);
          if (!COUNT && acc) {
            const int64_t slot = w + __popc(am & lt);
            if (slot < want) {
              idx_out[base + slot] = o;
              d2_out[base + slot] = d2;
            }
          }
          w += __popc(am);
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (COUNT) counts[q] = w;
      if (over || (!COUNT && w != want)) atomicAdd(err, 1);
    }
  }
}

}  // namespace

int range_points(cudaStream_t s, int f32, int count_only, int64_t m, const double *centers, const double *radii,
                 const int64_t *excl, const uint32_t *perm, const void *pos_sorted, const TreeView &tree,
                 const int64_t *offsets, int64_t *counts, int64_t *idx_tmp, double *d2_tmp, int *err, int num_sms) {
  const int grid = num_sms * 8;
  if (count_only) {
    if (f32) k_range_points<true, true><<<grid, kRW * 32, 0, s>>>(m, centers, radii, excl, perm, pos_sorted, tree,
                                                                   offsets, counts, idx_tmp, d2_tmp, err);
    else k_range_points<false, true><<<grid, kRW * 32, 0, s>>>(m, centers, radii, excl, perm, pos_sorted, tree,
                                                                offsets, counts, idx_tmp, d2_tmp, err);
  } else {
    if (f32) k_range_points<true, false><<<grid, kRW * 32, 0, s>>>(m, centers, radii, excl, perm, pos_sorted, tree,
                                                                    offsets, counts, idx_tmp, d2_tmp, err);
    else k_range_points<false, false><<<grid, kRW * 32, 0, s>>>(m, centers, radii, excl, perm, pos_sorted, tree,
                                                                 offsets, counts, idx_tmp, d2_tmp, err);
  }
  return 0;
}

int segmented_sort_pairs(cudaStream_t s, int64_t m, int64_t total, const int64_t *offsets, const int64_t *idx_in,
                         int64_t *idx_out, const double *d2_in, double *d2_out, void *temp, size_t temp_bytes) {
  size_t need = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, need, idx_in, idx_out, d2_in, d2_out, total, m, offsets, offsets + 1,
                                      s);
  if (need > temp_bytes) return -1;
  cub::DeviceSegmentedSort::SortPairs(temp, temp_bytes, idx_in, idx_out, d2_in, d2_out, total, m, offsets,
                                      offsets + 1, s);
  return 0;
}

int range_fill(cudaStream_t s, int f32, int n, const uint32_t *perm, const void *pos_sorted, const double *h_sorted,
               const TreeView &tree, const int64_t *offsets, int64_t total, int64_t *idx_out, double *d2_out,
               int *err, void *temp, size_t temp_bytes, int64_t *idx_tmp, double *d2_tmp, int num_sms) {
  const int grid = num_sms * 8;
  if (f32)
    k_range_fill<true><<<grid, kRW * 32, 0, s>>>(n, perm, pos_sorted, h_sorted, tree, offsets, idx_tmp, d2_tmp, err);
  else
    k_range_fill<false><<<grid, kRW * 32, 0, s>>>(n, perm, pos_sorted, h_sorted, tree, offsets, idx_tmp, d2_tmp, err);
  // each query's list sorted by index
  size_t need = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, need, idx_tmp, idx_out, d2_tmp, d2_out, total, n, offsets,
                                      offsets + 1, s);
  if (need > temp_bytes) return -1;
  cub::DeviceSegmentedSort::SortPairs(temp, temp_bytes, idx_tmp, idx_out, d2_tmp, d2_out, total, n, offsets,
                                      offsets + 1, s);
  return 0;
}

size_t range_sort_temp(int n, int64_t total) {
  size_t need = 0;
  cub::DeviceSegmentedSort::SortPairs(nullptr, need, (const int64_t *)nullptr, (int64_t *)nullptr,
                                      (const double *)nullptr, (double *)nullptr, total, n, (const int64_t *)nullptr,
                                      (const int64_t *)nullptr);
  return need;
}

}  // namespace sph
