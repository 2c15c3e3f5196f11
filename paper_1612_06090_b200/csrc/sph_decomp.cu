// Device helpers of the domain decomposition (paper_1612_06090_b200/distributed.py):
// record packing / row gathers around the NCCL all-to-alls, the search-free
// bound on h that sizes the ghost layer, and the per-group boxes the ranks
// exchange.  All HBM-bound; no reference counterpart (the reference runs in
// one shared-memory process).
#include "sph_internal.cuh"

namespace sph {
namespace {

constexpr int kDT = 256;

// row i of the record buffer = (x, y, z, m, h0, gid, key_hi, key_lo) of
// particle order[i]; the key travels as two exact 32-bit halves
template <typename PosT>
__global__ void k_pack_rows(int64_t n, const int64_t *__restrict__ order, const PosT *__restrict__ x,
                            const PosT *__restrict__ y, const PosT *__restrict__ z, const double *__restrict__ m,
                            const double *__restrict__ h0, const int64_t *__restrict__ gid,
                            const int64_t *__restrict__ keys, double *__restrict__ rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = order[i];
  const long long key = keys[j];
  double4 *o = reinterpret_cast<double4 *>(rows + 8 * i);
  o[0] = make_double4((double)x[j], (double)y[j], (double)z[j], m[j]);
  o[1] = make_double4(h0[j], (double)gid[j], (double)(key >> 32), (double)(key & 0xFFFFFFFFll));
}

// dst row i = src row idx[i] (width doubles per row)
__global__ void k_gather_rows(int64_t n, int width, const int64_t *__restrict__ idx, const double *__restrict__ src,
                              double *__restrict__ dst) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * width) return;
  const int64_t r = t / width;
  const int c = (int)(t - r * width);
  dst[t] = src[idx[r] * width + c];
}

// keys of received records (columns 6, 7) back to int64
__global__ void k_row_keys(int64_t n, const double *__restrict__ rows, int64_t *__restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((long long)rows[8 * i + 6] << 32) | (long long)rows[8 * i + 7];
}

// h <= sqrt(3) * side of the deepest key cube holding the particle and >= K
// others: the deepest common level of any window of K+1 consecutive sorted
// keys containing it (keys: 63-bit x-major octant paths, csrc/sph_tree.cu)
__global__ void k_level_bounds(int64_t n, int k, const int64_t *__restrict__ keys, double side0,
                               double *__restrict__ bound) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  if (n <= k) {
    bound[p] = INFINITY;
    return;
  }
  const int64_t s0 = p - k > 0 ? p - k : 0;
  const int64_t s1 = p < n - 1 - k ? p : n - 1 - k;
  int best = 0;
  for (int64_t s = s0; s <= s1; ++s) {
    const unsigned long long xo = (unsigned long long)keys[s] ^ (unsigned long long)keys[s + k];
    const int cpl = xo ? __clzll((long long)xo) - 1 : 63;
    best = max(best, min(cpl / 3, kMaxLevel));
  }
  bound[p] = side0 * ldexp(1.0, -best) * (1.7320508075688772 * (1.0 + 1e-9));
}

// a tighter bound from the particles themselves: the K-th smallest distance
// to ANY set of others bounds the K-th neighbour distance from above, so take
// the 2W key-consecutive records around p (W = 3K/2) and bin their squared
// distances (32 linear bins of d2 / d2max per thread): the upper edge of the
// bin holding the K-th is an upper bound.  Unfused fp64 (same as the torch
// restatement, bit for bit)
constexpr int kWinTile = 128;
constexpr int kWinBins = 32;
__global__ void __launch_bounds__(kWinTile) k_window_bounds(int64_t n, int k, int w, int width,
                                                            const double *__restrict__ rows,
                                                            double *__restrict__ bound) {
  extern __shared__ double sp[];  // (kWinTile + 2w) x 3 positions, then the bins
  const int64_t b0 = (int64_t)blockIdx.x * kWinTile;
  const int64_t lo = b0 - w > 0 ? b0 - w : 0;
  const int span = kWinTile + 4 * w;
  for (int t = threadIdx.x; t < span; t += blockDim.x) {
    const int64_t j = b0 - 2 * w + t;
    if (j >= 0 && j < n) {
      sp[3 * t] = rows[j * width];
      sp[3 * t + 1] = rows[j * width + 1];
      sp[3 * t + 2] = rows[j * width + 2];
    }
  }
  (void)lo;
  unsigned short *bins = reinterpret_cast<unsigned short *>(sp + 3 * span) + threadIdx.x * kWinBins;
  __syncthreads();
  const int64_t p = b0 + threadIdx.x;
  if (p >= n) return;
  if (n <= k) {
    bound[p] = INFINITY;
    return;
  }
  const int64_t base = b0 - 2 * w;
  int64_t s = p - w;
  if (s > n - 1 - 2 * w) s = n - 1 - 2 * w;
  if (s < 0) s = 0;
  int64_t e = s + 2 * w;
  if (e > n - 1) e = n - 1;
  const int lp = (int)(p - base);
  const double px = sp[3 * lp], py = sp[3 * lp + 1], pz = sp[3 * lp + 2];
  auto d2of = [&](int64_t j) {
    const int lj = (int)(j - base);
    const double dx = __dsub_rn(sp[3 * lj], px), dy = __dsub_rn(sp[3 * lj + 1], py), dz = __dsub_rn(sp[3 * lj + 2], pz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  };
  double d2max = 0.0;
  for (int64_t j = s; j <= e; ++j)
    if (j != p) d2max = fmax(d2max, d2of(j));
  if (!(d2max > 0.0)) return;  // coincident window: keep the cube bound
  for (int q = 0; q < kWinBins; ++q) bins[q] = 0;
  for (int64_t j = s; j <= e; ++j) {
    if (j == p) continue;
    const int bq = min((int)__dmul_rn(__ddiv_rn(d2of(j), d2max), (double)kWinBins), kWinBins - 1);
    ++bins[bq];
  }
  int cum = 0, bq = kWinBins - 1;
  for (int q = 0; q < kWinBins; ++q) {
    cum += bins[q];
    if (cum >= k) { bq = q; break; }
  }
  if (cum < k) return;  // fewer than K others in the window
  const double e2 = __dmul_rn((double)(bq + 1) / (double)kWinBins, d2max);
  bound[p] = fmin(bound[p], sqrt(e2) * (1.0 + 1e-9));
}

// per group of consecutive records: tight box of the positions and the
// largest bound -> (lo xyz, hi xyz, margin); one warp per group
__global__ void k_group_boxes(int64_t ng, const int64_t *__restrict__ starts, const int64_t *__restrict__ counts,
                              int width, const double *__restrict__ rows, const double *__restrict__ bound,
                              double *__restrict__ out) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ng) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY}, mb = 0.0;
  const int64_t s = starts[g], c = counts[g];
  for (int64_t i = lane; i < c; i += 32) {
    const double *r = rows + (s + i) * width;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], r[a]);
      hi[a] = fmax(hi[a], r[a]);
    }
    mb = fmax(mb, bound[s + i]);
  }
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fmin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, o));
  }
  if (lane == 0) {
    double *o = out + 7 * g;
    o[0] = lo[0]; o[1] = lo[1]; o[2] = lo[2];
    o[3] = hi[0]; o[4] = hi[1]; o[5] = hi[2];
    o[6] = mb;
  }
}

// squared gap between boxes, min-image per axis when periodic (plain fp64;
// the margins it is compared with carry a relative 1e-9)
__device__ __forceinline__ double box_gap2(const double *a, const double *b, int periodic, double box) {
  double s = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    double d = fmax(fmax(b[ax] - a[3 + ax], a[ax] - b[3 + ax]), 0.0);
    if (periodic) {
      const double dm = fmax(fmax((b[ax] - box) - a[3 + ax], a[ax] - (b[3 + ax] - box)), 0.0);
      const double dp = fmax(fmax((b[ax] + box) - a[3 + ax], a[ax] - (b[3 + ax] + box)), 0.0);
      d = fmin(d, fmin(dm, dp));
    }
    s += d * d;
  }
  return s;
}

// ghost marking: a particle of my group g is sent to rank q when it lies
// within the margin of some group f of q (margin = the largest bound on h of
// f's particles, so every neighbour of f's targets is covered).  One warp per
// my group: the lanes scan the foreign groups (box vs box), and for each hit
// the warp tests the group's particles (point vs box) and ORs rank bits.
__global__ void k_ghost_mask(int64_t ng, const double *__restrict__ gdesc, const int64_t *__restrict__ gstart,
                             const int64_t *__restrict__ gcount, int width, const double *__restrict__ rows,
                             int64_t nf, const double *__restrict__ fdesc, const int32_t *__restrict__ frank,
                             int periodic, double box, uint32_t *__restrict__ mask) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ng) return;
  double gb[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) gb[i] = gdesc[7 * g + i];
  const int64_t s = gstart[g], c = gcount[g];
  for (int64_t f0 = 0; f0 < nf; f0 += 32) {
    const int64_t f = f0 + lane;
    bool hit = false;
    double fb[7];
    if (f < nf) {
#pragma unroll
      for (int i = 0; i < 7; ++i) fb[i] = fdesc[7 * f + i];
      const double m = fb[6] * (1.0 + 1e-9);
      hit = box_gap2(gb, fb, periodic, box) <= m * m;
    }
    unsigned hm = __ballot_sync(0xffffffffu, hit);
    while (hm) {
      const int src = __ffs(hm) - 1;
      hm &= hm - 1u;
      double hb[7];
#pragma unroll
      for (int i = 0; i < 7; ++i) hb[i] = __shfl_sync(0xffffffffu, fb[i], src);
      const uint32_t bit = 1u << __shfl_sync(0xffffffffu, f < nf ? frank[f] : 0, src);
      const double m = hb[6] * (1.0 + 1e-9);
      for (int64_t i = lane; i < c; i += 32) {
        const double *r = rows + (s + i) * width;
        const double pb[6] = {r[0], r[1], r[2], r[0], r[1], r[2]};
        if (box_gap2(pb, hb, periodic, box) <= m * m) atomicOr(mask + s + i, bit);
      }
    }
  }
}

inline unsigned nb(int64_t n) { return (unsigned)((n + kDT - 1) / kDT); }

}  // namespace

void launch_pack_rows(cudaStream_t s, int64_t n, int precision_in, const int64_t *order, const void *x,
                      const void *y, const void *z, const double *m, const double *h0, const int64_t *gid,
                      const int64_t *keys, double *rows) {
  if (n <= 0) return;
  if (precision_in == 1)
    k_pack_rows<float><<<nb(n), kDT, 0, s>>>(n, order, (const float *)x, (const float *)y, (const float *)z, m, h0,
                                             gid, keys, rows);
  else
    k_pack_rows<double><<<nb(n), kDT, 0, s>>>(n, order, (const double *)x, (const double *)y, (const double *)z, m,
                                              h0, gid, keys, rows);
}

void launch_gather_rows(cudaStream_t s, int64_t n, int width, const int64_t *idx, const double *src, double *dst) {
  if (n > 0) k_gather_rows<<<nb(n * width), kDT, 0, s>>>(n, width, idx, src, dst);
}

void launch_row_keys(cudaStream_t s, int64_t n, const double *rows, int64_t *keys) {
  if (n > 0) k_row_keys<<<nb(n), kDT, 0, s>>>(n, rows, keys);
}

void launch_level_bounds(cudaStream_t s, int64_t n, int k, const int64_t *keys, double side0, double *bound) {
  if (n > 0) k_level_bounds<<<nb(n), kDT, 0, s>>>(n, k, keys, side0, bound);
}

void launch_window_bounds(cudaStream_t s, int64_t n, int k, int width, const double *rows, double *bound) {
  if (n <= 0) return;
  const int w = (3 * k + 1) / 2;
  const size_t smem = (size_t)(kWinTile + 4 * w) * 3 * sizeof(double) + kWinTile * kWinBins * sizeof(unsigned short);
  cudaFuncSetAttribute(k_window_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_window_bounds<<<(unsigned)((n + kWinTile - 1) / kWinTile), kWinTile, smem, s>>>(n, k, w, width, rows, bound);
}

void launch_ghost_mask(cudaStream_t s, int64_t ng, const double *gdesc, const int64_t *gstart, const int64_t *gcount,
                       int width, const double *rows, int64_t nf, const double *fdesc, const int32_t *frank,
                       int periodic, double box, uint32_t *mask) {
  if (ng > 0 && nf > 0)
    k_ghost_mask<<<nb(ng * 32), kDT, 0, s>>>(ng, gdesc, gstart, gcount, width, rows, nf, fdesc, frank, periodic, box,
                                             mask);
}

void launch_group_boxes(cudaStream_t s, int64_t ng, const int64_t *starts, const int64_t *counts, int width,
                        const double *rows, const double *bound, double *out) {
  if (ng > 0) k_group_boxes<<<nb(ng * 32), kDT, 0, s>>>(ng, starts, counts, width, rows, bound, out);
}

}  // namespace sph
