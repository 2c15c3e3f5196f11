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
// particle order[i]; the key travels as two exact 32-bit halves and the
// global id as its int64 bit pattern (exact for any id)
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
  o[1] = make_double4(h0[j], __longlong_as_double((long long)gid[j]), (double)(key >> 32), (double)(key & 0xFFFFFFFFll));
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
// bin holding the K-th is an upper bound.  fp32 arithmetic, made safe by a
// relative 1e-5 and an absolute slack (fp32 rounding of the coordinates)
constexpr int kWinTile = 128;
constexpr int kWinBins = 64;
__global__ void __launch_bounds__(kWinTile) k_window_bounds(int64_t n, int k, int w, int width,
                                                            const double *__restrict__ rows, float abs_slack,
                                                            double *__restrict__ bound) {
  extern __shared__ float4 sp4[];  // kWinTile + 4w positions, then the bins [bin][thread]
  const int64_t b0 = (int64_t)blockIdx.x * kWinTile;
  const int span = kWinTile + 4 * w;
  const int64_t base = b0 - 2 * w;
  for (int t = threadIdx.x; t < span; t += blockDim.x) {
    const int64_t j = base + t;
    if (j >= 0 && j < n) sp4[t] = make_float4((float)rows[j * width], (float)rows[j * width + 1],
                                              (float)rows[j * width + 2], 0.f);
  }
  unsigned short *bins = reinterpret_cast<unsigned short *>(sp4 + span) + threadIdx.x;
  __syncthreads();
  const int64_t p = b0 + threadIdx.x;
  if (p >= n) return;
  if (n <= k) {
    bound[p] = INFINITY;
    return;
  }
  int64_t s = p - w;
  if (s > n - 1 - 2 * w) s = n - 1 - 2 * w;
  if (s < 0) s = 0;
  int64_t e = s + 2 * w;
  if (e > n - 1) e = n - 1;
  const int ls = (int)(s - base), le = (int)(e - base), lp = (int)(p - base);
  const float4 q = sp4[lp];
  // one pass: bins over [0, b0^2] with b0 the bound already known (the key
  // cube's); candidates beyond it cannot improve the bound and are dropped
  const double b_in = bound[p];
  const float d2top = (float)fmin(b_in * b_in, 3.0e38);
  if (!(d2top > 0.f)) return;
  for (int b = 0; b < kWinBins; ++b) bins[b * kWinTile] = 0;
  const float scale = (float)kWinBins / d2top;
  for (int j = ls; j <= le; ++j) {
    const float4 c = sp4[j];
    const float dx = c.x - q.x, dy = c.y - q.y, dz = c.z - q.z;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const int bq = (int)(d2 * scale);
    if (j != lp && bq < kWinBins) ++bins[bq * kWinTile];
  }
  int cum = 0, bq = kWinBins;
  for (int b = 0; b < kWinBins; ++b) {
    cum += bins[b * kWinTile];
    if (cum >= k) { bq = b; break; }
  }
  if (bq >= kWinBins - 1) return;  // the K-th of the window is not below the known bound
  // upper edge of the bin (a bin index may be one too low from rounding: +1 bin)
  const double e2 = (double)(bq + 2) / (double)kWinBins * (double)d2top;
  bound[p] = fmin(b_in, sqrt(e2) * (1.0 + 1e-5) + (double)abs_slack);
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
// my group: the lanes scan top boxes of 1024 consecutive foreign groups, then
// the 32-group super boxes of the hit ones (box vs box), then their members, and for each hit member the warp
// tests the group's particles (point vs box) and ORs the rank bit.
__device__ __forceinline__ bool desc_hit(const double *gb, const double *__restrict__ d, int periodic, double box) {
  double fb[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) fb[i] = d[i];
  const double m = d[6] * (1.0 + 1e-9);
  return box_gap2(gb, fb, periodic, box) <= m * m;
}

__global__ void k_ghost_mask(int64_t ng, const double *__restrict__ gdesc, const int64_t *__restrict__ gstart,
                             const int64_t *__restrict__ gcount, int width, const double *__restrict__ rows,
                             int64_t nf, const double *__restrict__ fdesc, const int32_t *__restrict__ frank,
                             int64_t nsup, const double *__restrict__ sdesc, int64_t ntop,
                             const double *__restrict__ tdesc, int periodic, double box,
                             uint32_t *__restrict__ mask) {
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= ng) return;
  double gb[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) gb[i] = gdesc[7 * g + i];
  const int64_t s = gstart[g], c = gcount[g];
  // two levels of super boxes over the foreign descriptors (key order, so they are spatially tight): 1024
  // descriptors per top box, 32 per super box
  for (int64_t t0 = 0; t0 < ntop; t0 += 32) {
    const int64_t tv = t0 + lane;
    unsigned th = __ballot_sync(0xffffffffu, tv < ntop && desc_hit(gb, tdesc + 7 * tv, periodic, box));
    while (th) {
      const int64_t T = t0 + __ffs(th) - 1;
      th &= th - 1u;
      const int64_t sv = T * 32 + lane;
      unsigned sh = __ballot_sync(0xffffffffu, sv < nsup && desc_hit(gb, sdesc + 7 * sv, periodic, box));
      while (sh) {
        const int64_t S = T * 32 + __ffs(sh) - 1;
        sh &= sh - 1u;
        const int64_t f = S * 32 + lane;
        unsigned fm = __ballot_sync(0xffffffffu, f < nf && desc_hit(gb, fdesc + 7 * f, periodic, box));
        while (fm) {
          const int64_t fh = S * 32 + __ffs(fm) - 1;
          fm &= fm - 1u;
          double hb[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) hb[i] = fdesc[7 * fh + i];
          const double m = fdesc[7 * fh + 6] * (1.0 + 1e-9);
          const uint32_t bit = 1u << frank[fh];
          for (int64_t i = lane; i < c; i += 32) {
            const double *r = rows + (s + i) * width;
            const double pb[6] = {r[0], r[1], r[2], r[0], r[1], r[2]};
            if (box_gap2(pb, hb, periodic, box) <= m * m) atomicOr(mask + s + i, bit);
          }
        }
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

void launch_window_bounds(cudaStream_t s, int64_t n, int k, int width, const double *rows, double abs_slack,
                          double *bound) {
  if (n <= 0) return;
  const int w = (3 * k + 1) / 2;
  const size_t smem = (size_t)(kWinTile + 4 * w) * sizeof(float4) + kWinTile * kWinBins * sizeof(unsigned short);
  cudaFuncSetAttribute(k_window_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_window_bounds<<<(unsigned)((n + kWinTile - 1) / kWinTile), kWinTile, smem, s>>>(n, k, w, width, rows,
                                                                                    (float)abs_slack, bound);
}

// super boxes of 32 consecutive descriptors (box union, largest margin)
__global__ void k_super_desc(int64_t nf, const double *__restrict__ fdesc, int64_t nsup, double *__restrict__ sdesc) {
  const int64_t S = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (S >= nsup) return;
  double o[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, 0.0};
  for (int64_t f = S * 32; f < nf && f < S * 32 + 32; ++f) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      o[i] = fmin(o[i], fdesc[7 * f + i]);
      o[3 + i] = fmax(o[3 + i], fdesc[7 * f + 3 + i]);
    }
    o[6] = fmax(o[6], fdesc[7 * f + 6]);
  }
#pragma unroll
  for (int i = 0; i < 7; ++i) sdesc[7 * S + i] = o[i];
}

void launch_ghost_mask(cudaStream_t s, int64_t ng, const double *gdesc, const int64_t *gstart, const int64_t *gcount,
                       int width, const double *rows, int64_t nf, const double *fdesc, const int32_t *frank,
                       int periodic, double box, uint32_t *mask, double *scratch) {
  if (ng <= 0 || nf <= 0) return;
  const int64_t nsup = (nf + 31) / 32, ntop = (nsup + 31) / 32;
  double *top = scratch + 7 * nsup;  // scratch holds 7 * (nsup + ntop) doubles
  k_super_desc<<<nb(nsup), kDT, 0, s>>>(nf, fdesc, nsup, scratch);
  k_super_desc<<<nb(ntop), kDT, 0, s>>>(nsup, scratch, ntop, top);
  k_ghost_mask<<<nb(ng * 32), kDT, 0, s>>>(ng, gdesc, gstart, gcount, width, rows, nf, fdesc, frank, nsup, scratch, ntop,
                                           top, periodic, box, mask);
}

void launch_group_boxes(cudaStream_t s, int64_t ng, const int64_t *starts, const int64_t *counts, int width,
                        const double *rows, const double *bound, double *out) {
  if (ng > 0) k_group_boxes<<<nb(ng * 32), kDT, 0, s>>>(ng, starts, counts, width, rows, bound, out);
}

}  // namespace sph
