// sph_sort.cu -- stable LSD radix sort of the 63-bit octree keys with their
// original indices (the ordering step of octree.py:92-121: the reference's
// recursive stable 8-way partition equals a stable sort by the x-major octant
// path).  Hand-written "onesweep" form:
//
//   k_digit_hist   one read of the keys: the histograms of all 7 digits
//                  (9 bits each, 63 bits) at once, per-block shared atomics;
//   k_digit_scan   exclusive scan of each digit's histogram (global offsets);
//   k_onesweep     per digit, ONE kernel: each 4096-key tile ranks its keys
//                  stably (per-warp counters + match_any over a warp's
//                  contiguous segment), publishes its digit counts, obtains
//                  its exclusive prefix over earlier tiles by decoupled
//                  look-back (tiles take ids in launch order from an atomic
//                  counter, so every tile waits only on running/finished
//                  ones), reorders the tile in shared memory and writes each
//                  digit's run contiguously (coalesced).
//
// Per digit pass the keys and values are read once and written once (24 B
// per key); 7 passes ping-pong A->B->A->...->B, so the sorted keys land in
// the second buffer.
#include "sph_internal.cuh"

#include <algorithm>

namespace sph {
namespace {

constexpr int kDigitBits = 9;
constexpr int kBins = 1 << kDigitBits;  // 512
constexpr int kPasses = 7;              // 7 x 9 = 63 key bits
constexpr int kSortThreads = 512;       // one thread per digit value
constexpr int kIPT = 8;                 // keys per thread
constexpr int kTile = kSortThreads * kIPT;
constexpr int kSortWarps = kSortThreads / 32;
constexpr unsigned kFlagA = 1u << 30;   // tile aggregate published
constexpr unsigned kFlagP = 2u << 30;   // inclusive prefix published
constexpr unsigned kValMask = (1u << 30) - 1u;

// tile status words shared across the grid: relaxed, GPU-scope (every value
// is self-contained, no other data is published through them)
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned *p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_digit_hist(int n, const unsigned long long *__restrict__ keys,
                                                    unsigned *__restrict__ ghist) {
  __shared__ unsigned h[kPasses][kBins];
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) (&h[0][0])[i] = 0u;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
#pragma unroll
    for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p][(unsigned)(k >> (kDigitBits * p)) & (kBins - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) {
    const unsigned v = (&h[0][0])[i];
    if (v) atomicAdd(ghist + i, v);
  }
}

// exclusive scan of each pass's histogram (one block, one thread per bin)
__global__ void __launch_bounds__(kBins) k_digit_scan(const unsigned *__restrict__ ghist, unsigned *__restrict__ goff) {
  __shared__ unsigned wsum[kBins / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int p = 0; p < kPasses; ++p) {
    const unsigned v = ghist[p * kBins + t];
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    unsigned before = 0;
    for (int i = 0; i < w; ++i) before += wsum[i];
    goff[p * kBins + t] = before + incl - v;
    __syncthreads();
  }
}

struct SortSmem {
  unsigned long long keys[kTile];
  uint32_t vals[kTile];
  unsigned short whist[kSortWarps][kBins + 1];  // per-warp counters, then per-warp exclusive offsets (<= 4096: 16 bits keep three tiles per SM)
  unsigned dstart[kBins];                 // tile-local start of each digit's run
  unsigned gbase[kBins];                  // global position of each digit's run of this tile
  unsigned wsum[kSortWarps];
  int tile;
};

__global__ void __launch_bounds__(kSortThreads) k_onesweep(int n, int shift, const unsigned long long *__restrict__ kin,
                                                           const uint32_t *__restrict__ vin,
                                                           unsigned long long *__restrict__ kout,
                                                           uint32_t *__restrict__ vout,
                                                           const unsigned *__restrict__ goff,
                                                           unsigned *__restrict__ status, int *__restrict__ counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem &S = *reinterpret_cast<SortSmem *>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const unsigned lt = (1u << lane) - 1u;
  if (t == 0) S.tile = atomicAdd(counter, 1);
  for (int i = t; i < kSortWarps * (kBins + 1); i += kSortThreads) (&S.whist[0][0])[i] = 0;
  __syncthreads();
  const int tile = S.tile;
  const int64_t base = (int64_t)tile * kTile;
  // each warp ranks a contiguous segment of the tile, 32 keys per round, in
  // index order: rank = keys of the same digit earlier in the segment
  unsigned long long key[kIPT];
  uint32_t val[kIPT];
  unsigned rank[kIPT];
  int dig[kIPT];
  const int64_t seg = base + (int64_t)w * 32 * kIPT;
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int64_t i = seg + j * 32 + lane;
    const bool ok = i < n;
    key[j] = ok ? kin[i] : 0ull;
    val[j] = ok ? vin[i] : 0u;
    dig[j] = ok ? (int)((unsigned)(key[j] >> shift) & (kBins - 1)) : kBins;  // past the end: its own bin
  }
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int d = dig[j];
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned old = S.whist[w][d];
    rank[j] = old + __popc(peers & lt);
    __syncwarp();
    if (lane == 31 - __clz(peers)) S.whist[w][d] = (unsigned short)(old + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread t = digit t): per-warp exclusive offsets and the tile count
  unsigned cnt = 0;
  for (int ww = 0; ww < kSortWarps; ++ww) {
    const unsigned c = S.whist[ww][t];
    S.whist[ww][t] = (unsigned short)cnt;
    cnt += c;
  }
  // tile-local start of each digit's run: exclusive scan over digits
  {
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) S.wsum[w] = incl;
    __syncthreads();
    unsigned before = 0;
    for (int i = 0; i < w; ++i) before += S.wsum[i];
    S.dstart[t] = before + incl - cnt;
  }
  // decoupled look-back: this tile's exclusive prefix of digit t over earlier tiles
  {
    unsigned excl = 0;
    if (tile == 0) {
      st_relaxed(status + t, kFlagP | cnt);
    } else {
      st_relaxed(status + (size_t)tile * kBins + t, kFlagA | cnt);
      int prev = tile - 1;
      for (;;) {
        unsigned v;
        do {
          v = ld_relaxed(status + (size_t)prev * kBins + t);
        } while ((v & ~kValMask) == 0u);
        excl += v & kValMask;
        if (v & kFlagP) break;
        --prev;
      }
      st_relaxed(status + (size_t)tile * kBins + t, kFlagP | (excl + cnt));
    }
    S.gbase[t] = goff[t] + excl;
  }
  __syncthreads();
  // reorder the tile in shared memory (digit runs in index order) ...
#pragma unroll
  for (int j = 0; j < kIPT; ++j) {
    const int d = dig[j];
    if (d < kBins) {
      const unsigned pos = S.dstart[d] + S.whist[w][d] + rank[j];
      S.keys[pos] = key[j];
      S.vals[pos] = val[j];
    }
  }
  __syncthreads();
  // ... and write each run to its global place (consecutive threads, consecutive addresses)
  const int valid = (int)min((int64_t)kTile, (int64_t)n - base);
  for (int i = t; i < valid; i += kSortThreads) {
    const unsigned long long k = S.keys[i];
    const int d = (int)((unsigned)(k >> shift) & (kBins - 1));
    const size_t g = (size_t)S.gbase[d] + (unsigned)(i - S.dstart[d]);
    kout[g] = k;
    vout[g] = S.vals[i];
  }
}

}  // namespace

size_t radix_sort_temp_bytes(int n) {
  const size_t tiles = ((size_t)n + kTile - 1) / kTile;
  return sizeof(unsigned) * (2 * kPasses * kBins + tiles * kBins) + 64 * sizeof(int);
}

// keys_a/vals_a (input, overwritten) -> keys_b/vals_b (sorted, stable)
void radix_sort_pairs(cudaStream_t s, int n, unsigned long long *keys_a, uint32_t *vals_a, unsigned long long *keys_b,
                      uint32_t *vals_b, void *temp) {
  if (n <= 0) return;
  const int tiles = (n + kTile - 1) / kTile;
  unsigned *ghist = reinterpret_cast<unsigned *>(temp);
  unsigned *goff = ghist + kPasses * kBins;
  unsigned *status = goff + kPasses * kBins;
  int *counters = reinterpret_cast<int *>(status + (size_t)tiles * kBins);
  cudaMemsetAsync(ghist, 0, sizeof(unsigned) * kPasses * kBins, s);
  cudaMemsetAsync(counters, 0, sizeof(int) * kPasses, s);
  k_digit_hist<<<std::min((n + 4095) / 4096, 1184), 256, 0, s>>>(n, keys_a, ghist);
  k_digit_scan<<<1, kBins, 0, s>>>(ghist, goff);
  const size_t smem = sizeof(SortSmem);
  cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long *ki = keys_a, *ko = keys_b;
  uint32_t *vi = vals_a, *vo = vals_b;
  for (int p = 0; p < kPasses; ++p) {
    cudaMemsetAsync(status, 0, sizeof(unsigned) * (size_t)tiles * kBins, s);
    k_onesweep<<<tiles, kSortThreads, smem, s>>>(n, kDigitBits * p, ki, vi, ko, vo, goff + p * kBins, status,
                                                 counters + p);
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  // 7 passes: the last one wrote keys_b / vals_b
}

}  // namespace sph
