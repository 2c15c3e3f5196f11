// sph_scan.cu -- single-pass exclusive scan and stream compaction with
// decoupled look-back (the plumbing of the ordering and of the per-round
// target lists; no library kernels on the pass).
//
//   scan_exclusive_i32  out[i] = sum of in[0..i) (in place allowed), the node
//                       offsets of the search tree (k_node_count -> noff)
//   select_state        list_out = [p in list_in : state[p] == want] in
//                       order, *count_out = its length (the compacted target
//                       lists of the fallback rounds and the ghost seeding)
//
// A tile of 4096 items (512 threads x 8) reduces its items, publishes the
// aggregate, takes its exclusive prefix from earlier tiles by look-back (tile
// ids from an atomic counter, in launch order) and writes its outputs.
#include "sph_internal.cuh"

namespace sph {
namespace {

constexpr int kT = 512;
constexpr int kI = 8;
constexpr int kTileN = kT * kI;
constexpr unsigned long long kFA = 1ull << 62;
constexpr unsigned long long kFP = 2ull << 62;
constexpr unsigned long long kVM = (1ull << 62) - 1ull;

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// block-wide exclusive scan of one value per thread; returns the block total
__device__ __forceinline__ long long block_excl(long long v, long long &excl, long long *wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  long long before = 0, tot = 0;
  for (int i = 0; i < kT / 32; ++i) {
    if (i < w) before += wsum[i];
    tot += wsum[i];
  }
  excl = before + incl - v;
  return tot;
}

// the tile's exclusive prefix over earlier tiles (thread 0 looks back)
__device__ __forceinline__ long long lookback(int tile, long long agg, unsigned long long *status, long long *sh) {
  if (threadIdx.x == 0) {
    long long excl = 0;
    if (tile == 0) {
      st_relaxed64(status, kFP | (unsigned long long)agg);
    } else {
      st_relaxed64(status + tile, kFA | (unsigned long long)agg);
      for (int prev = tile - 1;; --prev) {
        unsigned long long v;
        do {
          v = ld_relaxed64(status + prev);
        } while ((v & ~kVM) == 0ull);
        excl += (long long)(v & kVM);
        if (v & kFP) break;
      }
      st_relaxed64(status + tile, kFP | (unsigned long long)(excl + agg));
    }
    *sh = excl;
  }
  __syncthreads();
  return *sh;
}

template <bool SELECT>
__global__ void __launch_bounds__(kT) k_scan(int n, const int *__restrict__ in, int *__restrict__ out,
                                             const uint32_t *__restrict__ list_in, const uint8_t *__restrict__ state,
                                             uint8_t want, uint32_t *__restrict__ list_out, int *__restrict__ count_out,
                                             unsigned long long *__restrict__ status, int *__restrict__ counter) {
  __shared__ long long wsum[kT / 32];
  __shared__ long long sh;
  __shared__ int stile;
  if (threadIdx.x == 0) stile = atomicAdd(counter, 1);
  __syncthreads();
  const int tile = stile;
  // thread t owns items [base + t*kI, base + t*kI + kI): contiguous, so the
  // block scan of per-thread sums gives each its start
  const long long base = (long long)tile * kTileN + (long long)threadIdx.x * kI;
  int v[kI];
  uint32_t item[kI];
  long long sum = 0;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const long long i = base + j;
    if constexpr (SELECT) {
      item[j] = i < n ? list_in[i] : 0u;
      v[j] = (i < n && state[item[j]] == want) ? 1 : 0;
    } else {
      v[j] = i < n ? in[i] : 0;
    }
    sum += v[j];
  }
  long long texcl;
  const long long agg = block_excl(sum, texcl, wsum);
  const long long prefix = lookback(tile, agg, status, &sh);
  long long run = prefix + texcl;
#pragma unroll
  for (int j = 0; j < kI; ++j) {
    const long long i = base + j;
    if (i < n) {
      if constexpr (SELECT) {
        if (v[j]) list_out[run] = item[j];
      } else {
        out[i] = (int)run;
      }
    }
    run += v[j];
  }
  if constexpr (SELECT) {
    // the last tile knows the total
    if (tile == (n + kTileN - 1) / kTileN - 1 && threadIdx.x == 0) *count_out = (int)(prefix + agg);
  }
}

}  // namespace

size_t scan_temp_bytes(int n) {
  return sizeof(unsigned long long) * ((size_t)(n + kTileN - 1) / kTileN + 1) + 64;
}

void scan_exclusive_i32(cudaStream_t s, const int *in, int *out, int n, void *temp) {
  if (n <= 0) return;
  const int tiles = (n + kTileN - 1) / kTileN;
  unsigned long long *status = reinterpret_cast<unsigned long long *>(temp);
  int *counter = reinterpret_cast<int *>(status + tiles);
  cudaMemsetAsync(temp, 0, sizeof(unsigned long long) * tiles + sizeof(int), s);
  k_scan<false><<<tiles, kT, 0, s>>>(n, in, out, nullptr, nullptr, 0, nullptr, nullptr, status, counter);
}

void select_state(cudaStream_t s, const uint32_t *list_in, int n_in, const uint8_t *state, uint8_t want,
                  uint32_t *list_out, int *count_out, void *temp) {
  if (n_in <= 0) {
    cudaMemsetAsync(count_out, 0, sizeof(int), s);
    return;
  }
  const int tiles = (n_in + kTileN - 1) / kTileN;
  unsigned long long *status = reinterpret_cast<unsigned long long *>(temp);
  int *counter = reinterpret_cast<int *>(status + tiles);
  cudaMemsetAsync(temp, 0, sizeof(unsigned long long) * tiles + sizeof(int), s);
  k_scan<true><<<tiles, kT, 0, s>>>(n_in, nullptr, nullptr, list_in, state, want, list_out, count_out, status,
                                    counter);
}

}  // namespace sph
