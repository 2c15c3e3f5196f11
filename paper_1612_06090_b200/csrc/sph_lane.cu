// One LANE per target: a warp serves a bundle of 32 consecutive sorted
// targets (spatial neighbours) that share one candidate stream.
//
// The per-target kernel (sph_warp.cu) spends ~3,200 warp instructions per
// target, most of them on per-candidate bookkeeping that is paid per 32
// candidate SLOTS (slot owner, ballots, list appends).  Here the roles are
// turned round: the candidates of the bundle's neighbourhood are staged into
// shared memory once (cp.async.bulk per search cell, double-buffered tiles on
// two mbarriers) and every lane tests each staged candidate against ITS OWN
// target (one broadcast LDS.128 + the fp32 d2 per 32 pair tests), so a pair
// test costs 1/32 of a warp instruction slot per op and nothing in the inner
// loops crosses lanes.  Per bundle (reference compute_density_pass,
// density.py:286-413; the radius search of density.py:215-246 replaced by an
// exact K-th selection):
//   radius  R_i = the tree's estimate R0 of the target's cell x the calq
//           quantile of h / R0 over a sparse calibration sample run through the
//           per-target kernel first, per half-octave class of R0 (cal != null);
//           or margin x the larger converged h of the two dense seeds around
//           the target (k_seed_radius, cal == null); lanes far from the
//           bundle's bulk or whose sphere crosses a periodic face are left to
//           the per-target kernel;
//   walk    the search tree once with the bundle box grown by max R (and the
//           bundle's bounding sphere); each hit cell is kept if it meets at
//           least one lane's own sphere; memory-adjacent cells merge into runs;
//   pass 1  stream the runs; each landed tile is rewritten in the bundle's
//           frame, (x', y', z', |c'|^2), so a pair test is three FFMAs; per
//           lane a 64-bin histogram of d2 over [0, R_i^2) (one column of
//           16-bit counters per lane) -> the bin holding the K-th neighbour;
//   pass 2  stream again: per lane the list of every candidate up to that
//           bin's upper edge (K + a few entries, 16-bit run codes);
//   select  per lane over its list, from the raw positions: exact unfused
//           fp64 d2 (octree.py:211-214) for entries in the guard band of the
//           bin, count below + rank inside -> d2_K (h = sqrt(d2_K),
//           density.py:226-245);
//   sum     rho = sum over list entries within h of m_j W(r/h), self included
//           (density.py:160-171, 249-261; kernel.py:30-45).
// Lanes the bundle cannot finish (fewer than K within R_i, list or bracket too
// crowded, table overflow) keep ST_NEED_HIST and are appended to fb_list for
// the per-target kernel, with a radius hint where the histogram gives one.
#include "sph_internal.cuh"
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kLWarps = 2;
#ifndef SPH_LANE_TILE
#define SPH_LANE_TILE 96
#endif
#ifndef SPH_LANE_CELLS
#define SPH_LANE_CELLS 256
#endif
constexpr int kTile = SPH_LANE_TILE;    // candidates per staged tile (>= the largest search cell)
constexpr int kCells = SPH_LANE_CELLS;   // runs of cells per bundle
#ifndef SPH_LANE_BINS
#define SPH_LANE_BINS 64
#endif
constexpr int kBins = SPH_LANE_BINS;     // histogram bins over [0, R^2)
constexpr int kLStack = 96;   // traversal stack (internal node ids)
constexpr int kInb = kTile / 8;  // in-bracket entries per lane (doubles; alias the tile buffers)
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard (as sph_warp.cu)
constexpr double kEpsD = 9.5367431640625e-07;
static_assert(kInb * 32 * 8 <= 2 * kTile * 16, "in-bracket buffer aliases the tile buffers");

// per warp: mbarriers | tile buffers (the walk's cell boxes and, after pass 2, the in-bracket doubles live there
// too) | run starts | stack | lists (16-bit run codes; the 16-bit histogram lives there until pass 2 starts) |
// run codes of the staged tile | run offsets (16-bit)
__host__ __device__ constexpr int lane_smem_bytes(int lcap) {
  return (16 + 2 * kTile * 16 + kCells * 4 + kLStack * 4 + lcap * 64 + 2 * kTile * 2 + (kCells + 8) * 2 + 15) & ~15;
}
static_assert(kCells <= 512 && kTile <= 128, "a list entry is (run << 7 | offset) in 16 bits");

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float warp_min(float v) {
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// counters (a.kn_counters): [0] bundles bailed (table / stack / cell size), [1] lanes with fewer than K within R,
// [2] lanes whose list would overflow, [3] lanes whose bracket could not be ranked, [13] lanes left out of their
// bundle (far from its bulk / periodic face)
__global__ void __launch_bounds__(kLWarps * 32) k_lane(const PassArgs a, int lcap, float rscale, float exc, int max_stream, const float *cal, float calq) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *wb = smem_raw + (size_t)wib * lane_smem_bytes(lcap);
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(wb);
  float4 *tile = reinterpret_cast<float4 *>(wb + 16);
  float4 *sbox = tile;
  double *inb = reinterpret_cast<double *>(tile);
  int *cstart = reinterpret_cast<int *>(tile + 2 * kTile);
  int *stk = cstart + kCells;
  unsigned short *list = reinterpret_cast<unsigned short *>(stk + kLStack);
  unsigned short *hist = list;
  unsigned short *tcode = list + lcap * 32;  // run code of each staged candidate (pass 2)
  unsigned short *coff = tcode + 2 * kTile;

  const float4 *__restrict__ pos = reinterpret_cast<const float4 *>(a.pos);
  const float4 *__restrict__ posj = a.posj;
  const float4 *__restrict__ crec = a.tree.crec;
  const int n = a.n;
  const int K = a.k;
  const unsigned lt_mask = (1u << lane) - 1u;
  const double norm = a.kernel_kind == 0 ? kWc6Norm : kM4Norm;
  const float boxf = (float)a.box;

  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned phase = 0;  // bit b: parity of the next wait on bars[b]

  unsigned long long tests = 0, accepted = 0;
  int c_bail = 0, c_few = 0, c_full = 0, c_rank = 0, c_out = 0;
  // calibration of the tree's radius estimate: the calq quantile of log(h / R0) over a sparse sample of
  // converged targets, per class of R0 (half octaves, 16 classes: the estimate's bias depends on the local
  // scale), 64 bins over [-1.5, 1.5) each; lane c < 16 holds class c's log-quantile, classes with fewer than
  // 64 samples use the quantile over all classes
  float qcls = 0.f;
  if (cal) {
    const int *cb = reinterpret_cast<const int *>(cal);
    auto quantile = [&](auto count_of) {  // count_of(bin) -> samples in that bin
      int total = 0;
      for (int bb = 0; bb < 64; ++bb) total += count_of(bb);
      if (total < 64) return make_float2(0.f, (float)total);
      const float want = calq * (float)total;
      int cum = 0, bb = 0;
      for (; bb < 63; ++bb) {
        const int c = count_of(bb);
        if ((float)(cum + c) >= want) break;
        cum += c;
      }
      const float frac = (want - (float)cum) / fmaxf((float)count_of(bb), 1.f);
      return make_float2(-1.5f + ((float)bb + fminf(frac, 1.f)) * (3.0f / 64.0f), (float)total);
    };
    const float2 all = quantile([&](int bb) {
      int c = 0;
      for (int k = 0; k < 16; ++k) c += cb[k * 64 + bb];
      return c;
    });
    const int mycls = lane & 15;
    const float2 mine = quantile([&](int bb) { return cb[mycls * 64 + bb]; });
    qcls = mine.y >= 64.f ? mine.x : all.x;
  }
  auto r0_class = [](float r0) { return (__float_as_int(r0) >> 22) & 15; };

  const int nb = (n + 31) >> 5;
  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(a.work_counter, 1);
    b = __shfl_sync(FULL, b, 0);
    if (b >= nb) break;
    const int p = b * 32 + lane;
    const bool want = p < n && a.state[p] == ST_NEED_HIST;
    bool act = want;
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    float R = 0.f;
    const float r0v = want ? a.radius[p] : 1.f;
    const float qf = cal ? expf(__shfl_sync(FULL, qcls, r0_class(r0v))) : 1.f;  // the class's h / R0 quantile
    if (want) {
      t = pos[p];
      R = r0v * rscale * qf;
      R = fminf(R, a.rmax);
      if (!(R > 0.f)) act = false;
      // spheres crossing a periodic face are searched with image shifts: the per-target kernel
      if (a.periodic) {
        const float m = R * 1.0001f;
        if (t.x - m < 0.f || t.y - m < 0.f || t.z - m < 0.f || t.x + m > boxf || t.y + m > boxf || t.z + m > boxf)
          act = false;
      }
    }
    unsigned am = __ballot_sync(FULL, act);
    bool done = false;  // this lane's target finished here
    // origin of the bundle's local frame (the mean of its targets) and each lane's reach from it
    float ox = 0.f, oy = 0.f, oz = 0.f, reach = 0.f;
    if (am) {
      const float na = (float)__popc(am);
      ox = warp_sum(act ? t.x : 0.f) / na;
      oy = warp_sum(act ? t.y : 0.f) / na;
      oz = warp_sum(act ? t.z : 0.f) / na;
      const float ddx = t.x - ox, ddy = t.y - oy, ddz = t.z - oz;
      reach = act ? sqrtf(ddx * ddx + ddy * ddy + ddz * ddz) + R : 0.f;
      // ---- lanes far from the bundle's bulk are left out (their spheres would widen the shared stream) ----
      if (exc > 0.f) {
        int rank = 0;
        for (int l = 0; l < 32; ++l) {
          const float v = __shfl_sync(FULL, reach, l);
          rank += (v > 0.f) && (v < reach || (v == reach && l < lane));
        }
        const unsigned mm = __ballot_sync(FULL, act && rank == (__popc(am) >> 1));
        const float med = __shfl_sync(FULL, reach, __ffs(mm) - 1);
        if (act && reach > exc * med) {
          act = false;
          ++c_out;
        }
        am = __ballot_sync(FULL, act);
      }
    }
    if (am) {
      const float R2g = act ? R * R * (1.0f + 16.0f * kEps) : -1.f;
      const float Rmax = warp_max(act ? R : 0.f);
      const float blx = warp_min(act ? t.x : INFINITY), bly = warp_min(act ? t.y : INFINITY),
                  blz = warp_min(act ? t.z : INFINITY);
      const float bhx = warp_max(act ? t.x : -INFINITY), bhy = warp_max(act ? t.y : -INFINITY),
                  bhz = warp_max(act ? t.z : -INFINITY);
      const float Rm2g = Rmax * Rmax * (1.0f + 16.0f * kEps);
      const float reach_max = warp_max(act ? reach : 0.f) * (1.0f + 16.0f * kEps);  // reach is itself rounded
      const float reach2g = reach_max * reach_max * (1.0f + 16.0f * kEps);

      // ---- walk: cells within Rmax of the bundle box, kept if they meet some lane's own sphere ----
      int start = a.tree.root_start;
      {
        const int pf = b * 32 + __ffs(am) - 1;
        const int4 an = a.tree.anc4[a.tree.cellof[pf]];
        // node cubes are rounded outward to fp32: one more ulp of the coordinates in the margin
        const float cmax = fmaxf(fmaxf(fmaxf(fabsf(blx), fabsf(bhx)), fmaxf(fabsf(bly), fabsf(bhy))),
                                 fmaxf(fabsf(blz), fabsf(bhz)));
        const float Dm = Rmax * (1.0f + 8.0f * kEps) + cmax * 2.4e-7f;
        const int my_anc = lane == 0 ? an.x : lane == 1 ? an.y : lane == 2 ? an.z : lane == 3 ? an.w : -1;
        bool holds = false;
        if (my_anc >= 0) {
          const float4 l4 = a.tree.nlo[my_anc], h4 = a.tree.nhi[my_anc];
          holds = l4.x <= blx - Dm && bhx + Dm <= h4.x && l4.y <= bly - Dm && bhy + Dm <= h4.y && l4.z <= blz - Dm &&
                  bhz + Dm <= h4.z;
        }
        const unsigned hm = __ballot_sync(FULL, holds);
        if (hm) start = __shfl_sync(FULL, my_anc, __ffs(hm) - 1);
      }
      if (lane == 0) stk[0] = start;
      int top = 1, nt = 0, total = 0, run_end = -1, run_cnt = 0;
      bool bail = false;
      __syncwarp();
      while (top > 0 && !bail) {
        const int np = min(top, 4);
        top -= np;
        const int pi = lane >> 3;
        const int par = pi < np ? stk[top + pi] : -1;
        __syncwarp();
        bool hit = false, is_cell = false;
        float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
        if (par >= 0) {
          const float4 *rec = crec + 16 * (size_t)par + 2 * (lane & 7);
          l4 = rec[0];
          h4 = rec[1];
          is_cell = __float_as_int(l4.w) < 0;
          const float gx = fmaxf(fmaxf(l4.x - bhx, blx - h4.x), 0.f);
          const float gy = fmaxf(fmaxf(l4.y - bhy, bly - h4.y), 0.f);
          const float gz = fmaxf(fmaxf(l4.z - bhz, blz - h4.z), 0.f);
          // ... and within the bundle's bounding sphere (centre o, radius = the largest reach)
          const float sx = fmaxf(fmaxf(l4.x - ox, ox - h4.x), 0.f);
          const float sy = fmaxf(fmaxf(l4.y - oy, oy - h4.y), 0.f);
          const float sz = fmaxf(fmaxf(l4.z - oz, oz - h4.z), 0.f);
          hit = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= Rm2g &&
                (sx * sx + sy * sy + sz * sz) * (1.0f - 4.0f * kEps) <= reach2g;
        }
        const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
        if (top + __popc(pm) > kLStack) { bail = true; break; }
        if (hit && !is_cell) stk[top + __popc(pm & lt_mask)] = __float_as_int(l4.w);
        top += __popc(pm);
        const unsigned cm = __ballot_sync(FULL, hit && is_cell);
        // room for the step's cells; a ragged bundle (long stream) is cheaper in the per-target kernel
        if (nt + __popc(cm) > kCells || total > max_stream) { bail = true; break; }
        if (cm) {
          if (hit && is_cell) {
            const int kk = __popc(cm & lt_mask);
            sbox[2 * kk] = l4;
            sbox[2 * kk + 1] = h4;
          }
          __syncwarp();
          const int nc = __popc(cm);
          for (int kk = 0; kk < nc; ++kk) {
            const float4 L = sbox[2 * kk], H = sbox[2 * kk + 1];
            const float gx = fmaxf(fmaxf(L.x - t.x, t.x - H.x), 0.f);
            const float gy = fmaxf(fmaxf(L.y - t.y, t.y - H.y), 0.f);
            const float gz = fmaxf(fmaxf(L.z - t.z, t.z - H.z), 0.f);
            const bool need = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= R2g;
            if (__any_sync(FULL, need)) {
              const int s0 = ~__float_as_int(L.w);
              const int cnt = __float_as_int(H.w) - s0;
              if (s0 == run_end && run_cnt + cnt <= kTile) {
                // next to the last kept cell in memory: one copy serves both
                run_cnt += cnt;
              } else {
                if (cnt > kTile) { bail = true; break; }
                if (lane == 0) {
                  cstart[nt] = s0;
                  coff[nt] = (unsigned short)total;
                }
                ++nt;
                run_cnt = cnt;
              }
              run_end = s0 + cnt;
              total += cnt;
            }
          }
        }
        __syncwarp();
      }
      if (lane == 0) coff[nt] = (unsigned short)total;
      __syncwarp();
      if (bail || nt == 0) {
        ++c_bail;
      } else {
        // ---- tile streaming: cells [c0, c0 + nc) whose candidates fit one tile ----
        auto issue = [&](int c0, int buf, int &nc, int &cnt) {
          const int base = coff[c0];
          const int ci = c0 + lane;
          const int e = ci < nt ? (int)coff[ci + 1] - base : INT_MAX;
          nc = __popc(__ballot_sync(FULL, e <= kTile));
          cnt = __shfl_sync(FULL, e, nc - 1);
          if (lane == 0) mbar_arrive_expect_tx(&bars[buf], (unsigned)cnt * 16u);
          __syncwarp();
          if (lane < nc) {
            const int o = (int)coff[ci] - base;
            bulk_g2s(tile + buf * kTile + o, posj + cstart[ci], (unsigned)(e - o) * 16u, &bars[buf]);
          }
        };
        auto stream = [&](auto codes, auto body4, auto body1) {
          constexpr bool kCodes = decltype(codes)::value;
          int c0 = 0, buf = 0, nc_cur = 0, cnt_cur = 0;
          issue(0, 0, nc_cur, cnt_cur);
          for (;;) {
            const int c1 = c0 + nc_cur;
            int nc_nxt = 0, cnt_nxt = 0;
            if (c1 < nt) issue(c1, buf ^ 1, nc_nxt, cnt_nxt);
            while (!mbar_try_wait(&bars[buf], (phase >> buf) & 1u)) {}
            phase ^= 1u << buf;
            float4 *tb = tile + buf * kTile;
            unsigned short *tc = tcode + buf * kTile;
            // staged (x, y, z, index) -> the bundle's frame: (x', y', z', |c'|^2); pass 2 also needs each
            // candidate's run code (run << 7 | offset in the run): the run by bisection of the tile's offsets
            const int sp0 = coff[c0];
            for (int q = lane; q < cnt_cur; q += 32) {
              const float4 c = tb[q];
              const float x = c.x - ox, y = c.y - oy, z = c.z - oz;
              tb[q] = make_float4(x, y, z, fmaf(x, x, fmaf(y, y, z * z)));
              if constexpr (kCodes) {
                const int sp = sp0 + q;
                int lo = c0, hi = c1;
                while (hi - lo > 1) {
                  const int mid = (lo + hi) >> 1;
                  if ((int)coff[mid] <= sp) lo = mid; else hi = mid;
                }
                tc[q] = (unsigned short)((lo << 7) | (sp - (int)coff[lo]));
              }
            }
            __syncwarp();
            // four candidates (and their codes) loaded ahead of their tests: the tests write shared
            // memory, so the compiler would not hoist the loads itself
            const float4 *tq = tb;
            const uint2 *iq = reinterpret_cast<const uint2 *>(tc);
            int left = cnt_cur;
#pragma unroll 2
            for (; left >= 4; left -= 4, tq += 4, ++iq) {
              uint2 cd = make_uint2(0u, 0u);
              if constexpr (kCodes) cd = iq[0];
              body4(tq[0], tq[1], tq[2], tq[3], cd);
            }
            const unsigned short *i1 = reinterpret_cast<const unsigned short *>(iq);
            for (int s = 0; s < left; ++s) body1(tq[s], kCodes ? (unsigned)i1[s] : 0u);
            __syncwarp();
            if (c1 >= nt) break;
            c0 = c1;
            nc_cur = nc_nxt;
            cnt_cur = cnt_nxt;
            buf ^= 1;
          }
        };

        // ---- pass 1: per-lane histogram of d2 over [0, R^2) ----
#pragma unroll
        for (int bb = 0; bb <= kBins; ++bb) hist[bb * 32 + lane] = 0;
        __syncwarp();
        // d2 = |c' - t'|^2 = (|c'|^2 - 2 t'.c') + |t'|^2 in the bundle's frame: three FFMAs per candidate.  The
        // value is within E = 2^-18 reach^2 of the exact d2 wherever it matters (|c'| <= reach), which only
        // decides what is listed; the select below works on the unfused differences of the raw positions.
        const float scale = act ? (float)kBins / (R * R) : 0.f;
        const float tpx = t.x - ox, tpy = t.y - oy, tpz = t.z - oz;
        const float m2x = act ? -2.0f * tpx : 0.f, m2y = act ? -2.0f * tpy : 0.f, m2z = act ? -2.0f * tpz : 0.f;
        const float t2s = act ? fmaf(tpx, tpx, fmaf(tpy, tpy, tpz * tpz)) * scale : 0.f;
        unsigned short *hcol = hist + lane;  // 16-bit counters: two lanes per bank word, at most 2-way conflicts
        // own column, plain read-modify-write (shared atomics cost 2 cycles per lane; reading four counters
        // ahead and fixing repeated bins in registers measured the same at 20 warps per SM)
        auto bin_of = [&](const float4 c) {
          const float sv = fmaf(m2x, c.x, fmaf(m2y, c.y, fmaf(m2z, c.z, c.w)));
          return __float2uint_rz(fminf(fmaf(sv, scale, t2s), (float)kBins)) << 5;  // bin kBins: beyond R
        };
        stream(
            std::false_type{},
            [&](const float4 q0, const float4 q1, const float4 q2, const float4 q3, const uint2) {
              const unsigned b0 = bin_of(q0), b1 = bin_of(q1), b2 = bin_of(q2), b3 = bin_of(q3);
              hcol[b0] += 1;
              hcol[b1] += 1;
              hcol[b2] += 1;
              hcol[b3] += 1;
            },
            [&](const float4 c, const unsigned) { hcol[bin_of(c)] += 1; });
        tests += (unsigned long long)total * (unsigned)__popc(am);
        // the bin holding the K-th other (self counted at d2 = 0): cumulative count >= K + 1
        int cum = 0, bsel = -1, csel = 0;
#pragma unroll
        for (int bb = 0; bb < kBins; ++bb) {
          cum += (int)hcol[bb << 5];
          if (bsel < 0 && cum >= K + 1) {
            bsel = bb;
            csel = cum;
          }
        }
        bool ok = act;
        if (ok && bsel < 0) {
          ok = false;
          ++c_few;
          // the per-target kernel starts from the radius the count within R suggests (its own growth rule)
          const int others = cum - 1;
          const float f = others > 0 ? cbrtf((float)(K + 8) / (float)others) * 1.1f : 2.f;
          a.radius[p] = fminf(R * fminf(fmaxf(f, 1.1f), 2.5f), a.rmax);
        }
        // a lane that does not finish below still knows the K-th lies in bin bsel: a tight radius for the
        // per-target kernel (overwritten when the lane finishes)
        if (ok) a.radius[p] = fminf(R * sqrtf((float)(bsel + 1) / (float)kBins) * 1.002f, a.rmax);
        if (ok && csel > lcap) {
          ok = false;
          ++c_full;
        }
        const unsigned okm = __ballot_sync(FULL, ok);
        if (okm) {
          // ---- pass 2: per-lane list of every candidate up to the bin's upper edge ----
          // sv <= thr_s <=> its pass-1 bin <= bsel: thr_s is the largest float whose scaled value stays below
          // bsel + 1 (the FFMA is monotone in sv; bisection over the ordered bit patterns), so the list length
          // is the histogram's count
          float thr_s = -INFINITY;
          if (ok) {
            const float B = (float)(bsel + 1);
            auto ord2f = [](unsigned o) { return __uint_as_float((o & 0x80000000u) ? (o ^ 0x80000000u) : ~o); };
            unsigned lo_o = 0x00800000u, hi_o = 0xff7fffffu;  // -FLT_MAX (listed), +FLT_MAX (not listed)
            while (hi_o - lo_o > 1u) {
              const unsigned mid = lo_o + ((hi_o - lo_o) >> 1);
              if (fmaf(ord2f(mid), scale, t2s) < B) lo_o = mid; else hi_o = mid;
            }
            thr_s = ord2f(lo_o);
          }
          const unsigned lp0 = smem_u32(list + lane);
          unsigned lp = lp0;
          auto keep = [&](const float4 c, const unsigned code) {
            const float sv = fmaf(m2x, c.x, fmaf(m2y, c.y, fmaf(m2z, c.z, c.w)));
            if (sv <= thr_s) {
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(lp), "h"((unsigned short)code) : "memory");
              lp += 64u;
            }
          };
          stream(
              std::true_type{},
              [&](const float4 q0, const float4 q1, const float4 q2, const float4 q3, const uint2 cd) {
                keep(q0, cd.x & 0xffffu);
                keep(q1, cd.x >> 16);
                keep(q2, cd.y & 0xffffu);
                keep(q3, cd.y >> 16);
              },
              keep);
          tests += (unsigned long long)total * (unsigned)__popc(okm);
          const int cnt = (int)((lp - lp0) >> 6);
          int maxcnt = cnt;
          for (int o = 16; o; o >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(FULL, maxcnt, o));

          // ---- select: exact count below the bin, exact fp64 d2 inside its guard band ----
          const double sc_d = (double)scale;
          const double E = 3.9e-6 * (double)reach * (double)reach;  // > 2^-18 reach^2
          const double tl = ok ? fmax((double)bsel / sc_d * (1.0 - 8.0 * kEpsD) - E, 0.0) : 0.0;
          const double th = ok ? fmax((double)(bsel + 1) / sc_d * (1.0 - 4.0 * kEpsD) - E, tl) : 0.0;
          const float lo_f = __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f;
          const float hi_f = __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f;
          // a list entry is a run code: sorted index = the run's start + the offset
          auto entry = [&](int slot) {
            const unsigned code = list[slot];
            return cstart[code >> 7] + (int)(code & 127u);
          };
          int below = 0, n_in = 0;
          auto classify = [&](const int j, const float4 c) {
            const float dx = c.x - t.x, dy = c.y - t.y, dz = c.z - t.z;
            const float af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (af < lo_f) {
              ++below;
            } else if (af <= hi_f) {
              const double ex = exact_d2(__dsub_rn((double)c.x, (double)t.x), __dsub_rn((double)c.y, (double)t.y),
                                         __dsub_rn((double)c.z, (double)t.z));
              if (ex < tl) {
                ++below;
              } else if (ex <= th) {
                if (n_in < kInb) inb[n_in * 32 + lane] = ex;
                ++n_in;
              }
            }
          };
          for (int e = 0; e < maxcnt; e += 4) {  // four gathers in flight
            int j[4];
            float4 c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) j[u] = e + u < cnt ? entry((e + u) * 32 + lane) : p;
#pragma unroll
            for (int u = 0; u < 4; ++u) c[u] = pos[j[u]];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (j[u] != p) classify(j[u], c[u]);
          }
          const int r = K - below;  // 1-based rank of the K-th inside the bracket
          if (ok && (n_in > kInb || r < 1 || r > n_in)) {
            ok = false;
            ++c_rank;
          }
          double d2k = INFINITY;
          if (ok) {
            for (int i = 0; i < n_in; ++i) {
              const double ei = inb[i * 32 + lane];
              int less = 0, eq = 0;
              for (int jj = 0; jj < n_in; ++jj) {
                const double ej = inb[jj * 32 + lane];
                less += ej < ei;
                eq += ej == ei;
              }
              if (less < r && r <= less + eq) d2k = ei;
            }
          }

          // ---- density over the list entries within h ----
          double rho = 0.0;
          if (ok && d2k > 0.0) {
            const double hh = __dsqrt_rn(d2k);
            const double norm_h3 = __ddiv_rn(norm, __dmul_rn(__dmul_rn(hh, hh), hh));
            const float d2k_f = __double2float_ru(d2k * (1.0 + kEpsD));
            const float inv_h = (float)(1.0 / hh);
            float accf = 0.f;
            auto term = [&](const float4 c) {
              const float dx = c.x - t.x, dy = c.y - t.y, dz = c.z - t.z;
              const float af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
              if (af < d2k_f) {
                ++accepted;
                const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
                const float q = rr * inv_h;
                const float wv = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
                if (q < 1.f) accf = fmaf(c.w, wv, accf);
              }
            };
            if (a.dens64) {
              // fp64 positions that are fp32 values (precision "auto"): every term as the reference computes it
              // (density.py:160-171: exact d2, sqrt, W, mass in fp64); only the order of the sum differs
              double accd = 0.0;
              for (int e = 0; e < cnt; ++e) {
                const int j = entry(e * 32 + lane);
                const float4 c = pos[j];
                const float dx = c.x - t.x, dy = c.y - t.y, dz = c.z - t.z;
                if (!(fmaf(dx, dx, fmaf(dy, dy, dz * dz)) < d2k_f)) continue;
                const double ex = exact_d2(__dsub_rn((double)c.x, (double)t.x), __dsub_rn((double)c.y, (double)t.y),
                                           __dsub_rn((double)c.z, (double)t.z));
                if (ex < d2k) {
                  ++accepted;
                  const double r_ = __dsqrt_rn(ex);
                  double wv;
                  if (a.kernel_kind == 0) {
                    wv = wc6_lowered(r_, hh, norm_h3);
                  } else {
                    const double q = __ddiv_rn(r_, hh);
                    wv = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
                  }
                  accd = __dadd_rn(accd, __dmul_rn(a.mass64[j], wv));
                }
              }
              rho = accd;
            } else {
            int e = 0;
            for (; e + 4 <= cnt; e += 4) {
              float4 c[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) c[u] = pos[entry((e + u) * 32 + lane)];
#pragma unroll
              for (int u = 0; u < 4; ++u) term(c[u]);
            }
            for (; e < cnt; ++e) term(pos[entry(e * 32 + lane)]);
            rho = __dmul_rn(norm_h3, (double)accf);
            }
          }
          if (ok) {
            a.d2k[p] = d2k;
            a.rho[p] = rho;
            a.radius[p] = R;
            a.state[p] = ST_FINAL;
            done = true;
          }
          __syncwarp();
        }
      }
    }
    // ---- what is left goes to the per-target kernel ----
    const unsigned fm = __ballot_sync(FULL, want && !done);
    if (fm && a.fb_list) {
      int base = 0;
      if (lane == 0) base = atomicAdd(a.fb_count, __popc(fm));
      base = __shfl_sync(FULL, base, 0);
      if (want && !done) a.fb_list[base + __popc(fm & lt_mask)] = (uint32_t)p;
    }
  }
  for (int o = 16; o; o >>= 1) {
    accepted += __shfl_xor_sync(FULL, accepted, o);
    c_few += __shfl_xor_sync(FULL, c_few, o);
    c_full += __shfl_xor_sync(FULL, c_full, o);
    c_rank += __shfl_xor_sync(FULL, c_rank, o);
    c_out += __shfl_xor_sync(FULL, c_out, o);
  }
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
    if (a.kn_counters) {
      if (c_bail) atomicAdd(a.kn_counters + 0, c_bail);
      if (c_few) atomicAdd(a.kn_counters + 1, c_few);
      if (c_full) atomicAdd(a.kn_counters + 2, c_full);
      if (c_rank) atomicAdd(a.kn_counters + 3, c_rank);
      if (c_out) atomicAdd(a.kn_counters + 13, c_out);
    }
  }
}

}  // namespace

int lane_list_cap(int k) {
  static const int extra = getenv("SPH_LANE_LEXTRA") ? atoi(getenv("SPH_LANE_LEXTRA")) : 16;
  return std::max(k + 1 + std::max(extra, 8), kBins + 1);  // the histogram rows alias the lists
}

// K up to 160 (measured at 64 and 128): beyond it the K-th's histogram bin holds more candidates than the
// in-bracket buffer and most lanes would fall back anyway
bool lane_supported(int k) { return k <= 160 && lane_smem_bytes(lane_list_cap(k)) * kLWarps <= 220 * 1024; }

void launch_lane(cudaStream_t s, const PassArgs &a, int lcap, float rscale, float exc, int max_stream, int num_sms,
                 const float *cal, float calq) {
  const int smem = kLWarps * lane_smem_bytes(lcap);
  const int ms = std::min(max_stream, 60000 - 4096);  // 16-bit run offsets (a step adds < 1024)
  int bps = 0;
  cudaFuncSetAttribute(k_lane, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_lane, kLWarps * 32, smem);
  k_lane<<<num_sms * std::max(bps, 1), kLWarps * 32, smem, s>>>(a, lcap, rscale, exc, ms, cal, calq);
}

}  // namespace sph
