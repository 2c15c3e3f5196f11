// One warp per target: neighbour search, exact K-th selection and density in
// a single persistent kernel (the default pass).
//
// For target i (reference compute_density_pass, density.py:286-413, with the
// todo loop replaced by a radius that only has to bound the K-th neighbour):
//   walk   the search tree with the target's own radius R: 32 pre-order nodes
//          per step (one per lane, skip pointers), every needed cell of the step
//          streamed at once, 32 candidates per step (one per lane);
//   count  each accepted candidate into a per-lane-column d2 histogram
//          (4 bins/octave) and append it to a shared-memory neighbour list;
//          once more than K are counted the radius shrinks to the upper edge
//          of the bin holding the K-th (adaptive shrink) and the list is
//          compacted to the new radius;
//   grow   fewer than K others within R: R grows and the walk restarts;
//   select the bin of the K-th gives a bracket [t_lo, t_hi]; exact fp64 d2
//          (octree.py:211-214 arithmetic) for list entries that may fall in
//          it, count below, rank inside -> d2_K (h = sqrt(d2_K), density.py:226-245);
//   sum    rho = sum over list entries within h of m_j W(r/h), self included
//          (density.py:160-171, 249-261; kernel.py:30-45), fp32 per pair or
//          fp64 term-for-term (dens64 / fp64 path).
// Targets the list cannot serve (overflow, bracket edge cases) keep their
// bracket in ST_NEED_BAND for the walking select/density passes (sph_pass.cu).
#include "sph_internal.cuh"
#include <cstdio>
#include <cstdlib>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef SPH_TARGET_WARPS
#define SPH_TARGET_WARPS 4
#endif
constexpr int kWarps = SPH_TARGET_WARPS;
#ifndef SPH_HIST_BPO_LOG2
#define SPH_HIST_BPO_LOG2 3
#endif
constexpr int kHistOctaves = 12;
constexpr int kBinBits = SPH_HIST_BPO_LOG2;           // log2 bins per octave of d2 / R^2
constexpr int kHistBase = (127 - kHistOctaves) << kBinBits;
constexpr int NB_HIST = (kHistOctaves << kBinBits) + 2;  // <= 128: four bins per lane
constexpr int kBinShift = 23 - kBinBits;
// one 32-bit counter per bin, updated with shared atomics; the region also
// holds the in-bracket doubles of the select
#ifndef SPH_HIST_REGION
#define SPH_HIST_REGION 1024
#endif
constexpr int kHistRegion = SPH_HIST_REGION;
constexpr int kInCapMain = kHistRegion / 8 < 256 ? kHistRegion / 8 : 256;  // in-bracket entries (alias the histogram)
constexpr int kInCapCollect = kHistRegion / 8;  // the collect instance has no histogram to keep
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard (as sph_pass.cu)
constexpr double kEpsD = 9.5367431640625e-07;
constexpr unsigned kNaNf = 0x7fc00000u;

struct alignas(32) D4 { double x, y, z, m; };
template <bool F32> struct Pos;
template <> struct Pos<true> { using T = float4; };
template <> struct Pos<false> { using T = D4; };

#ifndef SPH_TARGET_MINB
#define SPH_TARGET_MINB 7
#endif
#ifndef SPH_STACK
#define SPH_STACK 256
#endif
constexpr int kStack = SPH_STACK;  // traversal stack (node ids) per warp

__host__ __device__ constexpr int warp_smem_bytes(int cap) {
  return (32 + kHistRegion + cap * 8 + 2 * 32 * 4 + kStack * 4 + 15) & ~15;
}


__device__ __forceinline__ int hist_bin(float x) {  // x = d2 / R^2
  return min(max((__float_as_int(x) >> kBinShift) - kHistBase + 1, 0), NB_HIST - 1);
}

// COLLECT: second instance for the targets whose list overflowed in the main
// kernel: one walk with the radius of the bracket top t_hi, list only
template <bool F32, bool COLLECT>
__global__ void __launch_bounds__(kWarps * 32, SPH_TARGET_MINB) k_target(const PassArgs a, int cap, int *fallbacks) {
  using PT = typename Pos<F32>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float4 *simg = reinterpret_cast<float4 *>(smem_raw + wib * warp_smem_bytes(cap));  // image offsets of the shift
  unsigned char *wbase = smem_raw + wib * warp_smem_bytes(cap) + 32;
  unsigned *hist = reinterpret_cast<unsigned *>(wbase);
  double *inb = reinterpret_cast<double *>(wbase);  // after the histogram is read
  uint2 *list = reinterpret_cast<uint2 *>(wbase + kHistRegion);
  int *spfx = reinterpret_cast<int *>(wbase + kHistRegion + cap * 8);
  int *sbase = spfx + 32;
  int *stk = sbase + 32;
  const PT *__restrict__ pos = reinterpret_cast<const PT *>(a.pos);
  const float4 *__restrict__ nlo = a.tree.nlo;
  const float4 *__restrict__ nhi = a.tree.nhi;
  const int n_nodes = a.tree.n_nodes;
  const int n = a.n;
  const int K = a.k;
  const int center = a.periodic ? 13 : 0;
  const float boxf = (float)a.box;
  const bool f32sum = F32 && !a.dens64;
  const double norm = a.kernel_kind == 0 ? kWc6Norm : kM4Norm;
  const unsigned lt_mask = (1u << lane) - 1u;
  constexpr int kInCap = COLLECT ? kInCapCollect : kInCapMain;
  unsigned long long tests = 0, accepted = 0;
  int fb_over = 0, fb_bracket = 0, fb_stack = 0;

  const int count = a.list ? *a.list_count : a.static_count;
  // work in chunks of CH targets per atomic (the collect instance scans sparse
  // targets: whole warps of them)
  // a compacted list: one target per grab; the identity order: a.tchunk
  // consecutive targets (neighbours in space: their cell lists and candidates
  // stay in this SM's L1)
  const int CH = COLLECT ? (a.list ? 1 : 32) : max(1, min(a.tchunk, 32));
  // static_sched: warp w takes targets w, w + W, ... (no atomic; sorted
  // neighbours, whose costs are alike, land on different warps)
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarp = (gridDim.x * blockDim.x) >> 5;
  const bool stat = !COLLECT && a.static_sched;
  int snext = gwarp;
  unsigned pend = 0u;
  int cbase = 0;
  // the next chunk's index is requested while the current one is processed
  // (the atomic's latency hides behind a whole target)
  int t_pref = 0;
  if (!stat && lane == 0) t_pref = atomicAdd(a.work_counter, CH);
  for (;;) {
    if (!pend) {
      int t0 = 0;
      if (stat) {
        t0 = snext;
        snext += nwarp;
      } else {
        t0 = __shfl_sync(FULL, t_pref, 0);
        if (lane == 0 && t0 < count) t_pref = atomicAdd(a.work_counter, CH);
      }
      if (t0 >= count) break;
      cbase = t0;
      const int q = t0 + lane;
      bool want = false;
      if (lane < CH && q < count) {
        const int pq = a.list ? (int)a.list[q] : q;
        if constexpr (COLLECT) want = a.state[pq] == ST_NEED_BAND && a.ncount[pq] == 0x7fffffff;
        else want = a.state[pq] == ST_NEED_HIST;
      }
      pend = __ballot_sync(FULL, want);
      if (!pend) continue;
    }
    const int ti = cbase + __ffs(pend) - 1;
    pend &= pend - 1u;
    const int p = a.list ? (int)a.list[ti] : ti;

    double tx, ty, tz;
    {
      const PT t = pos[p];
      tx = t.x; ty = t.y; tz = t.z;
    }
    const float fx = (float)tx, fy = (float)ty, fz = (float)tz;
    float R = a.radius[p];
    if (!(R > 0.f)) R = 1e-30f;
    const float slack0 = F32 ? 0.f : fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))) * 1.2e-7f;
    // squared gap from the image frame x_i - s*box to the root box (the
    // shifted walks are tested with it, one shift per lane)
    auto image_gap2 = [&](int sx, int sy, int sz) {
      const float4 l4 = nlo[0], h4 = nhi[0];
      const float qx = (float)(tx - sx * a.box), qy = (float)(ty - sy * a.box), qz = (float)(tz - sz * a.box);
      const float sl = boxf * 4.8e-7f;
      const float gx = fmaxf(fmaxf(l4.x - qx, qx - h4.x) - sl, 0.f);
      const float gy = fmaxf(fmaxf(l4.y - qy, qy - h4.y) - sl, 0.f);
      const float gz = fmaxf(fmaxf(l4.z - qz, qz - h4.z) - sl, 0.f);
      return (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps);
    };

    // collect instance: phase 0 lists the bracket (counting what lies below it),
    // phase 1 lists everything within the selected h for the density; phase 2
    // (a bracket too crowded to list) counts it in 32 sub-bins and narrows it
    int cphase = 0, nrefine = 0;
    double d2k_c = 0.0, ctl = 0.0, cth = 0.0;
    if constexpr (COLLECT) {
      ctl = a.t_lo[p];
      cth = a.t_hi[p];
    }
    for (;;) {  // grow loop
      const float hR2 = COLLECT ? (float)(__double2float_ru((cphase == 1 ? d2k_c : cth) * (1.0 + kEpsD)) + 1e-37f)
                                : R * R;
      const float h_inv = 1.0f / hR2;
      float h_r2 = hR2;  // current acceptance radius^2 (shrinks)
      if (!COLLECT || cphase == 2)
        for (int bb = lane; bb < NB_HIST; bb += 32) hist[bb] = 0u;
      int seen = 0, seen_shrunk = 0;  // warp-uniform: counted candidates (self included)
      int ne = 0;                     // warp-uniform: list entries
      bool over = false;              // list overflowed: no list-based select
      bool stack_over = false;        // traversal stack overflowed: bundle passes instead
      int cand = 0;                   // candidates streamed (bounds the 16-bit histogram counters)
      __syncwarp();

      // adaptive shrink from the column histogram; compacts the list
      // first bin whose cumulative count (bin 0 less `sub`) exceeds T; four
      // consecutive bins per lane, one scan (NB_HIST when none)
      auto first_bin_over = [&](int T, unsigned sub) -> int {
        unsigned c[4], sum = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int b = 4 * lane + u;
          c[u] = b < NB_HIST ? hist[b] : 0u;
          if (b == 0) c[u] -= sub;
          sum += c[u];
        }
        unsigned incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += v;
        }
        const unsigned excl = incl - sum;
        const bool here = (int)incl > T && (int)excl <= T;
        int bin = NB_HIST;
        if (here) {
          unsigned cum = excl;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cum += c[u];
            if ((int)cum > T && bin == NB_HIST) bin = 4 * lane + u;
          }
        }
        const unsigned hm = __ballot_sync(FULL, here);
        return hm ? __shfl_sync(FULL, bin, __ffs(hm) - 1) : NB_HIST;
      };
      // adaptive shrink from the histogram (K others + self counted); compacts the list
      auto shrink = [&]() {
        const int bb = first_bin_over(K, 0u);
        if (bb < NB_HIST - 1) {
          const float edge = __int_as_float((kHistBase + bb) << kBinShift) * hR2 * (1.0f + 4.0f * kEps);
          if (edge < h_r2) {
            h_r2 = edge;
            if (!over && ne > K) {
              // in-place warp compaction of the list to the new radius
              int w = 0;
              for (int i0 = 0; i0 < ne; i0 += 32) {
                const int i = i0 + lane;
                uint2 e = make_uint2(0u, kNaNf);
                if (i < ne) e = list[i];
                const bool keep = i < ne && __uint_as_float(e.y) <= edge;
                const unsigned km = __ballot_sync(FULL, keep);
                __syncwarp();
                if (keep) list[w + __popc(km & lt_mask)] = e;
                w += __popc(km);
                __syncwarp();
              }
              ne = w;
            }
          }
        }
        seen_shrunk = seen;
      };

      // periodic images: shifts s in {0,-1,+1}^3, the unshifted one first (its
      // neighbours shrink the radius early); a shift is searched only if the
      // root box, seen from x_i - s*box, comes within the current radius
      double tl = 0.0, th = 0.0;
      float lo_c = -1.f;  // collect: candidates below the bracket are counted, not listed
      int cbelow = 0;
      float rinv_c = 0.f;  // phase 2: sub-bins per unit fp32 d2
      if constexpr (COLLECT) {
        tl = ctl;
        th = cth;
        lo_c = __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f;
        const float hi_c = __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f;
        rinv_c = 32.0f / fmaxf(hi_c - lo_c, 1e-37f);
      }
      bool grow = false, done_unreach = false;
      for (int pass = 0; pass < 1; ++pass) {
      // unshifted image first; then the shifted images whose root-box gap (one
      // shift per lane, tested once after the unshifted walk) is within the radius
      unsigned rest = 0u;
      for (int it = 0;; ++it) {
        int sidx = center;
        if (it > 0) {
          if (it == 1) {
            bool want = false;
            if (a.periodic && lane < 27 && lane != 13)
              want = image_gap2(lane / 9 - 1, (lane / 3) % 3 - 1, lane % 3 - 1) <= h_r2;
            rest = __ballot_sync(FULL, want);
          }
          if (!rest) break;
          sidx = __ffs(rest) - 1;
          rest &= rest - 1u;
        }
        const int sx = a.periodic ? sidx / 9 - 1 : 0, sy = a.periodic ? (sidx / 3) % 3 - 1 : 0,
                  sz = a.periodic ? sidx % 3 - 1 : 0;
        if (it > 0 && image_gap2(sx, sy, sz) > h_r2) continue;  // re-check with the radius as it is now
        const bool shifted = (sx | sy | sz) != 0;
        const double dsx = sx * a.box, dsy = sy * a.box, dsz = sz * a.box;
        // the target in the tree frame of this shift (x_i - s*box), plus slack
        const float pqx = sx ? (float)(tx - dsx) : fx, pqy = sy ? (float)(ty - dsy) : fy,
                    pqz = sz ? (float)(tz - dsz) : fz;
        const float pslack = shifted ? boxf * 4.8e-7f : slack0;
        if (lane == 0) {
          // fp32 image arithmetic with the box side in two words, box = hi + lo
          // (C3's side is no fp32 value): for a -1 shift the candidate moves by
          // -hi (exact: Sterbenz, the hit candidates sit within R of the face)
          // and the target takes the lo word, x_i + lo; for a +1 shift the
          // target moves, (x_i - hi) - lo; unshifted, x_i - 0.  Each adds one
          // rounding at the scale of the target's distance to the face (< R),
          // so the fp32 d2 stays within 2 (R / d) 2^-24 of the exact
          // image-augmented value: inside the 2^-20 guard band of the exact
          // recheck.  (Written branch-free: the hot loop's register allocation
          // is sensitive to this block.)
          const float bl = a.box_lo;
          simg[0] = make_float4(sx < 0 ? -boxf : 0.f, sy < 0 ? -boxf : 0.f, sz < 0 ? -boxf : 0.f, 0.f);
          simg[1] = make_float4((sx > 0 ? fx - boxf : fx) - (float)sx * bl, (sy > 0 ? fy - boxf : fy) - (float)sy * bl,
                                (sz > 0 ? fz - boxf : fz) - (float)sz * bl, 0.f);
        }
        __syncwarp();

        // ---- warp traversal: pop up to 32 nodes (one per lane), test, push the
        // children of hit internal nodes (child lists), stream the hit cells ----
        // unshifted: start at the lowest ancestor of the target's cell whose box
        // holds the whole search sphere (no cell outside it can be within R)
        // a neighbour-cell list of the target's own cell (built for the radius
        // its seeds imply) replaces the unshifted traversal when it covers R
        int lbase = -1, llen = 0, lnear = 0, lfar_off = 0;
        if (!shifted && a.clist) {
          const int ci = a.cellidx[a.tree.cellof[p]];
          if (ci >= 0) {
            const int len = a.clen[ci];
            const float cr2 = a.crad2[ci];
            if (len >= 0 && h_r2 <= cr2) {
              lbase = ci * a.clcap;
              llen = len;
              lnear = a.cnear[ci];
              lfar_off = a.clcap - len;  // far records sit at the back of the list
              // far records lie beyond near_frac * D of the cell box: skipped
              // when the radius is below that
              if (h_r2 <= a.near_frac2 * cr2 * (1.0f - 16.0f * kEps)) llen = lnear;
            }
          }
        }
        int start = a.tree.root_start;
        if (!shifted && lbase < 0) {
          const int4 an = a.tree.anc4[a.tree.cellof[p]];
          const float rr = sqrtf(h_r2) * (1.0f + 8.0f * kEps) + pslack;
          const int my_anc = lane == 0 ? an.x : lane == 1 ? an.y : lane == 2 ? an.z : lane == 3 ? an.w : -1;
          bool holds = false;
          if (my_anc >= 0) {
            const float4 l4 = nlo[my_anc], h4 = nhi[my_anc];
            holds = l4.x <= pqx - rr && pqx + rr <= h4.x && l4.y <= pqy - rr && pqy + rr <= h4.y &&
                    l4.z <= pqz - rr && pqz + rr <= h4.z;
          }
          const unsigned hm = __ballot_sync(FULL, holds);
          if (hm) start = __shfl_sync(FULL, my_anc, __ffs(hm) - 1);
        }
        // the stack holds hit internal nodes; a step expands up to 4 of them,
        // one child record per lane (8 slots each: box + node id or cell range)
        if (lane == 0) stk[0] = start;
        int top = lbase < 0 ? 1 : 0, li = 0;
        __syncwarp();
        while (lbase >= 0 ? li < llen : top > 0) {
          const float4 *rec = nullptr;
          if (lbase >= 0) {  // 32 listed cells per step
            if (li + lane < llen) {
              const int e = li + lane;
              rec = a.tree.crec + 2 * (size_t)a.clist[(size_t)lbase + (e < lnear ? e : e + lfar_off)];
            }
            li += 32;
          } else {
            const int np = min(top, 4);
            top -= np;
            const int pi = lane >> 3;
            const int par = pi < np ? stk[top + pi] : -1;
            __syncwarp();
            if (par >= 0) rec = a.tree.crec + 16 * (size_t)par + 2 * (lane & 7);
          }
          bool hit = false, is_cell = false;
          int node = -1, my_start = 0, my_end = 0;
          if (rec) {
            const float4 l4 = rec[0], h4 = rec[1];
            const int code = __float_as_int(l4.w);
            is_cell = code < 0;
            node = code;
            const float gx = fmaxf(fmaxf(l4.x - pqx, pqx - h4.x) - pslack, 0.f);
            const float gy = fmaxf(fmaxf(l4.y - pqy, pqy - h4.y) - pslack, 0.f);
            const float gz = fmaxf(fmaxf(l4.z - pqz, pqz - h4.z) - pslack, 0.f);
            hit = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= h_r2;
            if (hit && is_cell) {
              my_start = ~code;
              my_end = __float_as_int(h4.w);
            }
          }
          const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
          if (top + __popc(pm) > kStack) { stack_over = true; break; }
          if (hit && !is_cell) stk[top + __popc(pm & lt_mask)] = node;
          top += __popc(pm);
          const bool need = hit && is_cell;
          const int len = need ? my_end - my_start : 0;
          int incl = len;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
          }
          const int total = __shfl_sync(FULL, incl, 31);
          __syncwarp();
          if (total == 0) continue;
          cand += total;
          tests += (unsigned)total;
          if (cand > (1 << 20)) { stack_over = true; break; }  // 16-bit counters: bundle passes
          // needed cells compacted (all ranges non-empty, so their stream ends
          // are distinct): lane r holds the end of cell r in the stream
          const unsigned nm = __ballot_sync(FULL, need);
          if (need) {
            const int ci = __popc(nm & lt_mask);
            spfx[ci] = incl;
            sbase[ci] = my_start - (incl - len);
          }
          __syncwarp();
          const int cend = lane < __popc(nm) ? spfx[lane] : 0x7fffffff;

          // ---- stream the step's candidates, 32 per chunk ----
          for (int c0 = 0; c0 < total; c0 += 32) {
            const int s = c0 + lane;
            bool in = false;
            int j = 0;
            float af = 0.f;
            // owner of stream slot s = #{cells whose end <= s}: the cells ending
            // before the chunk plus a bit mask of the ends inside it
            const unsigned ev = (cend > c0 && cend <= c0 + 31) ? 1u << (cend - c0 - 1) : 0u;
            const unsigned emask = __reduce_or_sync(FULL, ev);
            const int owner = __popc(__ballot_sync(FULL, cend <= c0)) + __popc(emask & lt_mask);
            if (s < total) {
              j = sbase[owner] + s;
              const PT c = pos[j];
              if constexpr (F32) {
                // unshifted: cs = 0 and tf = the target, so this is c.x - fx exactly
                const float4 cs = simg[0], tf = simg[1];
                const float dx = (c.x + cs.x) - tf.x, dy = (c.y + cs.y) - tf.y, dz = (c.z + cs.z) - tf.z;
                af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                in = af <= h_r2;
              } else {
                double cx = c.x, cy = c.y, cz = c.z;
                if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
                const double ad = exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
                in = ad <= (double)h_r2;
                af = (float)ad;
              }
              if (!COLLECT && in) atomicAdd(&hist[hist_bin(af * h_inv)], 1u);
            }
            bool lst = in;
            if constexpr (COLLECT) {
              if (cphase == 0 && lst && af < lo_c && !(j == p && sidx == center)) {
                ++cbelow;
                lst = false;
              }
              if (cphase == 2) {
                if (in && !(j == p && sidx == center)) {
                  if (af < lo_c) ++cbelow;
                  else atomicAdd(&hist[min(max((int)((af - lo_c) * rinv_c), 0), 31)], 1u);
                }
                lst = false;
              }
            }
            int nin = __popc(__ballot_sync(FULL, in));
            seen += nin;
            if (!over && ne + nin > cap) {
              // full list: shrink first (the histogram already holds this step)
              if (!COLLECT && seen > K + 1) {
                shrink();
                if (lst && !(af <= h_r2)) lst = false;  // counted, beyond the new radius
              }
              if (ne + __popc(__ballot_sync(FULL, lst)) > cap) over = true;
            }
            if (!over) {
              const unsigned lm = __ballot_sync(FULL, lst);
              if (lst) list[ne + __popc(lm & lt_mask)] = make_uint2((unsigned)j | ((unsigned)sidx << 27), __float_as_uint(af));
              ne += __popc(lm);
            }
          }
          __syncwarp();
          if (!COLLECT && seen > K + 1 && seen - seen_shrunk >= (K >> a.tshrink)) shrink();
        }
        if (stack_over) break;
      }
      __syncwarp();
      if (a.dbg && fallbacks && lane == 0) atomicAdd(fallbacks + 3, 1);  // walks (debug)
      if (stack_over || COLLECT) break;

      // ---- counted enough? ----
      const int others = seen - 1;  // the target itself (d2 = 0)
      if (others < K) {
        if (R >= a.rmax) {
          if (lane == 0) {
            a.state[p] = ST_UNREACHABLE;
            a.d2k[p] = INFINITY;
          }
          done_unreach = true;
        } else {
          float f = others > 0 ? cbrtf((float)(K + 8) / (float)others) * 1.15f : 2.f;
          f = fminf(fmaxf(f, 1.26f), 2.5f);
          R = fminf(R * f, a.rmax);
          grow = true;
        }
        break;
      }

      // ---- bracket of the K-th from the histogram ----
      {
        const int bb0 = first_bin_over(K - 1, 1u);  // cumulative others >= K
        const int bb = bb0 < NB_HIST ? bb0 : NB_HIST - 1;
        const double R2d = (double)hR2;
        if (bb == 0) {
          tl = 0.0;
          th = (double)__int_as_float(kHistBase << kBinShift) * R2d * (1.0 + 8.0 * kEpsD);
        } else if (bb >= NB_HIST - 1) {
          tl = R2d * (1.0 - 8.0 * kEpsD);
          th = R2d * (1.0 + 8.0 * kEpsD);
        } else {
          tl = (double)__int_as_float((kHistBase + bb - 1) << kBinShift) * R2d * (1.0 - 8.0 * kEpsD);
          th = (double)__int_as_float((kHistBase + bb) << kBinShift) * R2d * (1.0 + 8.0 * kEpsD);
        }
        // the list holds every candidate with d2 <= h_r2 (2^-20 guard)
        th = fmin(th, (double)h_r2 * (1.0 - 4.0 * kEpsD));
        if (th < tl) th = tl;
      }
      __syncwarp();
      }  // pass loop
      if (stack_over) { ++fb_stack; break; }  // the bundle passes take it (state unchanged)
      if (done_unreach) break;
      if (grow) continue;

      auto fallback = [&]() {
        if (lane == 0) {
          a.t_lo[p] = tl;
          a.t_hi[p] = th;
          a.radius[p] = R;
          a.state[p] = ST_NEED_BAND;
          // no usable list: the collect instance next, then the walking select
          if (a.ncount) a.ncount[p] = COLLECT ? 0x7ffffffe : 0x7fffffff;
          if (!COLLECT && a.fb_list) a.fb_list[atomicAdd(a.fb_count, 1)] = (uint32_t)p;
        }
      };
      if constexpr (COLLECT) {
        if (cphase == 2) {
          // the sub-bin holding the K-th (fp32 d2; the exact select re-checks)
          const int below_c = (int)__reduce_add_sync(FULL, (unsigned)cbelow);
          const int rr = K - below_c;
          const unsigned cnt = hist[lane];
          unsigned incl = cnt;
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
          }
          const unsigned hm = __ballot_sync(FULL, rr >= 1 && (int)incl >= rr);
          if (!hm || nrefine >= 6) { ++fb_over; fallback(); break; }
          const int sb = __ffs(hm) - 1;
          const double w = 1.0 / (double)rinv_c;
          ctl = fmax(ctl, ((double)lo_c + sb * w) * (1.0 - 4.0 * kEpsD));
          cth = fmin(cth, ((double)lo_c + (sb + 1) * w) * (1.0 + 4.0 * kEpsD));
          if (!(cth > ctl)) cth = ctl;
          cphase = 0;
          ++nrefine;
          continue;
        }
        if (over && cphase == 0 && nrefine < 6) {  // too crowded to list: narrow it first
          cphase = 2;
          continue;
        }
      }
      if (over) { ++fb_over; fallback(); break; }

      double d2k;
      auto image_d2 = [&](const PT &c, int sidx) {
        double cx = c.x, cy = c.y, cz = c.z;
        if (a.periodic && sidx != 13) {
          const int sx = sidx / 9 - 1, sy = (sidx / 3) % 3 - 1, sz = sidx % 3 - 1;
          cx = __dadd_rn(cx, sx * a.box); cy = __dadd_rn(cy, sy * a.box); cz = __dadd_rn(cz, sz * a.box);
        }
        return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
      };
      if (COLLECT && cphase == 1) {
        d2k = d2k_c;
      } else {
        // ---- exact count below the bracket, collect the bracket ----
        const float lo_f = __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f;
        const float hi_f = __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f;
        int below = cbelow, n_in = 0;
        for (int i0 = 0; i0 < ne; i0 += 32) {
          const int i = i0 + lane;
          bool inb_ = false;
          double e = 0.0;
          if (i < ne) {
            const uint2 le = list[i];
            const float af = __uint_as_float(le.y);
            const int j = (int)(le.x & ((1u << 27) - 1u));
            const int sidx = (int)(le.x >> 27);
            if (!(j == p && sidx == center)) {
              if (af < lo_f) {
                ++below;
              } else if (af <= hi_f) {
                e = image_d2(pos[j], sidx);
                if (e < tl) ++below;
                else if (e <= th) inb_ = true;
              }
            }
          }
          const unsigned bm = __ballot_sync(FULL, inb_);
          if (inb_ && n_in + __popc(bm & lt_mask) < kInCap) inb[n_in + __popc(bm & lt_mask)] = e;  // see kInCap
          n_in += __popc(bm);
        }
        __syncwarp();
        below = (int)__reduce_add_sync(FULL, (unsigned)below);
        const int r = K - below;  // 1-based rank of the K-th inside the bracket
        if (!COLLECT && n_in <= kInCap && r > n_in && R < a.rmax) {
          // the K-th lies above the (clipped) list radius, at the very edge of
          // R: search again with a slightly larger radius
          R = fminf(R * 1.26f, a.rmax);
          continue;
        }
        if constexpr (COLLECT) {
          if (n_in > kInCap && nrefine < 6) {  // too many in the bracket to rank: narrow it
            cphase = 2;
            continue;
          }
        }
        if (n_in > kInCap || r < 1 || r > n_in) {
          if (lane == 0 && a.dbg && fallbacks && atomicAdd(fallbacks + 2, 1) < 10)
            printf("[target miss] p=%d ne=%d seen=%d K=%d below=%d n_in=%d tl=%.9g th=%.9g h_r2=%.9g R2=%.9g\n", p, ne,
                   seen, K, below, n_in, tl, th, (double)h_r2, (double)hR2);
          ++fb_bracket;
          fallback();
          break;
        }

        // ---- the r-th smallest of the bracket ----
        double v = INFINITY;
        for (int i = lane; i < n_in; i += 32) {
          const double ei = inb[i];
          int less = 0, eq = 0;
          for (int jj = 0; jj < n_in; ++jj) {
            const double ej = inb[jj];
            less += ej < ei;
            eq += ej == ei;
          }
          if (less < r && r <= less + eq) v = ei;
        }
        for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
        d2k = v;

        if constexpr (COLLECT) {
          if (d2k > 0.0) {  // phase 1: everything within h, for the density sum
            d2k_c = d2k;
            cphase = 1;
            continue;
          }
        }
      }

      // ---- density over the list entries within h ----
      double rho = 0.0;
      if (d2k > 0.0) {
        double accd = 0.0;
        float accf = 0.f;
        const double hh = __dsqrt_rn(d2k);
        const double norm_h3 = __ddiv_rn(norm, __dmul_rn(__dmul_rn(hh, hh), hh));
        const float d2k_f = __double2float_ru(d2k * (1.0 + kEpsD));
        const float inv_h = (float)(1.0 / hh);
        for (int i = lane; i < ne; i += 32) {
          const uint2 le = list[i];
          const float af = __uint_as_float(le.y);
          if (!(af < d2k_f)) continue;
          ++accepted;
          const int j = (int)(le.x & ((1u << 27) - 1u));
          const PT c = pos[j];
          if (f32sum) {
            if constexpr (F32) {
              const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
              const float q = rr * inv_h;
              const float wv = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
              if (q < 1.f) accf = fmaf(c.w, wv, accf);
            }
          } else {
            const double e = image_d2(c, (int)(le.x >> 27));
            if (e < d2k) {
              const double r_ = __dsqrt_rn(e);
              double wv;
              if (a.kernel_kind == 0) {
                wv = wc6_lowered(r_, hh, norm_h3);
              } else {
                const double q = __ddiv_rn(r_, hh);
                wv = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
              }
              double mj;
              if constexpr (F32) mj = a.mass64[j]; else mj = c.m;
              accd = __dadd_rn(accd, __dmul_rn(mj, wv));
            }
          }
        }
        for (int o = 16; o; o >>= 1) {
          accd += __shfl_xor_sync(FULL, accd, o);
          accf += __shfl_xor_sync(FULL, accf, o);
        }
        rho = f32sum ? __dmul_rn(norm_h3, (double)accf) : accd;
      }
      if (lane == 0) {
        a.d2k[p] = d2k;
        a.rho[p] = rho;
        a.radius[p] = R;
        a.state[p] = ST_FINAL;
      }
      break;
    }
  }
  // statistics
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
    if (fallbacks) {
      if (fb_over) atomicAdd(fallbacks, fb_over);
      if (fb_bracket) atomicAdd(fallbacks + 1, fb_bracket);
      if (fb_stack) atomicAdd(fallbacks + 4, fb_stack);
    }
  }
}

// Child records for the per-target traversal: for every internal node k (and
// a virtual node V = n_nodes whose only child is the root) 8 slots of
// {child box lo, code} {child box hi, end}: code >= 0 is an internal child's
// node id, code < 0 a cell holding particles [~code, end); absent slots have an
// empty box (never hit).  Also the parent of each node and the cell of each
// sorted particle.
__device__ __forceinline__ void child_record(const float4 *__restrict__ nlo, const float4 *__restrict__ nhi,
                                             int n_nodes, int n, int c, float4 &lo, float4 &hi) {
  lo = nlo[c];
  hi = nhi[c];
  const bool cell = __float_as_int(lo.w) == c + 1;
  const int start = __float_as_int(hi.w);
  const int end = c + 1 < n_nodes ? __float_as_int(nhi[c + 1].w) : n;
  lo.w = __int_as_float(cell ? ~start : c);
  hi.w = __int_as_float(cell ? end : 0);
}

__global__ void k_kids(const float4 *__restrict__ nlo, const float4 *__restrict__ nhi, int n_nodes, int n,
                       float4 *__restrict__ crec, int *__restrict__ parent, int *__restrict__ cellof) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > n_nodes) return;
  const float4 empty_lo = make_float4(INFINITY, INFINITY, INFINITY, __int_as_float(INT_MIN));
  const float4 empty_hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
  float4 *rec = crec + 16 * (size_t)k;
  int i = 0;
  if (k == n_nodes) {  // virtual node above the root
    float4 lo, hi;
    child_record(nlo, nhi, n_nodes, n, 0, lo, hi);
    rec[0] = lo;
    rec[1] = hi;
    i = 1;
  } else {
    if (k == 0) parent[0] = -1;
    const int skip = __float_as_int(nlo[k].w);
    if (skip != k + 1) {
      int c = k + 1;
      while (c < skip && i < 8) {
        float4 lo, hi;
        child_record(nlo, nhi, n_nodes, n, c, lo, hi);
        rec[2 * i] = lo;
        rec[2 * i + 1] = hi;
        ++i;
        parent[c] = k;
        c = __float_as_int(nlo[c].w);
      }
    } else {
      const int s0 = __float_as_int(nhi[k].w);
      const int e0 = k + 1 < n_nodes ? __float_as_int(nhi[k + 1].w) : n;
      for (int j = s0; j < e0; ++j) cellof[j] = k;
    }
  }
  for (; i < 8; ++i) {
    rec[2 * i] = empty_lo;
    rec[2 * i + 1] = empty_hi;
  }
}

// the first four ancestors of every node (-1 above the root)
__global__ void k_anc(const int *__restrict__ parent, int n_nodes, int4 *__restrict__ anc4) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_nodes) return;
  const int a1 = parent[k];
  const int a2 = a1 >= 0 ? parent[a1] : -1;
  const int a3 = a2 >= 0 ? parent[a2] : -1;
  const int a4 = a3 >= 0 ? parent[a3] : -1;
  anc4[k] = make_int4(a1, a2, a3, a4);
}

// Initial search radius per cell (the per-target path): density estimates
// from the smallest ancestors (cell included) holding >= K/2 and >= 2K
// particles, the smaller of the two times r0_scale, capped by sqrt(3) x the
// side of the smallest ancestor holding >= K+1 (it surely contains K others).
__global__ void k_r0(const float4 *__restrict__ nlo, const float4 *__restrict__ nhi, const int *__restrict__ nsize,
                     const int *__restrict__ parent, int n_nodes, int n, int k, float r0_scale, float rmax,
                     float root_side, float *__restrict__ r0) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_nodes || __float_as_int(nlo[c].w) != c + 1) return;
  const int a0 = parent[c];
  double side = a0 >= 0 ? 0.5 * ((double)nhi[a0].x - (double)nlo[a0].x) : root_side;  // the cell's cube
  int cnt = nsize[c];
  int a = a0;
  double est_a = 0.0, est_b = 0.0, bound = 0.0;
  for (;;) {
    const double est = side * cbrt(3.0 * k / (4.0 * 3.14159265358979323846 * (double)max(cnt, 1)));
    const bool top = a < 0;
    if (est_a == 0.0 && (cnt >= (k + 1) / 2 || top)) est_a = est;
    if (bound == 0.0 && (cnt >= k + 1 || top)) bound = 1.7320508075688772 * side * (1.0 + 1e-6);
    if (cnt >= 2 * k || top) { est_b = est; break; }
    cnt = nsize[a];
    side = (double)nhi[a].x - (double)nlo[a].x;  // the ancestor's (padded) cube
    a = parent[a];
  }
  float R = (float)fmin(r0_scale * fmin(est_a, est_b), bound);
  if (!(R > 0.f)) R = rmax;
  R = fminf(R, rmax);
  const int s0 = __float_as_int(nhi[c].w);
  const int e0 = c + 1 < n_nodes ? __float_as_int(nhi[c + 1].w) : n;
  for (int q = s0; q < e0; ++q) r0[q] = R;
}

// Neighbour-cell lists (per-target path, after the seeds): for every cell with
// targets still to search, D = the largest initial radius of its targets and
// the list of every cell whose box lies within D of its box (the child
// records of those cells).  Any particle within D of a target of the cell is
// in a listed cell.  len = -1: no list (no targets, or more than cap cells).
__global__ void __launch_bounds__(128) k_cell_lists(const float4 *__restrict__ nlo, const float4 *__restrict__ nhi,
                                                    const float4 *__restrict__ crec, const int *__restrict__ cellnode,
                                                    const int *__restrict__ ncells, const uint8_t *__restrict__ state,
                                                    const float *__restrict__ r0, const int4 *__restrict__ anc4,
                                                    int n_nodes, int n, int root_start, int cap,
                                                    unsigned *__restrict__ clist, int *__restrict__ clen,
                                                    float *__restrict__ crad2, int *__restrict__ cnear,
                                                    float near_frac, float d_pct) {
  __shared__ int s_stk[4][kStack];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int *stk = s_stk[wib];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int nc = *ncells;
  const unsigned lt = (1u << lane) - 1u;
  for (int ci = gw; ci < nc; ci += nw) {
    const int c = cellnode[ci];
    const float4 cl = nlo[c], chh = nhi[c];
    const int s0 = __float_as_int(chh.w);
    const int e0 = c + 1 < n_nodes ? __float_as_int(nhi[c + 1].w) : n;
    // D = the d_pct quantile of the cell's target radii (cells hold <= 32
    // particles: one per lane); targets above it walk the tree instead
    float D = 0.f;
    {
      const int q = s0 + lane;
      const float Rq = (q < e0 && lane < 32 && state[q] == ST_NEED_HIST) ? r0[q] : 0.f;
      const unsigned tm = __ballot_sync(FULL, Rq > 0.f);
      const int cnt = __popc(tm);
      float mx = Rq;
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
      D = mx;
      if (cnt > 0 && d_pct < 1.0f && e0 - s0 <= 32) {
        // rank of each lane's radius among the targets (ties by lane)
        int rank = 0;
        for (int l = 0; l < 32; ++l) {
          const float v = __shfl_sync(FULL, Rq, l);
          rank += (v > 0.f) && (v < Rq || (v == Rq && l < lane));
        }
        const int want = min(cnt - 1, (int)ceilf(d_pct * (float)(cnt - 1)));
        const unsigned pm = __ballot_sync(FULL, Rq > 0.f && rank == want);
        if (pm) D = __shfl_sync(FULL, Rq, __ffs(pm) - 1);
      }
    }
    if (!(D > 0.f)) {
      if (lane == 0) clen[ci] = -1;
      continue;
    }
    const float D2 = D * D * (1.0f + 16.0f * kEps);
    // start at the lowest of the first four ancestors whose box holds the
    // cell box grown by D (nothing outside it is within D)
    int start = root_start;
    {
      const int4 an = anc4[c];
      const float Dm = D * (1.0f + 8.0f * kEps);
      const int my_anc = lane == 0 ? an.x : lane == 1 ? an.y : lane == 2 ? an.z : lane == 3 ? an.w : -1;
      bool holds = false;
      if (my_anc >= 0) {
        const float4 l4 = nlo[my_anc], h4 = nhi[my_anc];
        holds = l4.x <= cl.x - Dm && chh.x + Dm <= h4.x && l4.y <= cl.y - Dm && chh.y + Dm <= h4.y &&
                l4.z <= cl.z - Dm && chh.z + Dm <= h4.z;
      }
      const unsigned hm = __ballot_sync(FULL, holds);
      if (hm) start = __shfl_sync(FULL, my_anc, __ffs(hm) - 1);
    }
    // records whose gap to the cell box exceeds near_frac * D go to the back
    // of the list: targets whose radius is below that skip them entirely
    const float N2 = near_frac * near_frac * D * D;
    int len = 0, nnear = 0, nfar = 0;
    if (lane == 0) stk[0] = start;
    int top = 1;
    bool over = false;
    __syncwarp();
    while (top > 0) {
      const int np = min(top, 4);
      top -= np;
      const int pi = lane >> 3;
      const int par = pi < np ? stk[top + pi] : -1;
      __syncwarp();
      bool hit = false, is_cell = false;
      float g2 = 0.f;
      float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
      if (par >= 0) {
        const float4 *rec = crec + 16 * (size_t)par + 2 * (lane & 7);
        l4 = rec[0];
        h4 = rec[1];
        is_cell = __float_as_int(l4.w) < 0;
        const float gx = fmaxf(fmaxf(l4.x - chh.x, cl.x - h4.x), 0.f);
        const float gy = fmaxf(fmaxf(l4.y - chh.y, cl.y - h4.y), 0.f);
        const float gz = fmaxf(fmaxf(l4.z - chh.z, cl.z - h4.z), 0.f);
        g2 = gx * gx + gy * gy + gz * gz;
        hit = g2 * (1.0f - 4.0f * kEps) <= D2;
      }
      const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
      if (top + __popc(pm) > kStack) { over = true; break; }
      if (hit && !is_cell) stk[top + __popc(pm & lt)] = __float_as_int(l4.w);
      top += __popc(pm);
      const bool far = g2 * (1.0f - 4.0f * kEps) > N2;
      const unsigned cm = __ballot_sync(FULL, hit && is_cell && !far);
      const unsigned fm = __ballot_sync(FULL, hit && is_cell && far);
      if (len + __popc(cm) + __popc(fm) > cap) { over = true; break; }
      if (hit && is_cell) {
        // the list holds the child-record index (parent * 8 + slot): 4 bytes
        // per entry instead of the 32-byte record, so lists and records stay in L2
        const int slot = far ? cap - 1 - (nfar + __popc(fm & lt)) : nnear + __popc(cm & lt);
        clist[(size_t)ci * cap + slot] = (unsigned)par * 8u + (unsigned)(lane & 7);
      }
      nnear += __popc(cm);
      nfar += __popc(fm);
      len = nnear + nfar;
      __syncwarp();
    }
    if (lane == 0) {
      clen[ci] = over ? -1 : len;
      cnear[ci] = nnear;
      crad2[ci] = D * D;
    }
  }
}

// cell index of every node (-1 for internal nodes) and the node of every cell
__global__ void k_cell_index(const float4 *__restrict__ nlo, int n_nodes, int *__restrict__ cellidx,
                             int *__restrict__ cellnode, int *__restrict__ ncells) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_nodes) return;
  if (__float_as_int(nlo[k].w) == k + 1) {
    const int ci = atomicAdd(ncells, 1);
    cellidx[k] = ci;
    cellnode[ci] = k;
  } else {
    cellidx[k] = -1;
  }
}

// the same with the node count on the device (grid over an upper bound)
__global__ void k_cell_index_dev(const float4 *__restrict__ nlo, const int *__restrict__ n_nodes_dev,
                                 int *__restrict__ cellidx, int *__restrict__ cellnode, int *__restrict__ ncells) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= *n_nodes_dev) return;
  if (__float_as_int(nlo[k].w) == k + 1) {
    const int ci = atomicAdd(ncells, 1);
    cellidx[k] = ci;
    cellnode[ci] = k;
  } else {
    cellidx[k] = -1;
  }
}

}  // namespace

void launch_cell_index_dev(cudaStream_t s, const float4 *nlo, const int *n_nodes_dev, int max_nodes, int *cellidx,
                           int *cellnode, int *ncells) {
  k_cell_index_dev<<<(max_nodes + 255) / 256, 256, 0, s>>>(nlo, n_nodes_dev, cellidx, cellnode, ncells);
}

void launch_cell_index(cudaStream_t s, const float4 *nlo, int n_nodes, int *cellidx, int *cellnode, int *ncells) {
  k_cell_index<<<(n_nodes + 255) / 256, 256, 0, s>>>(nlo, n_nodes, cellidx, cellnode, ncells);
}

void launch_cell_lists(cudaStream_t s, const PassArgs &a, const int *cellnode, const int *ncells, int cap,
                       unsigned *clist, int *clen, float *crad2, int *cnear, float near_frac, float d_pct,
                       int num_sms, int ncell_host) {
  // one warp per cell: each list is one latency-bound walk, so as many
  // walks in flight as the cells (more blocks than resident slots balance too)
  const int blocks = ncell_host > 0 ? (ncell_host + 3) / 4 : num_sms * 16;
  k_cell_lists<<<blocks, 128, 0, s>>>(a.tree.nlo, a.tree.nhi, a.tree.crec, cellnode, ncells, a.state, a.radius,
                                           a.tree.anc4, a.tree.n_nodes, a.n, a.tree.root_start, cap, clist, clen,
                                           crad2, cnear, near_frac, d_pct);
}

void launch_r0(cudaStream_t s, const float4 *nlo, const float4 *nhi, const int *nsize, const int *parent, int n_nodes,
               int n, int k, float r0_scale, float rmax, float root_side, float *r0) {
  k_r0<<<(n_nodes + 255) / 256, 256, 0, s>>>(nlo, nhi, nsize, parent, n_nodes, n, k, r0_scale, rmax, root_side, r0);
}

void launch_kids(cudaStream_t s, const float4 *nlo, const float4 *nhi, int n_nodes, int n, float4 *crec, int *parent,
                 int4 *anc4, int *cellof) {
  k_kids<<<(n_nodes + 1 + 255) / 256, 256, 0, s>>>(nlo, nhi, n_nodes, n, crec, parent, cellof);
  k_anc<<<(n_nodes + 255) / 256, 256, 0, s>>>(parent, n_nodes, anc4);
}

int target_list_cap(int k) {
  // per-target list entries (measured best: 4K = 256 at K = 64 on C2, 3K = 384 at K = 128 on C5)
  static const int mult = getenv("SPH_TLISTCAP") ? atoi(getenv("SPH_TLISTCAP")) : 0;
  return std::min(std::max((mult > 0 ? mult : k <= 64 ? 4 : 3) * k, 128), 1024);
}

template <bool F32, bool COLLECT>
void launch_target_t(cudaStream_t s, const PassArgs &a, int cap, int *fallbacks, int num_sms) {
  const int smem = kWarps * warp_smem_bytes(cap);
  int bps = 0;
  cudaFuncSetAttribute(k_target<F32, COLLECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_target<F32, COLLECT>, kWarps * 32, smem);
  k_target<F32, COLLECT><<<num_sms * std::max(bps, 1), kWarps * 32, smem, s>>>(a, cap, fallbacks);
}

void launch_target(cudaStream_t s, int f32, const PassArgs &a, int cap, int *fallbacks, int num_sms, bool collect) {
  if (f32) {
    if (collect) launch_target_t<true, true>(s, a, cap, fallbacks, num_sms);
    else launch_target_t<true, false>(s, a, cap, fallbacks, num_sms);
  } else {
    if (collect) launch_target_t<false, true>(s, a, cap, fallbacks, num_sms);
    else launch_target_t<false, false>(s, a, cap, fallbacks, num_sms);
  }
}

}  // namespace sph
