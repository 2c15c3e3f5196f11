// sph_pass.cu -- the neighbour kernels.
//
// One warp serves a bundle of 32 targets (consecutive entries of a target
// list in sorted order, so spatially coherent).  The warp walks the
// pre-order search tree once per periodic image shift with a stackless
// skip-pointer walk: 32 nodes are box-tested at a time (one per lane) and
// the walk itself is a warp-uniform bit scan over the hit mask.  Cells the
// bundle box (grown by the largest lane radius) touches are merged into
// contiguous particle ranges; each range is staged 32 candidates at a time
// in shared memory and every lane tests its own target against each
// staged candidate (broadcast reads).  What a lane does with a candidate
// depends on the mode:
//
//   MODE_HIST   counts candidates in 32 d^2 bins over [0, R_i^2]: yields the
//               bracket bin of the K-th neighbour, or a retry with larger R
//   MODE_BAND   exact K-th d^2: counts exactly (unfused fp64) what lies below
//               the bracket, keeps the in-bracket values, selects the rank;
//               overfull brackets are refined with a 16-bin sub-histogram
//   MODE_DENS   rho_i = sum_j m_j W(r_ij, h_i), h_i = sqrt(d2_K)
//   MODE_COUNT  fixed-h neighbour counts (parity entry point)
//
// fp32 path: candidate tests run in fp32 (positions are exact fp32 values);
// any candidate whose fp32 d^2 lies within a relative 2^-20 of a threshold is
// re-tested in unfused fp64 on the widened values, so counts and the K-th
// d^2 are exactly the reference's fp64 results.
#include "sph_internal.cuh"


#include <algorithm>

namespace sph {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 4;
// geometric histogram: bin = exponent and top two mantissa bits of d2/R_b^2,
// 4 bins per octave of d2 over [2^-12, 1) plus an underflow bin and x == 1
constexpr int kHistOctaves = 12;
constexpr int kHistBase = (127 - kHistOctaves) << 2;
constexpr int NB_HIST = kHistOctaves * 4 + 2;
constexpr int BAND_CAP = 32;
constexpr int NB_BAND = 16;
constexpr unsigned kCellTag = 0xff000000u;  // neighbour-list entry: .y = tag | count -> whole cell [.x, .x + count)
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard
constexpr double kEpsD = 9.5367431640625e-07;

struct alignas(32) D4 { double x, y, z, m; };

template <bool F32> struct Stage;
template <> struct Stage<true> { using T = float4; };
template <> struct Stage<false> { using T = D4; };

// per warp: two staging buffers of 32 candidates + their sorted indices,
// the range prefix sums and range bases, then the mode's per-lane tables
template <bool F32>
constexpr int stage_bytes() {
  return 2 * 32 * (F32 ? 16 : 32) + 4 * 32 * 4;
}
template <int MODE, bool F32>
constexpr int mode_smem_per_warp() {
  return stage_bytes<F32>() +
         (MODE == MODE_HIST ? NB_HIST * 32 * 4 : MODE == MODE_BAND ? (BAND_CAP * 32 * 8 + NB_BAND * 32 * 4) : 0);
}

__device__ __forceinline__ float warp_min(float v) {
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// unfused fp64 d2 of candidate image x_j + s*box from target x_i
__device__ __forceinline__ double exact_image_d2(double cx, double cy, double cz, bool shifted, double dsx,
                                                 double dsy, double dsz, double tx, double ty, double tz) {
  if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
  return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
}

// squared gap between two boxes
__device__ __forceinline__ float box_gap2(float4 lo, float4 hi, float qlx, float qly, float qlz, float qhx,
                                          float qhy, float qhz) {
  const float gx = fmaxf(fmaxf(lo.x - qhx, qlx - hi.x), 0.f);
  const float gy = fmaxf(fmaxf(lo.y - qhy, qly - hi.y), 0.f);
  const float gz = fmaxf(fmaxf(lo.z - qhz, qlz - hi.z), 0.f);
  return gx * gx + gy * gy + gz * gz;
}

// One task: a spatially coherent group of <= 32 targets (one per lane) runs
// one sweep of MODE and leaves its per-target results / next state in the
// PassArgs arrays.  Returns nothing; `b` is the task index (diagnostics).
template <int MODE, bool F32>
__device__ __forceinline__ void run_task(const PassArgs &a, const int2 task, const int b, unsigned char *wbase,
                                         unsigned long long &tests, unsigned long long &accepted) {
  using StageT = typename Stage<F32>::T;
  const int lane = threadIdx.x & 31;
  StageT *stage = reinterpret_cast<StageT *>(wbase);
  int *sidxbuf = reinterpret_cast<int *>(wbase + 2 * 32 * sizeof(StageT));
  int *spfx = sidxbuf + 64;
  int *srsm = spfx + 32;
  unsigned char *mbase = wbase + stage_bytes<F32>();
  unsigned *hist = reinterpret_cast<unsigned *>(mbase);                           // HIST
  double *band = reinterpret_cast<double *>(mbase);                               // BAND
  unsigned *bh = reinterpret_cast<unsigned *>(mbase + BAND_CAP * 32 * 8);         // BAND
  const StageT *__restrict__ pos = reinterpret_cast<const StageT *>(a.pos);
  const float4 *__restrict__ nlo = a.tree.nlo;
  const float4 *__restrict__ nhi = a.tree.nhi;
  const int n_nodes = a.tree.n_nodes;
  const int n = a.n;
  const int K = a.k;
    const long long dbg_t0 = a.dbg ? clock64() : 0;
    const unsigned long long dbg_tests0 = tests;
    int dbg_subs = 0;
    float dbg_rb = 0.f;
    unsigned long long dbg_win = 0, dbg_cvis = 0, dbg_cneed = 0, dbg_flush = 0;
    const bool active = lane < task.y;
    const int p = (int)a.members[task.x + (active ? lane : 0)];
    const unsigned amask = __ballot_sync(FULL, active);

    // target position (exact) and fp32 copy
    double tx, ty, tz;
    float fx, fy, fz;
    {
      const int src = __shfl_sync(FULL, p, __ffs(amask) - 1);
      const int pp = active ? p : src;
      if constexpr (F32) {
        const float4 v = reinterpret_cast<const float4 *>(a.pos)[pp];
        fx = v.x; fy = v.y; fz = v.z;
        tx = v.x; ty = v.y; tz = v.z;
      } else {
        const D4 v = reinterpret_cast<const D4 *>(a.pos)[pp];
        tx = v.x; ty = v.y; tz = v.z;
        fx = (float)tx; fy = (float)ty; fz = (float)tz;
      }
    }

    // ---- per-lane state ----
    float rad = 0.f;
    float hR2 = 0.f;  // HIST: histogram range R_b^2 of this lane's sub-bundle
    float h_fin = 0.f;  // HIST: final (shrunk) acceptance radius^2: the recorded list is complete below it
    int ne = 0;         // HIST: neighbour-list entries recorded for this lane's target
    // BAND
    double lo = 0.0, hi = -1.0, scale = 0.0, emin = INFINITY, emax = -INFINITY;
    float lo_f = -1.f, hi_f = -2.f;
    int c_below = 0, n_in = 0;
    // DENS
    double d2k = 0.0, hh = 0.0, norm_h3 = 0.0, accd = 0.0;
    float d2k_f = -1.f, inv_h = 0.f, accf = 0.f;
    // COUNT
    double r2 = -1.0;
    float r2_lo_f = -1.f, r2_hi_f = -2.f;
    int cnt = 0;

    if constexpr (MODE == MODE_HIST) {
#pragma unroll
      for (int bb = 0; bb < NB_HIST; ++bb) hist[bb * 32 + lane] = 0u;
      if (active) rad = a.radius[p];
    } else if constexpr (MODE == MODE_BAND) {
#pragma unroll
      for (int bb = 0; bb < NB_BAND; ++bb) bh[bb * 32 + lane] = 0u;
      if (active) {
        lo = a.t_lo[p];
        hi = a.t_hi[p];
        scale = hi > lo ? (double)NB_BAND / (hi - lo) : 0.0;
        lo_f = __double2float_rd(lo * (1.0 - kEpsD)) - 1e-37f;
        hi_f = __double2float_ru(hi * (1.0 + kEpsD)) + 1e-37f;
        rad = __double2float_ru(sqrt(hi) * (1.0 + kEpsD)) + 1e-30f;
      }
    } else if constexpr (MODE == MODE_DENS) {
      if (active) {
        d2k = a.d2k[p];
        hh = __dsqrt_rn(d2k);
        norm_h3 = __ddiv_rn(a.kernel_kind == 0 ? kWc6Norm : kM4Norm, __dmul_rn(__dmul_rn(hh, hh), hh));
        d2k_f = __double2float_ru(d2k * (1.0 + kEpsD));
        inv_h = (float)(1.0 / hh);
        rad = __double2float_ru(hh * (1.0 + kEpsD)) + 1e-30f;
      }
    } else {  // COUNT
      if (active) {
        const double hf = a.hfix[p];
        r2 = __dmul_rn(hf, hf);
        r2_lo_f = __double2float_rd(r2 * (1.0 - kEpsD)) - 1e-37f;
        r2_hi_f = __double2float_ru(r2 * (1.0 + kEpsD)) + 1e-37f;
        rad = __double2float_ru(fabs(hf) * (1.0 + kEpsD)) + 1e-30f;
        if (!(rad >= 0.f)) rad = 0.f;  // NaN h: counts nothing (d2 <= NaN is false)
      }
    }

    // ---- spatially coherent sub-bundles ----
    // A list chunk can hold targets from distant places (compacted retry
    // lists in clustered data); each sub-bundle = the pending targets within
    // 1.5 radii (Chebyshev) of its leader, walked and tested on its own.
    unsigned pending = amask;
    while (pending) {
      const int leader = __ffs(pending) - 1;
      const float lx = __shfl_sync(FULL, fx, leader), ly = __shfl_sync(FULL, fy, leader),
                  lz = __shfl_sync(FULL, fz, leader);
      const float D = INFINITY;  // tasks are already coherent groups
      const bool mem = ((pending >> lane) & 1u) && fabsf(fx - lx) <= D && fabsf(fy - ly) <= D &&
                       fabsf(fz - lz) <= D;
      const unsigned mmask = __ballot_sync(FULL, mem) | (1u << leader);
      const bool member = (mmask >> lane) & 1u;
      pending &= ~mmask;
      const int n_mem = __popc(mmask);
      ++dbg_subs;

      // sub-bundle box and radius
      float bx0 = member ? (F32 ? fx : __double2float_rd(tx)) : INFINITY;
      float by0 = member ? (F32 ? fy : __double2float_rd(ty)) : INFINITY;
      float bz0 = member ? (F32 ? fz : __double2float_rd(tz)) : INFINITY;
      float bx1 = member ? (F32 ? fx : __double2float_ru(tx)) : -INFINITY;
      float by1 = member ? (F32 ? fy : __double2float_ru(ty)) : -INFINITY;
      float bz1 = member ? (F32 ? fz : __double2float_ru(tz)) : -INFINITY;
      bx0 = warp_min(bx0); by0 = warp_min(by0); bz0 = warp_min(bz0);
      bx1 = warp_max(bx1); by1 = warp_max(by1); bz1 = warp_max(bz1);
      const float Rb = warp_max(member ? rad : 0.f);
      float R2b = Rb * Rb * (1.0f + 4.0f * kEps) + 1e-37f;
      dbg_rb = fmaxf(dbg_rb, Rb);

      // effective per-lane thresholds for this sub-bundle (non-members: none)
      float h_r2 = -1.f, h_inv = 0.f;  // HIST
      if constexpr (MODE == MODE_HIST) {
        if (member) {
          hR2 = rad * rad;
          h_r2 = hR2;
          h_fin = hR2;
          h_inv = 1.0f / hR2;
        }
      }
      double h_r2d = (double)h_r2;
      const double h_invd = (double)h_inv;
      int seen = 0;  // HIST: candidates counted so far (self included)
      int seen_shrunk = 0;
      // Adaptive shrink: once >= K others are counted, the K-th lies at or
      // below the upper edge of the bin holding the K-th so far; farther
      // candidates cannot change it, so the lane stops looking beyond.  A
      // recorded neighbour list is compacted to the new radius.
      auto shrink = [&](int, float &hr2) {
        int cum = 0, bb = 0;
        for (; bb < NB_HIST; ++bb) {
          cum += (int)hist[bb * 32 + lane];
          if (cum > K) break;
        }
        if (bb < NB_HIST - 1) {
          const float edge = __int_as_float((kHistBase + bb) << 21) * hR2 * (1.0f + 4.0f * kEps);
          if (edge < hr2) {
            hr2 = edge;
            h_fin = edge;
          }
        }
      };
      const float e_lo_f = member ? lo_f : -1.f, e_hi_f = member ? hi_f : -2.f;
      const float e_d2k_f = member ? d2k_f : -1.f;
      const double e_d2k = member ? d2k : -1.0;
      const float e_r2_lo_f = member ? r2_lo_f : -1.f, e_r2_hi_f = member ? r2_hi_f : -2.f;
      const double e_r2 = member ? r2 : -1.0;

      const int n_shift = a.periodic ? 27 : 1;
      for (int sidx = 0; sidx < n_shift; ++sidx) {
        const int sx = a.periodic ? sidx / 9 - 1 : 0;
        const int sy = a.periodic ? (sidx / 3) % 3 - 1 : 0;
        const int sz = a.periodic ? sidx % 3 - 1 : 0;
        const bool shifted = (sx | sy | sz) != 0;
        // candidates j are images x_j + s*box: query the tree around x_i - s*box
        float qlx = bx0, qly = by0, qlz = bz0, qhx = bx1, qhy = by1, qhz = bz1;
        if (shifted) {
          const double bxs = a.box;
          qlx = __double2float_rd((double)bx0 - sx * bxs); qhx = __double2float_ru((double)bx1 - sx * bxs);
          qly = __double2float_rd((double)by0 - sy * bxs); qhy = __double2float_ru((double)by1 - sy * bxs);
          qlz = __double2float_rd((double)bz0 - sz * bxs); qhz = __double2float_ru((double)bz1 - sz * bxs);
          if (box_gap2(nlo[0], nhi[0], qlx, qly, qlz, qhx, qhy, qhz) > R2b) continue;
        }
        const float boxf = (float)a.box;
        // image offsets with the box side in two fp32 words, box = hi + lo (see
        // k_target): -1 shift: candidate - hi (exact), target + lo; +1 shift:
        // the target moves, (x_i - hi) - lo
        const float bxh = boxf, bxl = (float)(a.box - (double)boxf);
        const float csx = sx < 0 ? -bxh : 0.f, csy = sy < 0 ? -bxh : 0.f, csz = sz < 0 ? -bxh : 0.f;
        const float tfx = sx < 0 ? fx + bxl : sx > 0 ? (fx - bxh) - bxl : fx,
                    tfy = sy < 0 ? fy + bxl : sy > 0 ? (fy - bxh) - bxl : fy,
                    tfz = sz < 0 ? fz + bxl : sz > 0 ? (fz - bxh) - bxl : fz;
        const double dsx = sx * a.box, dsy = sy * a.box, dsz = sz * a.box;
        // this lane's target in the tree frame of the shift (x_i - s*box), plus slack
        const float pqx = shifted ? (float)(tx - dsx) : fx, pqy = shifted ? (float)(ty - dsy) : fy,
                    pqz = shifted ? (float)(tz - dsz) : fz;
        const float pslack = shifted ? boxf * 4.8e-7f : (F32 ? 0.f : fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))) * 1.2e-7f);

        // range list: lane r holds range r
        int rs = 0, re = 0;
        int nr = 0, last_e = -1;

        // ---- stackless pre-order walk, interleaved with candidate processing ----
        // A window of 32 consecutive pre-order nodes is box-tested at once (one
        // per lane).  A missed node hides its subtree (the nodes up to its skip
        // pointer); the visited nodes of the window are the hits not hidden by
        // an earlier miss, found with one OR-reduction, and the walk jumps to
        // the farthest skip of an unhidden miss.  Only visited cells are then
        // handled one by one, in pre-order.
        int kk = 0;
        unsigned pend = 0u;
        int w = 0;
        float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
        int my_start = n, next_start = n;
        for (;;) {
          bool full = false;
          for (;;) {
            if (!pend) {
              if (kk >= n_nodes) break;
              w = kk;
              ++dbg_win;
              const int my = w + lane;
              bool hit = false;
              int my_skip = n_nodes;
              my_start = n;
              l4 = make_float4(0.f, 0.f, 0.f, 0.f);
              h4 = l4;
              if (my < n_nodes) {
                l4 = nlo[my];
                h4 = nhi[my];
                my_skip = __float_as_int(l4.w);
                my_start = __float_as_int(h4.w);
                hit = box_gap2(l4, h4, qlx, qly, qlz, qhx, qhy, qhz) <= R2b;
              }
              // Internal nodes with many particles that are small next to the
              // group's search region: keep them only if some member's own
              // sphere reaches them (a dense clump at the edge of the group box
              // would otherwise be descended cell by cell).
              {
                const bool big = hit && my_skip != my + 1 &&
                                 fmaxf(h4.x - l4.x, fmaxf(h4.y - l4.y, h4.z - l4.z)) < 2.0f * Rb &&
                                 a.tree.nsize[my] > 128;
                const unsigned bigm = __ballot_sync(FULL, big);
                if (bigm) {
                  float wr2;
                  if constexpr (MODE == MODE_HIST) wr2 = h_r2;
                  else if constexpr (MODE == MODE_BAND) wr2 = e_hi_f;
                  else if constexpr (MODE == MODE_DENS) wr2 = e_d2k_f;
                  else wr2 = e_r2_hi_f;
                  bool keep = false;
                  unsigned mm = __ballot_sync(FULL, member);
                  while (mm) {
                    const int m = __ffs(mm) - 1;
                    mm &= mm - 1u;
                    const float mx = __shfl_sync(FULL, pqx, m), my_ = __shfl_sync(FULL, pqy, m),
                                mz = __shfl_sync(FULL, pqz, m), mr2 = __shfl_sync(FULL, wr2, m),
                                ms = __shfl_sync(FULL, pslack, m);
                    const float gx = fmaxf(fmaxf(l4.x - mx, mx - h4.x) - ms, 0.f);
                    const float gy = fmaxf(fmaxf(l4.y - my_, my_ - h4.y) - ms, 0.f);
                    const float gz = fmaxf(fmaxf(l4.z - mz, mz - h4.z) - ms, 0.f);
                    keep = keep || (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= mr2;
                  }
                  if (big) hit = keep;
                }
              }
              next_start = __shfl_down_sync(FULL, my_start, 1);
              if (lane == 31) next_start = (w + 32 < n_nodes) ? __float_as_int(nhi[w + 32].w) : n;
              unsigned cov = 0u;
              if (my < n_nodes && !hit) {
                const int e = min(my_skip - w, 32);
                cov = (e >= 32 ? 0xffffffffu : ((1u << e) - 1u)) & ~((2u << lane) - 1u);
              }
              const unsigned covered = __reduce_or_sync(FULL, cov);
              const unsigned hitm = __ballot_sync(FULL, hit);
              const unsigned cellm = __ballot_sync(FULL, my < n_nodes && my_skip == my + 1);
              const bool jump = my < n_nodes && !hit && !((covered >> lane) & 1u);
              const int far = (int)__reduce_max_sync(FULL, jump ? (unsigned)my_skip : 0u);
              kk = max(w + 32, far);
              pend = hitm & ~covered & cellm;
              continue;
            }
            const int bb = __ffs(pend) - 1;
            ++dbg_cvis;
            {
                  // Cell: classify it against each member's own thresholds from
                  // its box alone.  If no member needs its particles (outside
                  // every sphere, or wholly inside one histogram bin / wholly
                  // below the bracket), count it without pair tests and skip it.
                  const float cx0 = __shfl_sync(FULL, l4.x, bb), cy0 = __shfl_sync(FULL, l4.y, bb),
                              cz0 = __shfl_sync(FULL, l4.z, bb), cx1 = __shfl_sync(FULL, h4.x, bb),
                              cy1 = __shfl_sync(FULL, h4.y, bb), cz1 = __shfl_sync(FULL, h4.z, bb);
                  const int s0 = __shfl_sync(FULL, my_start, bb);
                  const int e0 = __shfl_sync(FULL, next_start, bb);
                  const float gx = fmaxf(fmaxf(cx0 - pqx, pqx - cx1) - pslack, 0.f);
                  const float gy = fmaxf(fmaxf(cy0 - pqy, pqy - cy1) - pslack, 0.f);
                  const float gz = fmaxf(fmaxf(cz0 - pqz, pqz - cz1) - pslack, 0.f);
                  const float gap2 = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps);
                  const float fxa = fmaxf(pqx - cx0, cx1 - pqx) + pslack;
                  const float fya = fmaxf(pqy - cy0, cy1 - pqy) + pslack;
                  const float fza = fmaxf(pqz - cz0, cz1 - pqz) + pslack;
                  const float dmax2 = (fxa * fxa + fya * fya + fza * fza) * (1.0f + 4.0f * kEps);
                  const int ncell = e0 - s0;
                  const int self_in = (!shifted && s0 <= p && p < e0) ? 1 : 0;
                  bool need = false;
                  int sc = -1;
                  if constexpr (MODE == MODE_HIST) {
                    if (gap2 <= h_r2) {
                      const int b0 = min(max((__float_as_int(gap2 * h_inv) >> 21) - kHistBase + 1, 0), NB_HIST - 1);
                      const int b1 = min(max((__float_as_int(dmax2 * h_inv) >> 21) - kHistBase + 1, 0), NB_HIST - 1);
                      if (dmax2 <= h_r2 && b0 == b1) sc = b0; else need = true;
                    }
                  } else if constexpr (MODE == MODE_BAND) {
                    if (!(gap2 > e_hi_f)) {
                      if (dmax2 < e_lo_f) sc = ncell - self_in; else need = true;
                    }
                  } else if constexpr (MODE == MODE_COUNT) {
                    if (!(gap2 > e_r2_hi_f)) {
                      if (dmax2 <= e_r2_lo_f) sc = ncell - self_in; else need = true;
                    }
                  } else {
                    need = gap2 < e_d2k_f;
                  }
                  if (!((a.shortcut >> MODE) & 1)) need = need || sc >= 0;
                  if (!__any_sync(FULL, need)) {
                    if constexpr (MODE == MODE_HIST) {
                      if (sc >= 0) {
                        hist[sc * 32 + lane] += (unsigned)ncell;
                        seen += ncell;
                      }
                    } else if constexpr (MODE == MODE_BAND) {
                      if (sc > 0) c_below += sc;
                    } else if constexpr (MODE == MODE_COUNT) {
                      if (sc > 0) cnt += sc;
                    }
                    pend &= pend - 1u;
                    continue;
                  }
                  ++dbg_cneed;
                  if (s0 == last_e) {
                    if (lane == nr - 1) re = e0;
                  } else {
                    if (nr == 32) { full = true; --dbg_cneed; break; }  // resume at this cell after processing
                    if (lane == nr) { rs = s0; re = e0; }
                    ++nr;
                  }
                  last_e = e0;
            }
            pend &= pend - 1u;
          }
          {
            // Pack the ranges into one candidate stream, 32 per chunk, double
            // buffered: the next chunk's loads are in flight while this chunk
            // is tested.  Stream index s maps to range r = #{pfx <= s}.
            ++dbg_flush;
            const int len = lane < nr ? re - rs : 0;
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(FULL, incl, o);
              if (lane >= o) incl += v;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            spfx[lane] = incl;
            srsm[lane] = rs - (incl - len);
            __syncwarp();
            auto cand_of = [&](int sidx) -> int {
              int r = 0;
#pragma unroll
              for (int step = 16; step; step >>= 1)
                if (spfx[r + step - 1] <= sidx) r += step;
              return srsm[r] + sidx;
            };
            int my_ci = lane < total ? cand_of(lane) : 0;
            StageT v_cur;
            if (lane < total) v_cur = pos[my_ci];
            for (int c0 = 0; c0 < total; c0 += 32) {
              StageT *stb = stage + ((c0 >> 5) & 1) * 32;
              int *sti = sidxbuf + ((c0 >> 5) & 1) * 32;
              const int nc = min(32, total - c0);
              // slots past nc hold a NaN sentinel: every test below is a
              // comparison that is false for NaN, so the batch of 4 needs no tail
              if (lane < nc) { stb[lane] = v_cur; sti[lane] = my_ci; }
              else { StageT z = v_cur; z.x = __int_as_float(0x7fc00000); stb[lane] = z; sti[lane] = -1; }
              __syncwarp();
              if (c0 + 32 + lane < total) {
                my_ci = cand_of(c0 + 32 + lane);
                v_cur = pos[my_ci];
              }
              tests += (unsigned long long)nc * n_mem;
              // batches of BU loaded before any shared store: the candidate
              // loads and distance math of a batch overlap (DENS keeps BU=1:
              // its register budget is taken by the kernel evaluation)
              constexpr int BU = MODE == MODE_DENS ? 1 : 4;
              const int ncr = (nc + BU - 1) & ~(BU - 1);
#pragma unroll 1
              for (int j0 = 0; j0 < ncr; j0 += BU) {
               StageT cb[BU];
               int ib[BU];
#pragma unroll
               for (int u = 0; u < BU; ++u) { cb[u] = stb[j0 + u]; ib[u] = sti[j0 + u]; }
#pragma unroll
               for (int u = 0; u < BU; ++u) {
                const StageT c = cb[u];
                const int cidx = ib[u];
                float af = 0.f;
                double ad = 0.0;
                if constexpr (F32) {
                  float dx, dy, dz;
                  if (shifted) {
                    // box side in two fp32 words (see k_target): within the guard band
                    dx = (c.x + csx) - tfx; dy = (c.y + csy) - tfy; dz = (c.z + csz) - tfz;
                  } else {
                    dx = c.x - fx; dy = c.y - fy; dz = c.z - fz;
                  }
                  af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
                } else {
                  double cx = c.x, cy = c.y, cz = c.z;
                  if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
                  ad = exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
                }
#define EXACT_D2() exact_image_d2((double)c.x, (double)c.y, (double)c.z, shifted, dsx, dsy, dsz, tx, ty, tz)
                const bool is_self = (cidx == p) && !shifted;

                if constexpr (MODE == MODE_HIST) {
                  // geometric bins: exponent + 2 mantissa bits of d2 / R_b^2
                  bool in;
                  float x;
                  if constexpr (F32) { in = af <= h_r2; x = af * h_inv; }
                  else { in = ad <= h_r2d; x = (float)(ad * h_invd); }
                  if (in) {
                    const int bin = min(max((__float_as_int(x) >> 21) - kHistBase + 1, 0), NB_HIST - 1);
                    atomicAdd(&hist[bin * 32 + lane], 1u);  // no return value: no LDS->STS chain
                    ++seen;
                  }
                } else if constexpr (MODE == MODE_BAND) {
                  if (!is_self) {
                    double e = -1.0;
                    if constexpr (F32) {
                      if (af < e_lo_f) ++c_below;
                      else if (af <= e_hi_f) e = EXACT_D2();
                    } else {
                      e = member ? ad : -1.0;
                    }
                    if (e >= 0.0) {
                      if (e < lo) ++c_below;
                      else if (e <= hi) {
                        if (n_in < BAND_CAP) band[n_in * 32 + lane] = e;
                        ++n_in;
                        emin = fmin(emin, e);
                        emax = fmax(emax, e);
                        const int bin = min(max((int)((e - lo) * scale), 0), NB_BAND - 1);
                        atomicAdd(&bh[bin * 32 + lane], 1u);
                      }
                    }
                  }
                } else if constexpr (MODE == MODE_DENS) {
                  if constexpr (F32) {
                    if (af < e_d2k_f) {
                      if (a.dens64) {
                        // fp64 evaluation of the accepted pair, term-for-term the reference's
                        const double e = EXACT_D2();
                        if (e < d2k) {
                          const double r_ = __dsqrt_rn(e);
                          double w;
                          if (a.kernel_kind == 0) {
                            w = wc6_lowered(r_, hh, norm_h3);
                          } else {
                            const double q = __ddiv_rn(r_, hh);
                            w = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
                          }
                          accd = __dadd_rn(accd, __dmul_rn(a.mass64[cidx], w));
                        }
                      } else {
                        const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
                        const float q = rr * inv_h;
                        const float w = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
                        if (q < 1.f) accf = fmaf(c.w, w, accf);
                      }
                      ++accepted;
                    }
                  } else {
                    if (ad < e_d2k) {
                      const double r_ = __dsqrt_rn(ad);
                      double w;
                      if (a.kernel_kind == 0) {
                        w = wc6_lowered(r_, hh, norm_h3);
                      } else {
                        const double q = __ddiv_rn(r_, hh);
                        w = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
                      }
                      accd = __dadd_rn(accd, __dmul_rn(c.m, w));
                      ++accepted;
                    }
                  }
                } else {  // COUNT
                  if (!is_self) {
                    if constexpr (F32) {
                      if (af <= e_r2_lo_f) ++cnt;
                      else if (af <= e_r2_hi_f) cnt += EXACT_D2() <= r2;
                    } else {
                      cnt += ad <= e_r2;
                    }
                  }
                }
               }
              }
              if constexpr (MODE == MODE_HIST) h_r2d = (double)h_r2;
            }
            __syncwarp();
          }
          if constexpr (MODE == MODE_HIST) {
            if (member && seen > K) shrink(seen, h_r2);
            h_r2d = (double)h_r2;
            R2b = fminf(R2b, warp_max(member ? h_r2 : 0.f) * (1.0f + 4.0f * kEps) + 1e-37f);
          }
          nr = 0;
          last_e = -1;
          if (!full) break;
        }
      }
    }

    if (a.dbg && lane == 0) {
      unsigned long long *d = a.dbg + 8ull * b;
      d[4] = dbg_win;
      d[5] = dbg_cvis;
      d[6] = dbg_cneed;
      d[7] = dbg_flush;
      d[0] = (unsigned long long)(clock64() - dbg_t0);
      d[1] = tests - dbg_tests0;
      d[2] = ((unsigned long long)(unsigned)p << 32) | ((unsigned)__popc(amask) << 8) | (unsigned)dbg_subs;
      d[3] = (unsigned long long)__float_as_uint(dbg_rb);
    }
    // ---- per-mode finish ----
    if constexpr (MODE == MODE_HIST) {
      if (active) {
        unsigned total = 0;
#pragma unroll
        for (int bb = 0; bb < NB_HIST; ++bb) total += hist[bb * 32 + lane];
        total -= 1u;  // the target itself (d2 = 0, bin 0)
        const float Rused = sqrtf(hR2);
        if ((int)total < K) {
          if (Rused >= a.rmax) {
            a.state[p] = ST_UNREACHABLE;
            a.d2k[p] = INFINITY;
          } else {
            float f = total > 0 ? cbrtf((float)(K + 8) / (float)total) * 1.15f : 2.f;
            f = fminf(fmaxf(f, 1.26f), 2.5f);
            a.radius[p] = fminf(fmaxf(Rused, rad) * f, a.rmax);
          }
        } else {
          int cum = 0, bb = 0;
          for (; bb < NB_HIST; ++bb) {
            const int hcount = (int)hist[bb * 32 + lane] - (bb == 0 ? 1 : 0);
            if (cum + hcount >= K) break;
            cum += hcount;
          }
          const double R2d = (double)hR2;
          double tl, th;
          if (bb == 0) {
            tl = 0.0;
            th = (double)__int_as_float(kHistBase << 21) * R2d * (1.0 + 8.0 * kEpsD);
          } else if (bb >= NB_HIST - 1) {
            tl = R2d * (1.0 - 8.0 * kEpsD);
            th = R2d * (1.0 + 8.0 * kEpsD);
          } else {
            tl = (double)__int_as_float((kHistBase + bb - 1) << 21) * R2d * (1.0 - 8.0 * kEpsD);
            th = (double)__int_as_float((kHistBase + bb) << 21) * R2d * (1.0 + 8.0 * kEpsD);
          }
          a.t_lo[p] = tl;
          a.t_hi[p] = th;
          a.radius[p] = Rused;
          a.state[p] = ST_NEED_BAND;
        }
      }
    } else if constexpr (MODE == MODE_BAND) {
      if (active) {
        const int r = K - c_below;  // 1-based rank inside the bracket
        if (r <= 0) {
          a.t_hi[p] = nextafter(lo, -INFINITY);
          a.t_lo[p] = 0.0;
        } else if (r > n_in) {
          const float Rr = a.radius[p];
          a.t_lo[p] = nextafter(hi, INFINITY);
          a.t_hi[p] = (double)Rr * (double)Rr * (1.0 + 16.0 * kEpsD);
        } else if (n_in <= BAND_CAP) {
          double v = 0.0;
          for (int i = 0; i < n_in; ++i) {
            const double ei = band[i * 32 + lane];
            int less = 0, eq = 0;
            for (int j2 = 0; j2 < n_in; ++j2) {
              const double ej = band[j2 * 32 + lane];
              less += ej < ei;
              eq += ej == ei;
            }
            if (less < r && r <= less + eq) { v = ei; break; }
          }
          a.d2k[p] = v;
          a.state[p] = ST_DONE;
        } else if (emin == emax) {
          a.d2k[p] = emin;
          a.state[p] = ST_DONE;
        } else {
          int cum = 0, bb = 0;
          for (; bb < NB_BAND; ++bb) {
            const int hcount = (int)bh[bb * 32 + lane];
            if (cum + hcount >= r) break;
            cum += hcount;
          }
          bb = min(bb, NB_BAND - 1);
          const double width = hi - lo;
          double nl = bb == 0 ? lo : lo + (double)bb / scale - width * 1e-12;
          double nh = bb == NB_BAND - 1 ? hi : lo + (double)(bb + 1) / scale + width * 1e-12;
          nl = fmax(nextafter(nl, -INFINITY), fmax(lo, emin));
          nh = fmin(nextafter(nh, INFINITY), fmin(hi, emax));
          a.t_lo[p] = nl;
          a.t_hi[p] = nh;
        }
      }
    } else if constexpr (MODE == MODE_DENS) {
      if (active) {
        a.rho[p] = (F32 && !a.dens64) ? __dmul_rn(norm_h3, (double)accf) : accd;
      }
    } else {
      if (active) a.counts[p] = cnt;
    }
}

template <int MODE, bool F32>
__global__ void __launch_bounds__(kWarps * 32) k_pass(const PassArgs a) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *wbase = smem_raw + wib * mode_smem_per_warp<MODE, F32>();
  unsigned long long tests = 0, accepted = 0;
  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(a.work_counter, 1);
    b = __shfl_sync(FULL, b, 0);
    if (b >= *a.task_count) break;
    run_task<MODE, F32>(a, a.tasks[b], b, wbase, tests, accepted);
  }
  // statistics
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
  }
}


// Group the pending targets of a list into spatially coherent tasks: each
// warp takes 32 consecutive list entries (sorted order) and splits them
// greedily into groups whose members lie within sub_d * (leader radius) of
// the leader (Chebyshev).  Groups are written contiguously to `members` and
// described by (offset, count) in `tasks`; the pass kernels then schedule
// tasks dynamically, one per warp, so distant targets never share a walk.
template <int MODE, bool F32>
__global__ void k_form(const PassArgs a, int count, uint8_t want) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int c = gw; c * 32 < count; c += nw) {
    const int t = c * 32 + lane;
    bool active = t < count;
    const int p = a.list ? (int)a.list[active ? t : c * 32] : (active ? t : c * 32);
    if constexpr (MODE != MODE_COUNT) active = active && a.state[p] == want;
    float rad = 0.f;
    if (active) {
      if constexpr (MODE == MODE_HIST) rad = a.radius[p];
      else if constexpr (MODE == MODE_BAND) rad = (float)sqrt(a.t_hi[p]);
      else if constexpr (MODE == MODE_DENS) rad = (float)sqrt(a.d2k[p]);
      else rad = fabsf((float)a.hfix[p]);
      if (!(rad >= 0.f)) rad = 0.f;
    }
    float fx, fy, fz;
    if constexpr (F32) {
      const float4 v = reinterpret_cast<const float4 *>(a.pos)[p];
      fx = v.x; fy = v.y; fz = v.z;
    } else {
      const D4 v = reinterpret_cast<const D4 *>(a.pos)[p];
      fx = (float)v.x; fy = (float)v.y; fz = (float)v.z;
    }
    unsigned pending = __ballot_sync(FULL, active);
    while (pending) {
      // leader: the pending target nearest the centre of the pending targets' box,
      // so that a group uses its whole +-D extent instead of starting at a corner
      const bool pend_me = (pending >> lane) & 1u;
      float cx = 0.5f * (warp_min(pend_me ? fx : INFINITY) + warp_max(pend_me ? fx : -INFINITY));
      float cy = 0.5f * (warp_min(pend_me ? fy : INFINITY) + warp_max(pend_me ? fy : -INFINITY));
      float cz = 0.5f * (warp_min(pend_me ? fz : INFINITY) + warp_max(pend_me ? fz : -INFINITY));
      const float dc = pend_me ? fmaxf(fabsf(fx - cx), fmaxf(fabsf(fy - cy), fabsf(fz - cz))) : INFINITY;
      const float dmin = warp_min(dc);
      const int leader = __ffs(__ballot_sync(FULL, pend_me && dc == dmin)) - 1;
      const float lx = __shfl_sync(FULL, fx, leader), ly = __shfl_sync(FULL, fy, leader),
                  lz = __shfl_sync(FULL, fz, leader);
      const float D = a.sub_d * __shfl_sync(FULL, rad, leader) + 1e-30f;
      const bool mem = ((pending >> lane) & 1u) && fabsf(fx - lx) <= D && fabsf(fy - ly) <= D &&
                       fabsf(fz - lz) <= D;
      const unsigned mmask = __ballot_sync(FULL, mem) | (1u << leader);
      pending &= ~mmask;
      const int nm = __popc(mmask);
      int off = 0;
      if (lane == 0) {
        off = atomicAdd(a.member_cursor, nm);
        const int slot = atomicAdd(a.task_count, 1);
        a.tasks[slot] = make_int2(off, nm);
      }
      off = __shfl_sync(FULL, off, 0);
      if ((mmask >> lane) & 1u) a.members[off + __popc(mmask & ((1u << lane) - 1u))] = (uint32_t)p;
    }
  }
}

template <int MODE, bool F32>
void launch_one(cudaStream_t s, const PassArgs &a, int num_sms) {
  constexpr int smem = kWarps * mode_smem_per_warp<MODE, F32>();
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaFuncSetAttribute(k_pass<MODE, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_pass<MODE, F32>, kWarps * 32, smem);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  k_pass<MODE, F32><<<num_sms * blocks_per_sm, kWarps * 32, smem, s>>>(a);
}

}  // namespace

template <int MODE, bool F32>
void launch_form(cudaStream_t s, const PassArgs &a, int count, uint8_t want, int num_sms) {
  const int warps = (count + 31) / 32;
  const int blocks = std::max(1, std::min((warps + 7) / 8, num_sms * 16));
  k_form<MODE, F32><<<blocks, 256, 0, s>>>(a, count, want);
}

void launch_pass(cudaStream_t s, int mode, int f32, const PassArgs &a, int count, uint8_t want, int num_sms) {
  cudaMemsetAsync(a.work_counter, 0, sizeof(int), s);
  cudaMemsetAsync(a.task_count, 0, sizeof(int), s);
  cudaMemsetAsync(a.member_cursor, 0, sizeof(int), s);
#define SPH_PASS_CASE(M, F)                 \
  launch_form<M, F>(s, a, count, want, num_sms); \
  launch_one<M, F>(s, a, num_sms);
  if (f32) {
    switch (mode) {
      case MODE_HIST: SPH_PASS_CASE(MODE_HIST, true) break;
      case MODE_BAND: SPH_PASS_CASE(MODE_BAND, true) break;
      case MODE_DENS: SPH_PASS_CASE(MODE_DENS, true) break;
      default: SPH_PASS_CASE(MODE_COUNT, true) break;
    }
  } else {
    switch (mode) {
      case MODE_HIST: SPH_PASS_CASE(MODE_HIST, false) break;
      case MODE_BAND: SPH_PASS_CASE(MODE_BAND, false) break;
      case MODE_DENS: SPH_PASS_CASE(MODE_DENS, false) break;
      default: SPH_PASS_CASE(MODE_COUNT, false) break;
    }
  }
#undef SPH_PASS_CASE
}

size_t select_temp_needed(int n) { return scan_temp_bytes(n); }

// list_out = [p in list_in : state[p] == want], order preserved (sph_scan.cu)
void launch_select(cudaStream_t s, const uint32_t *list_in, int n_in, const uint8_t *state, uint8_t want,
                   uint32_t *list_out, int *count_out, void *temp, size_t temp_bytes) {
  (void)temp_bytes;
  select_state(s, list_in, n_in, state, want, list_out, count_out, temp);
}

}  // namespace sph
