// sph_knn.cu -- neighbour sweeps organised as "walk once, sweep narrow".
//
// A super-group (SG) is a spatially coherent set of <= 32 targets (k_form).
// Its warp walks the pre-order tree ONCE, in the search (HIST) phase, with
// one lane per target and each lane's own search radius, and records every
// cell some lane's sphere touches (the list is kept for the later phases:
// select and density radii never exceed the search radius).  Every sweep then
// runs in sub-tasks of 32/LPT targets with LPT lanes per target:
//
//   filter   the recorded cells, 32 at a time (one per lane), against each
//            sub-task target's sphere / bracket (cells wholly below a select
//            bracket are counted without pair tests, one warp reduction per
//            target); the needed cells become contiguous particle ranges
//   stream   candidates through shared memory, 32 per chunk, double
//            buffered; lane s of a target tests candidates j = s (mod LPT)
//   reduce   the LPT partial results of each target (histogram columns,
//            counts, band lists, density sums) in a fixed order
//
// The candidate set of a sub-task is the union of 32/LPT spheres instead of
// 32, and the walk and its per-cell bookkeeping are paid once per SG instead
// of once per sweep.  Per-candidate arithmetic and the fp32-with-fp64-recheck
// exactness argument are those of sph_pass.cu.
#include "sph_internal.cuh"

#include <algorithm>

namespace sph {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 4;
constexpr int LPT = 4;                // lanes per target in a sweep
constexpr int TPW = 32 / LPT;         // targets per sub-task
constexpr int kHistOctaves = 12;
constexpr int kHistBase = (127 - kHistOctaves) << 2;
constexpr int NB_HIST = kHistOctaves * 4 + 2;
constexpr int LANE_BAND_CAP = 8;      // band entries per lane (32 per target)
constexpr int NB_BAND = 16;
constexpr int kScratch = 16384;       // recorded cells per warp
constexpr float kEps = 9.5367431640625e-07f;
constexpr double kEpsD = 9.5367431640625e-07;

struct alignas(32) D4 { double x, y, z, m; };
template <bool F32> struct Stage;
template <> struct Stage<true> { using T = float4; };
template <> struct Stage<false> { using T = D4; };

// per-target data of a sub-task, shared by the filter (one LDS per field)
struct TgtInfo {
  float px, py, pz, r2;    // position (tree frame of the current shift) and sweep radius^2
  float lo_f, pslack, pad0, pad1;
};

template <bool F32>
constexpr int stage_bytes() { return 2 * 32 * (F32 ? 16 : 32) + 4 * 32 * 4; }
constexpr int table_bytes() {
  return (NB_HIST * 32 * 4) > (LANE_BAND_CAP * 32 * 8 + NB_BAND * 32 * 4) ? (NB_HIST * 32 * 4)
                                                                          : (LANE_BAND_CAP * 32 * 8 + NB_BAND * 32 * 4);
}
template <bool F32>
constexpr int warp_smem() { return stage_bytes<F32>() + table_bytes() + TPW * (int)sizeof(TgtInfo); }

__device__ __forceinline__ float warp_min(float v) {
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ float box_gap2(float4 lo, float4 hi, float qlx, float qly, float qlz, float qhx,
                                          float qhy, float qhz) {
  const float gx = fmaxf(fmaxf(lo.x - qhx, qlx - hi.x), 0.f);
  const float gy = fmaxf(fmaxf(lo.y - qhy, qly - hi.y), 0.f);
  const float gz = fmaxf(fmaxf(lo.z - qhz, qlz - hi.z), 0.f);
  return gx * gx + gy * gy + gz * gz;
}
__device__ __forceinline__ double exact_image_d2(double cx, double cy, double cz, bool shifted, double dsx,
                                                 double dsy, double dsz, double tx, double ty, double tz) {
  if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
  return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
}
__device__ __forceinline__ int hist_bin(float x) { return max((__float_as_int(x) >> 21) - kHistBase + 1, 0); }
__device__ __forceinline__ void shift_of(int periodic, int sidx, int &sx, int &sy, int &sz) {
  sx = periodic ? sidx / 9 - 1 : 0;
  sy = periodic ? (sidx / 3) % 3 - 1 : 0;
  sz = periodic ? sidx % 3 - 1 : 0;
}

// ---------------------------------------------------------------------------
// HIST phase walk: one lane per target, radius rad (0 = not walking).  Records
// (node | shift << 27) of every cell some lane's sphere touches, in
// pre-order per shift.  Returns the count, or -1 on overflow.
// ---------------------------------------------------------------------------
__device__ int record_walk(const V3Args &v, double tx, double ty, double tz, float fx, float fy, float fz,
                           bool in, float rad, int *out, int cap) {
  const PassArgs &a = v.a;
  const int lane = threadIdx.x & 31;
  const float4 *__restrict__ nlo = a.tree.nlo;
  const float4 *__restrict__ nhi = a.tree.nhi;
  const int n_nodes = a.tree.n_nodes;
  const bool f32 = v.f32;
  float bx0 = in ? (f32 ? fx : __double2float_rd(tx)) : INFINITY;
  float by0 = in ? (f32 ? fy : __double2float_rd(ty)) : INFINITY;
  float bz0 = in ? (f32 ? fz : __double2float_rd(tz)) : INFINITY;
  float bx1 = in ? (f32 ? fx : __double2float_ru(tx)) : -INFINITY;
  float by1 = in ? (f32 ? fy : __double2float_ru(ty)) : -INFINITY;
  float bz1 = in ? (f32 ? fz : __double2float_ru(tz)) : -INFINITY;
  bx0 = warp_min(bx0); by0 = warp_min(by0); bz0 = warp_min(bz0);
  bx1 = warp_max(bx1); by1 = warp_max(by1); bz1 = warp_max(bz1);
  const float Rb = warp_max(in ? rad : 0.f);
  const float R2b = Rb * Rb * (1.0f + 4.0f * kEps) + 1e-37f;
  const float my_r2 = in ? rad * rad * (1.0f + 4.0f * kEps) + 1e-37f : -1.f;
  int cnt = 0;
  const int n_shift = a.periodic ? 27 : 1;
  for (int s = 0; s < n_shift; ++s) {
    int sx, sy, sz;
    shift_of(a.periodic, s, sx, sy, sz);
    float qlx = bx0, qly = by0, qlz = bz0, qhx = bx1, qhy = by1, qhz = bz1;
    const bool shifted = (sx | sy | sz) != 0;
    if (shifted) {
      const double bxs = a.box;
      qlx = __double2float_rd((double)bx0 - sx * bxs); qhx = __double2float_ru((double)bx1 - sx * bxs);
      qly = __double2float_rd((double)by0 - sy * bxs); qhy = __double2float_ru((double)by1 - sy * bxs);
      qlz = __double2float_rd((double)bz0 - sz * bxs); qhz = __double2float_ru((double)bz1 - sz * bxs);
      if (box_gap2(nlo[0], nhi[0], qlx, qly, qlz, qhx, qhy, qhz) > R2b) continue;
    }
    const double dsx = sx * a.box, dsy = sy * a.box, dsz = sz * a.box;
    const float pqx = shifted ? (float)(tx - dsx) : fx, pqy = shifted ? (float)(ty - dsy) : fy,
                pqz = shifted ? (float)(tz - dsz) : fz;
    const float boxf = (float)a.box;
    const float pslack = shifted ? boxf * 4.8e-7f
                                 : (f32 ? 0.f : fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz))) * 1.2e-7f);
    int kk = 0;
    while (kk < n_nodes) {
      const int w = kk;
      const int my = w + lane;
      bool hit = false;
      int my_skip = n_nodes;
      float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
      if (my < n_nodes) {
        l4 = nlo[my];
        h4 = nhi[my];
        my_skip = __float_as_int(l4.w);
        hit = box_gap2(l4, h4, qlx, qly, qlz, qhx, qhy, qhz) <= R2b;
      }
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
      unsigned pend = hitm & ~covered & cellm;
      while (pend) {
        const int bb = __ffs(pend) - 1;
        pend &= pend - 1u;
        const float cx0 = __shfl_sync(FULL, l4.x, bb), cy0 = __shfl_sync(FULL, l4.y, bb),
                    cz0 = __shfl_sync(FULL, l4.z, bb), cx1 = __shfl_sync(FULL, h4.x, bb),
                    cy1 = __shfl_sync(FULL, h4.y, bb), cz1 = __shfl_sync(FULL, h4.z, bb);
        const float gx = fmaxf(fmaxf(cx0 - pqx, pqx - cx1) - pslack, 0.f);
        const float gy = fmaxf(fmaxf(cy0 - pqy, pqy - cy1) - pslack, 0.f);
        const float gz = fmaxf(fmaxf(cz0 - pqz, pqz - cz1) - pslack, 0.f);
        const bool touch = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= my_r2;
        if (__any_sync(FULL, touch)) {
          if (cnt >= cap) return -1;
          if (lane == 0) out[cnt] = (int)((unsigned)(w + bb) | ((unsigned)s << 27));
          ++cnt;
        }
      }
    }
  }
  return cnt;
}

// ---------------------------------------------------------------------------
// One sweep of MODE over a recorded cell list for one sub-task.
// ---------------------------------------------------------------------------
template <int MODE, bool F32>
struct Sub {
  // lane's target (t = lane / LPT) and its state
  int p;
  bool tv;                   // this lane's target slot is occupied
  double tx, ty, tz;
  float fx, fy, fz;
  // HIST
  float hR2, h_r2, h_inv;
  int seen;
  // BAND
  double lo, hi, scale, emin, emax;
  float lo_f, hi_f;
  int c_below, n_in;
  // DENS
  double d2k, hh, norm_h3, accd;
  float d2k_f, inv_h, accf;
  float rad;
};

template <int MODE, bool F32>
__device__ __forceinline__ void sweep_list(const V3Args &v, Sub<MODE, F32> &S, const int *list, int nlist,
                                           unsigned char *wbase, unsigned long long &tests,
                                           unsigned long long &accepted) {
  using StageT = typename Stage<F32>::T;
  const PassArgs &a = v.a;
  const int lane = threadIdx.x & 31;
  const int t = lane / LPT, sl = lane % LPT;
  StageT *stage = reinterpret_cast<StageT *>(wbase);
  int *sidxbuf = reinterpret_cast<int *>(wbase + 2 * 32 * sizeof(StageT));
  int *spfx = sidxbuf + 64;
  int *srsm = spfx + 32;
  unsigned char *tb = wbase + stage_bytes<F32>();
  unsigned *hist = reinterpret_cast<unsigned *>(tb);
  double *band = reinterpret_cast<double *>(tb);
  unsigned *bh = reinterpret_cast<unsigned *>(tb + LANE_BAND_CAP * 32 * 8);
  TgtInfo *ti = reinterpret_cast<TgtInfo *>(tb + table_bytes());
  const StageT *__restrict__ pos = reinterpret_cast<const StageT *>(a.pos);
  const float4 *__restrict__ nlo = a.tree.nlo;
  const float4 *__restrict__ nhi = a.tree.nhi;
  const int n_nodes = a.tree.n_nodes;
  const int n = a.n;
  const unsigned tmask = __ballot_sync(FULL, S.tv && sl == 0);  // bit t*LPT per occupied target
  const int ntg = __popc(tmask);
  if (!ntg) return;
  const float boxf = (float)a.box;

  int rs = 0, re = 0, nr = 0, last_e = -1;
  int cur_shift = -1;
  bool shifted = false;
  float csx = 0.f, csy = 0.f, csz = 0.f, tfx = S.fx, tfy = S.fy, tfz = S.fz;
  double dsx = 0.0, dsy = 0.0, dsz = 0.0;

  auto set_shift = [&](int sidx) {
    cur_shift = sidx;
    int sx, sy, sz;
    shift_of(a.periodic, sidx, sx, sy, sz);
    shifted = (sx | sy | sz) != 0;
    csx = sx < 0 ? -boxf : 0.f; csy = sy < 0 ? -boxf : 0.f; csz = sz < 0 ? -boxf : 0.f;
    tfx = sx > 0 ? S.fx - boxf : S.fx; tfy = sy > 0 ? S.fy - boxf : S.fy; tfz = sz > 0 ? S.fz - boxf : S.fz;
    dsx = sx * a.box; dsy = sy * a.box; dsz = sz * a.box;
    // per-target filter data in the tree frame of this shift
    __syncwarp();
    if (S.tv && sl == 0) {
      TgtInfo g;
      g.px = shifted ? (float)(S.tx - dsx) : S.fx;
      g.py = shifted ? (float)(S.ty - dsy) : S.fy;
      g.pz = shifted ? (float)(S.tz - dsz) : S.fz;
      float r2;
      if constexpr (MODE == MODE_HIST) r2 = S.h_r2;
      else if constexpr (MODE == MODE_BAND) r2 = S.hi_f;
      else r2 = S.d2k_f;
      g.r2 = r2 * (1.0f + 4.0f * kEps) + 1e-37f;
      g.lo_f = MODE == MODE_BAND ? S.lo_f : -1.f;
      g.pslack = shifted ? boxf * 4.8e-7f
                         : (F32 ? 0.f : fmaxf(fabsf(S.fx), fmaxf(fabsf(S.fy), fabsf(S.fz))) * 1.2e-7f);
      g.pad0 = g.pad1 = 0.f;
      ti[t] = g;
    }
    __syncwarp();
  };

  auto flush = [&]() {
    const int len = lane < nr ? re - rs : 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vv = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += vv;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    spfx[lane] = incl;
    srsm[lane] = rs - (incl - len);
    __syncwarp();
    auto cand_of = [&](int s) -> int {
      int r = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1)
        if (spfx[r + step - 1] <= s) r += step;
      return srsm[r] + s;
    };
    int my_ci = lane < total ? cand_of(lane) : 0;
    StageT v_cur;
    if (lane < total) v_cur = pos[my_ci];
    const float e_lo_f = S.tv ? S.lo_f : -1.f, e_hi_f = S.tv ? S.hi_f : -2.f;
    const float e_d2k_f = S.tv ? S.d2k_f : -1.f;
    const double e_d2k = S.tv ? S.d2k : -1.0;
    const float h_r2 = S.tv ? S.h_r2 : -1.f;
    const double h_r2d = (double)h_r2, h_invd = (double)S.h_inv;
    for (int c0 = 0; c0 < total; c0 += 32) {
      StageT *stb = stage + ((c0 >> 5) & 1) * 32;
      int *sti = sidxbuf + ((c0 >> 5) & 1) * 32;
      const int nc = min(32, total - c0);
      if (lane < nc) { stb[lane] = v_cur; sti[lane] = my_ci; }
      __syncwarp();
      if (c0 + 32 + lane < total) {
        my_ci = cand_of(c0 + 32 + lane);
        v_cur = pos[my_ci];
      }
      tests += (unsigned long long)nc * ntg;
#pragma unroll 2
      for (int j = sl; j < nc; j += LPT) {
        const StageT c = stb[j];
        const int cidx = sti[j];
        float af = 0.f;
        double ad = 0.0;
        if constexpr (F32) {
          float dx, dy, dz;
          if (shifted) {
            dx = (c.x + csx) - tfx; dy = (c.y + csy) - tfy; dz = (c.z + csz) - tfz;
          } else {
            dx = c.x - S.fx; dy = c.y - S.fy; dz = c.z - S.fz;
          }
          af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        } else {
          double cx = c.x, cy = c.y, cz = c.z;
          if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
          ad = exact_d2(__dsub_rn(cx, S.tx), __dsub_rn(cy, S.ty), __dsub_rn(cz, S.tz));
        }
#define SPH_EXACT() exact_image_d2((double)c.x, (double)c.y, (double)c.z, shifted, dsx, dsy, dsz, S.tx, S.ty, S.tz)
        if constexpr (MODE == MODE_HIST) {
          bool inr;
          float x;
          if constexpr (F32) { inr = af <= h_r2; x = af * S.h_inv; }
          else { inr = ad <= h_r2d; x = (float)(ad * h_invd); }
          if (inr) {
            hist[hist_bin(x) * 32 + lane] += 1u;
            ++S.seen;
          }
        } else if constexpr (MODE == MODE_BAND) {
          if (!((cidx == S.p) && !shifted)) {
            double e = -1.0;
            if constexpr (F32) {
              if (af < e_lo_f) ++S.c_below;
              else if (af <= e_hi_f) e = SPH_EXACT();
            } else {
              e = S.tv ? ad : -1.0;
            }
            if (e >= 0.0) {
              if (e < S.lo) ++S.c_below;
              else if (e <= S.hi) {
                if (S.n_in < LANE_BAND_CAP) band[S.n_in * 32 + lane] = e;
                ++S.n_in;
                S.emin = fmin(S.emin, e);
                S.emax = fmax(S.emax, e);
                const int bin = min(max((int)((e - S.lo) * S.scale), 0), NB_BAND - 1);
                bh[bin * 32 + lane] += 1u;
              }
            }
          }
        } else {  // DENS
          if constexpr (F32) {
            if (af < e_d2k_f) {
              if (a.dens64) {
                const double e = SPH_EXACT();
                if (e < S.d2k) {
                  const double r_ = __dsqrt_rn(e);
                  double w;
                  if (a.kernel_kind == 0) {
                    w = wc6_lowered(r_, S.hh, S.norm_h3);
                  } else {
                    const double q = __ddiv_rn(r_, S.hh);
                    w = q < 1.0 ? S.norm_h3 * m4_profile(q) : 0.0;
                  }
                  S.accd = __dadd_rn(S.accd, __dmul_rn(a.mass64[cidx], w));
                }
              } else {
                const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
                const float q = rr * S.inv_h;
                const float w = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
                if (q < 1.f) S.accf = fmaf(c.w, w, S.accf);
              }
              ++accepted;
            }
          } else {
            if (ad < e_d2k) {
              const double r_ = __dsqrt_rn(ad);
              double w;
              if (a.kernel_kind == 0) {
                w = wc6_lowered(r_, S.hh, S.norm_h3);
              } else {
                const double q = __ddiv_rn(r_, S.hh);
                w = q < 1.0 ? S.norm_h3 * m4_profile(q) : 0.0;
              }
              S.accd = __dadd_rn(S.accd, __dmul_rn(c.m, w));
              ++accepted;
            }
          }
        }
#undef SPH_EXACT
      }
    }
    __syncwarp();
    nr = 0;
    last_e = -1;
    if constexpr (MODE == MODE_HIST) {
      // adaptive shrink: the target's K-th so far bounds its radius
      int seen_t = S.seen;
      for (int o = 1; o < LPT; o <<= 1) seen_t += __shfl_xor_sync(FULL, seen_t, o);
      if (S.tv && seen_t > a.k) {
        int cum = 0, bb = 0;
        const int base = t * LPT;
        for (; bb < NB_HIST; ++bb) {
          const unsigned *row = hist + bb * 32 + base;
          int rowsum = 0;
#pragma unroll
          for (int q = 0; q < LPT; ++q) rowsum += (int)row[q];
          cum += rowsum;
          if (cum > a.k) break;
        }
        if (bb < NB_HIST - 1) {
          const float edge = __int_as_float((kHistBase + bb) << 21) * S.hR2 * (1.0f + 4.0f * kEps);
          S.h_r2 = fminf(S.h_r2, edge);
        }
      }
      __syncwarp();
      if (S.tv && sl == 0) ti[t].r2 = S.h_r2 * (1.0f + 4.0f * kEps) + 1e-37f;
      __syncwarp();
    }
  };

  // ---- filter the recorded cells (one per lane) against every target ----
  for (int c0 = 0; c0 < nlist; c0 += 32) {
    const int nc = min(32, nlist - c0);
    int code = 0, node = 0, cs = n, ce = n, csh = 0;
    float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
    if (lane < nc) {
      code = list[c0 + lane];
      node = code & ((1 << 27) - 1);
      csh = (int)((unsigned)code >> 27);
      l4 = nlo[node];
      h4 = nhi[node];
      cs = __float_as_int(h4.w);
      ce = node + 1 < n_nodes ? __float_as_int(nhi[node + 1].w) : n;
    }
    // cells of one shift at a time (lists are recorded shift by shift)
    unsigned todo = __ballot_sync(FULL, lane < nc);
    while (todo) {
      const int first = __ffs(todo) - 1;
      const int sh = __shfl_sync(FULL, csh, first);
      const bool mine = ((todo >> lane) & 1u) && csh == sh;
      todo &= ~__ballot_sync(FULL, mine);
      if (sh != cur_shift) {
        if (nr) flush();
        set_shift(sh);
      }
      unsigned needm = 0u;   // bit t: target t needs this cell's particles
      unsigned belowm = 0u;  // bit t: the cell lies wholly below target t's select bracket
      for (int tt = 0; tt < TPW; ++tt) {
        if (!((tmask >> (tt * LPT)) & 1u)) continue;
        const TgtInfo g = ti[tt];
        const float gx = fmaxf(fmaxf(l4.x - g.px, g.px - h4.x) - g.pslack, 0.f);
        const float gy = fmaxf(fmaxf(l4.y - g.py, g.py - h4.y) - g.pslack, 0.f);
        const float gz = fmaxf(fmaxf(l4.z - g.pz, g.pz - h4.z) - g.pslack, 0.f);
        const float gap2 = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps);
        bool need = mine && gap2 <= g.r2;
        if constexpr (MODE == MODE_BAND) {
          const float fxa = fmaxf(g.px - l4.x, h4.x - g.px) + g.pslack;
          const float fya = fmaxf(g.py - l4.y, h4.y - g.py) + g.pslack;
          const float fza = fmaxf(g.pz - l4.z, h4.z - g.pz) + g.pslack;
          const float dmax2 = (fxa * fxa + fya * fya + fza * fza) * (1.0f + 4.0f * kEps);
          if (need && dmax2 < g.lo_f) {
            belowm |= 1u << tt;
            need = false;
          }
        }
        if (need) needm |= 1u << tt;
      }
      if constexpr (MODE == MODE_BAND) {
        // a cell every sub-task target either skips or has wholly below its
        // bracket is counted from its box; if any target needs its particles,
        // all targets test them (no double counting)
        const bool use_sc = needm == 0u;
        if (!use_sc) belowm = 0u;
        if (__any_sync(FULL, belowm != 0u)) {
          for (int tt = 0; tt < TPW; ++tt) {
            if (!((tmask >> (tt * LPT)) & 1u)) continue;
            const int p_t = __shfl_sync(FULL, S.p, tt * LPT);
            int add = 0;
            if ((belowm >> tt) & 1u)
              add = (ce - cs) - ((sh == (a.periodic ? 13 : 0)) && cs <= p_t && p_t < ce ? 1 : 0);
            const int tot = (int)__reduce_add_sync(FULL, (unsigned)add);
            if (lane == tt * LPT) S.c_below += tot;
          }
        }
      }
      // append needed cells in list order (merging contiguous ones)
      unsigned nm = __ballot_sync(FULL, needm != 0u);
      while (nm) {
        const int bb = __ffs(nm) - 1;
        nm &= nm - 1u;
        const int s0 = __shfl_sync(FULL, cs, bb), e0 = __shfl_sync(FULL, ce, bb);
        if (s0 == last_e) {
          if (lane == nr - 1) re = e0;
        } else {
          if (nr == 32) flush();
          if (lane == nr) { rs = s0; re = e0; }
          ++nr;
        }
        last_e = e0;
      }
    }
  }
  if (nr) flush();
}

template <int MODE, bool F32>
__global__ void __launch_bounds__(kWarps * 32) k_v3(const V3Args v) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  const PassArgs &a = v.a;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *wbase = smem_raw + wib * warp_smem<F32>();
  unsigned char *tb = wbase + stage_bytes<F32>();
  unsigned *hist = reinterpret_cast<unsigned *>(tb);
  double *band = reinterpret_cast<double *>(tb);
  unsigned *bh = reinterpret_cast<unsigned *>(tb + LANE_BAND_CAP * 32 * 8);
  int *scratch = v.scratch + (size_t)(blockIdx.x * kWarps + wib) * kScratch;
  const int K = a.k;
  unsigned long long tests = 0, accepted = 0;

  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(a.work_counter, 1);
    b = __shfl_sync(FULL, b, 0);
    if (b >= *v.sg_count) break;
    const int sgi = v.sg_begin + b;
    int4 sg = v.sgs[sgi];
    const bool mem = lane < sg.y;
    const int p = mem ? (int)v.members[sg.x + lane] : 0;
    bool valid = false;
    if (mem) {
      const uint8_t st = a.state[p];
      if constexpr (MODE == MODE_HIST) valid = st == ST_NEED_HIST;
      else if constexpr (MODE == MODE_BAND) valid = st == ST_NEED_BAND && v.owner[p] == sgi;
      else valid = st == ST_DONE && v.owner[p] == sgi;
    }
    unsigned vmask = __ballot_sync(FULL, valid);
    if (!vmask) continue;

    const int *list;
    int nlist;
    if constexpr (MODE == MODE_HIST) {
      // the one walk of this group: each lane its own radius
      double tx = 0, ty = 0, tz = 0;
      float fx = 0, fy = 0, fz = 0;
      const int p_first = __shfl_sync(FULL, p, __ffs(vmask) - 1);
      const int pp = valid ? p : p_first;
      if constexpr (F32) {
        const float4 q = reinterpret_cast<const float4 *>(a.pos)[pp];
        fx = q.x; fy = q.y; fz = q.z; tx = q.x; ty = q.y; tz = q.z;
      } else {
        const D4 q = reinterpret_cast<const D4 *>(a.pos)[pp];
        tx = q.x; ty = q.y; tz = q.z; fx = (float)tx; fy = (float)ty; fz = (float)tz;
      }
      const float rad = valid ? a.radius[p] : 0.f;
      nlist = record_walk(v, tx, ty, tz, fx, fy, fz, valid, rad, scratch, kScratch);
      if (nlist < 0) {
        // too many cells for the scratch list: these targets take the round-by-round path
        if (valid) a.state[p] = ST_LEGACY;
        if (lane == 0) atomicAdd(v.legacy_count, __popc(vmask));
        continue;
      }
      // keep the list for the select and density phases
      int off = 0;
      if (lane == 0) off = atomicAdd(v.list_cursor, nlist);
      off = __shfl_sync(FULL, off, 0);
      if (off + nlist <= v.list_cap) {
        for (int i = lane; i < nlist; i += 32) v.list_pool[off + i] = scratch[i];
        if (lane == 0) v.sgs[sgi] = make_int4(sg.x, sg.y, off, nlist);
      } else if (lane == 0) {
        v.sgs[sgi] = make_int4(sg.x, sg.y, -1, 0);
      }
      __syncwarp();
      list = scratch;
    } else {
      if (sg.z < 0) {
        // no stored list: walk again with the phase radius
        double tx = 0, ty = 0, tz = 0;
        float fx = 0, fy = 0, fz = 0;
        const int p_first = __shfl_sync(FULL, p, __ffs(vmask) - 1);
      const int pp = valid ? p : p_first;
        if constexpr (F32) {
          const float4 q = reinterpret_cast<const float4 *>(a.pos)[pp];
          fx = q.x; fy = q.y; fz = q.z; tx = q.x; ty = q.y; tz = q.z;
        } else {
          const D4 q = reinterpret_cast<const D4 *>(a.pos)[pp];
          tx = q.x; ty = q.y; tz = q.z; fx = (float)tx; fy = (float)ty; fz = (float)tz;
        }
        float rad = 0.f;
        if (valid) rad = MODE == MODE_BAND ? (float)(sqrt(a.t_hi[p]) * (1.0 + 2.0 * kEpsD)) + 1e-30f
                                           : (float)(sqrt(a.d2k[p]) * (1.0 + 2.0 * kEpsD)) + 1e-30f;
        nlist = record_walk(v, tx, ty, tz, fx, fy, fz, valid, rad, scratch, kScratch);
        if (nlist < 0) {
          if (valid) a.state[p] = ST_LEGACY;
          if (lane == 0) atomicAdd(v.legacy_count, __popc(vmask));
          continue;
        }
        list = scratch;
      } else {
        list = v.list_pool + sg.z;
        nlist = sg.w;
      }
    }

    // ---- sub-tasks of TPW targets, LPT lanes each ----
    while (vmask) {
      unsigned sub = 0u;
      {
        unsigned mm = vmask;
        for (int i = 0; i < TPW && mm; ++i) {
          sub |= mm & (0u - mm);
          mm &= mm - 1u;
        }
      }
      vmask &= ~sub;
      const int t = lane / LPT, sl = lane % LPT;
      const int nsub = __popc(sub);
      Sub<MODE, F32> S;
      S.tv = t < nsub;
      const int ml = S.tv ? (int)__fns(sub, 0, t + 1) : 0;
      S.p = __shfl_sync(FULL, p, ml);
      if constexpr (F32) {
        const float4 q = reinterpret_cast<const float4 *>(a.pos)[S.p];
        S.fx = q.x; S.fy = q.y; S.fz = q.z; S.tx = q.x; S.ty = q.y; S.tz = q.z;
      } else {
        const D4 q = reinterpret_cast<const D4 *>(a.pos)[S.p];
        S.tx = q.x; S.ty = q.y; S.tz = q.z; S.fx = (float)S.tx; S.fy = (float)S.ty; S.fz = (float)S.tz;
      }
      S.seen = 0; S.c_below = 0; S.n_in = 0; S.emin = INFINITY; S.emax = -INFINITY;
      S.lo = 0.0; S.hi = -1.0; S.scale = 0.0; S.lo_f = -1.f; S.hi_f = -2.f;
      S.hR2 = 0.f; S.h_r2 = -1.f; S.h_inv = 0.f;
      S.d2k = 0.0; S.hh = 0.0; S.norm_h3 = 0.0; S.accd = 0.0; S.d2k_f = -1.f; S.inv_h = 0.f; S.accf = 0.f;
      S.rad = 0.f;
      if constexpr (MODE == MODE_HIST) {
#pragma unroll
        for (int bb = 0; bb < NB_HIST; ++bb) hist[bb * 32 + lane] = 0u;
        if (S.tv) {
          const float R = a.radius[S.p];
          S.hR2 = R * R;
          S.h_r2 = S.hR2;
          S.h_inv = 1.0f / S.hR2;
        }
      } else if constexpr (MODE == MODE_BAND) {
#pragma unroll
        for (int bb = 0; bb < NB_BAND; ++bb) bh[bb * 32 + lane] = 0u;
        if (S.tv) {
          S.lo = a.t_lo[S.p];
          S.hi = a.t_hi[S.p];
          S.scale = S.hi > S.lo ? (double)NB_BAND / (S.hi - S.lo) : 0.0;
          S.lo_f = __double2float_rd(S.lo * (1.0 - kEpsD)) - 1e-37f;
          S.hi_f = __double2float_ru(S.hi * (1.0 + kEpsD)) + 1e-37f;
        }
      } else {
        if (S.tv) {
          S.d2k = a.d2k[S.p];
          S.hh = __dsqrt_rn(S.d2k);
          S.norm_h3 = __ddiv_rn(a.kernel_kind == 0 ? kWc6Norm : kM4Norm, __dmul_rn(__dmul_rn(S.hh, S.hh), S.hh));
          S.d2k_f = __double2float_ru(S.d2k * (1.0 + kEpsD));
          S.inv_h = (float)(1.0 / S.hh);
        }
      }
      __syncwarp();
      sweep_list<MODE, F32>(v, S, list, nlist, wbase, tests, accepted);
      __syncwarp();

      // ---- reduce the LPT lanes of each target and finish ----
      const int base = t * LPT;
      if constexpr (MODE == MODE_HIST) {
        if (S.tv && sl == 0) {
          unsigned total = 0;
          for (int bb = 0; bb < NB_HIST; ++bb)
            for (int q = 0; q < LPT; ++q) total += hist[bb * 32 + base + q];
          total -= 1u;  // the target itself
          const float Rused = sqrtf(S.hR2);
          if ((int)total < K) {
            if (Rused >= a.rmax) {
              a.state[S.p] = ST_UNREACHABLE;
              a.d2k[S.p] = INFINITY;
            } else {
              // grow: the next round groups this target anew
              float f = total > 0 ? cbrtf((float)(K + 8) / (float)total) * 1.15f : 2.f;
              f = fminf(fmaxf(f, 1.26f), 2.5f);
              a.radius[S.p] = fminf(Rused * f, a.rmax);
            }
          } else {
            int cum = 0, bb = 0;
            for (; bb < NB_HIST; ++bb) {
              int hc = 0;
              for (int q = 0; q < LPT; ++q) hc += (int)hist[bb * 32 + base + q];
              if (bb == 0) hc -= 1;
              if (cum + hc >= K) break;
              cum += hc;
            }
            const double R2d = (double)S.hR2;
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
            a.t_lo[S.p] = tl;
            a.t_hi[S.p] = th;
            a.state[S.p] = ST_NEED_BAND;
            v.owner[S.p] = sgi;
          }
        }
      } else if constexpr (MODE == MODE_BAND) {
        int cb = S.c_below, ni = S.n_in, ovf = S.n_in > LANE_BAND_CAP ? 1 : 0;
        double emn = S.emin, emx = S.emax;
        for (int o = 1; o < LPT; o <<= 1) {
          cb += __shfl_xor_sync(FULL, cb, o);
          ni += __shfl_xor_sync(FULL, ni, o);
          ovf |= __shfl_xor_sync(FULL, ovf, o);
          emn = fmin(emn, __shfl_xor_sync(FULL, emn, o));
          emx = fmax(emx, __shfl_xor_sync(FULL, emx, o));
        }
        int nq[LPT];
#pragma unroll
        for (int q = 0; q < LPT; ++q) nq[q] = __shfl_sync(FULL, S.n_in, base + q);
        // rank-r value of the target's in-bracket entries: every lane ranks its
        // own entries against all of the target's, then a min over the lanes
        double sel_out = INFINITY;
        {
          const int r = K - cb;
          if (S.tv && !ovf && r >= 1 && r <= ni) {
            for (int ia = 0; ia < min(S.n_in, LANE_BAND_CAP); ++ia) {
              const double ei = band[ia * 32 + lane];
              int less = 0, eq = 0;
              for (int qb = 0; qb < LPT; ++qb)
                for (int ib = 0; ib < nq[qb]; ++ib) {
                  const double ej = band[ib * 32 + base + qb];
                  less += ej < ei;
                  eq += ej == ei;
                }
              if (less < r && r <= less + eq) sel_out = fmin(sel_out, ei);
            }
          }
          for (int o = 1; o < LPT; o <<= 1) sel_out = fmin(sel_out, __shfl_xor_sync(FULL, sel_out, o));
        }
        if (S.tv && sl == 0) {
          const int r = K - cb;  // 1-based rank inside the bracket
          if (r <= 0) {
            a.t_hi[S.p] = nextafter(S.lo, -INFINITY);
            a.t_lo[S.p] = 0.0;
          } else if (r > ni) {
            const float Rr = a.radius[S.p];
            a.t_lo[S.p] = nextafter(S.hi, INFINITY);
            a.t_hi[S.p] = (double)Rr * (double)Rr * (1.0 + 16.0 * kEpsD);
          } else if (!ovf) {
            a.d2k[S.p] = sel_out;
            a.state[S.p] = ST_DONE;
          } else if (emn == emx) {
            a.d2k[S.p] = emn;
            a.state[S.p] = ST_DONE;
          } else {
            int cum = 0, bb = 0;
            for (; bb < NB_BAND; ++bb) {
              int hc = 0;
              for (int q = 0; q < LPT; ++q) hc += (int)bh[bb * 32 + base + q];
              if (cum + hc >= r) break;
              cum += hc;
            }
            bb = min(bb, NB_BAND - 1);
            const double width = S.hi - S.lo;
            double nl = bb == 0 ? S.lo : S.lo + (double)bb / S.scale - width * 1e-12;
            double nh = bb == NB_BAND - 1 ? S.hi : S.lo + (double)(bb + 1) / S.scale + width * 1e-12;
            nl = fmax(nextafter(nl, -INFINITY), fmax(S.lo, emn));
            nh = fmin(nextafter(nh, INFINITY), fmin(S.hi, emx));
            a.t_lo[S.p] = nl;
            a.t_hi[S.p] = nh;
          }
        }
      } else {  // DENS
        double accd = S.accd;
        float accf = S.accf;
        for (int o = 1; o < LPT; o <<= 1) {
          accd = __dadd_rn(accd, __shfl_xor_sync(FULL, accd, o));
          accf += __shfl_xor_sync(FULL, accf, o);
        }
        if (S.tv && sl == 0) {
          a.rho[S.p] = (F32 && !a.dens64) ? __dmul_rn(S.norm_h3, (double)accf) : accd;
          a.state[S.p] = ST_FINAL;
        }
      }
      __syncwarp();
    }
  }
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
  }
}

template <int MODE, bool F32>
int v3_blocks(int num_sms) {
  static int bps = 0;
  if (!bps) {
    cudaFuncSetAttribute(k_v3<MODE, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarps * warp_smem<F32>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_v3<MODE, F32>, kWarps * 32, kWarps * warp_smem<F32>());
    if (bps < 1) bps = 1;
  }
  return num_sms * bps;
}

}  // namespace

size_t v3_scratch_ints(int num_sms) {
  int m = 0;
  m = std::max(m, v3_blocks<MODE_HIST, true>(num_sms));
  m = std::max(m, v3_blocks<MODE_BAND, true>(num_sms));
  m = std::max(m, v3_blocks<MODE_DENS, true>(num_sms));
  m = std::max(m, v3_blocks<MODE_HIST, false>(num_sms));
  m = std::max(m, v3_blocks<MODE_BAND, false>(num_sms));
  m = std::max(m, v3_blocks<MODE_DENS, false>(num_sms));
  return (size_t)m * kWarps * kScratch;
}

void launch_v3(cudaStream_t s, int mode, const V3Args &v, int num_sms) {
  cudaMemsetAsync(v.a.work_counter, 0, sizeof(int), s);
  const int smem32 = kWarps * warp_smem<true>(), smem64 = kWarps * warp_smem<false>();
  if (v.f32) {
    if (mode == MODE_HIST) k_v3<MODE_HIST, true><<<v3_blocks<MODE_HIST, true>(num_sms), kWarps * 32, smem32, s>>>(v);
    else if (mode == MODE_BAND) k_v3<MODE_BAND, true><<<v3_blocks<MODE_BAND, true>(num_sms), kWarps * 32, smem32, s>>>(v);
    else k_v3<MODE_DENS, true><<<v3_blocks<MODE_DENS, true>(num_sms), kWarps * 32, smem32, s>>>(v);
  } else {
    if (mode == MODE_HIST) k_v3<MODE_HIST, false><<<v3_blocks<MODE_HIST, false>(num_sms), kWarps * 32, smem64, s>>>(v);
    else if (mode == MODE_BAND) k_v3<MODE_BAND, false><<<v3_blocks<MODE_BAND, false>(num_sms), kWarps * 32, smem64, s>>>(v);
    else k_v3<MODE_DENS, false><<<v3_blocks<MODE_DENS, false>(num_sms), kWarps * 32, smem64, s>>>(v);
  }
}

}  // namespace sph
