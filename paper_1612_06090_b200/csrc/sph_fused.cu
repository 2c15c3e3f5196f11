// sph_fused.cu -- the density pass as one persistent kernel over target tasks.
//
// A task is a spatially coherent group of <= 32 targets (k_form); one warp
// owns it from start to finish, one target per lane:
//
//   search   radius R_i (tree density estimate, biased low); per-lane
//            geometric histogram of d^2 over [0, R_i^2]; lanes with fewer
//            than K neighbours grow R_i from their count and go again
//            (the reference's grow-until-K loop, density.py:226-230, but
//            per lane and without a host round trip)
//   select   the K-th smallest d^2 exactly: count what lies below the
//            histogram bracket, keep the bracket's values (unfused fp64),
//            pick rank K; overfull brackets are split and re-swept
//   density  rho_i = sum_j m_j W(r_ij, h_i), h_i = sqrt(d2_K)
//
// Each sweep walks the pre-order search tree (stackless, 32 nodes box-tested
// per step, one per lane), classifies every cell the group's box touches
// against every lane's own sphere and thresholds from the cell box alone
// (outside / wholly below the bracket / wholly inside one histogram bin:
// counted without pair tests), and streams the particles of the remaining
// cells through shared memory, 32 at a time, double-buffered.  The select
// sweep records the cells it touched so that bracket refinements and the
// density sweep replay the list instead of walking again.
#include "sph_internal.cuh"

#include <algorithm>

namespace sph {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 4;
constexpr int kHistOctaves = 12;
constexpr int kHistBase = (127 - kHistOctaves) << 2;
constexpr int NB_HIST = kHistOctaves * 4 + 2;
constexpr int BAND_CAP = 32;
constexpr int NB_BAND = 16;
constexpr int kCellList = 4096;       // recorded cells per warp (global scratch)
constexpr int kMaxSearchRounds = 24;
constexpr int kMaxBandRounds = 48;
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard
constexpr double kEpsD = 9.5367431640625e-07;

enum : int { L_NONE = 0, L_HIST = 1, L_BAND = 2, L_DONE = 3, L_UNREACH = 4 };
enum : int { SW_HIST = 0, SW_BAND = 1, SW_DENS = 2 };

struct alignas(32) D4 { double x, y, z, m; };
template <bool F32> struct Stage;
template <> struct Stage<true> { using T = float4; };
template <> struct Stage<false> { using T = D4; };

template <bool F32>
constexpr int stage_bytes() { return 2 * 32 * (F32 ? 16 : 32) + 4 * 32 * 4; }
constexpr int table_bytes() {
  return (BAND_CAP * 32 * 8 + NB_BAND * 32 * 4) > (NB_HIST * 32 * 4) ? (BAND_CAP * 32 * 8 + NB_BAND * 32 * 4)
                                                                     : (NB_HIST * 32 * 4);
}
template <bool F32>
constexpr int warp_smem() { return stage_bytes<F32>() + table_bytes(); }

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
__device__ __forceinline__ int hist_bin(float x) {
  return min(max((__float_as_int(x) >> 21) - kHistBase + 1, 0), NB_HIST - 1);
}

// Per-lane state of one task.  Everything a sweep needs lives here so the
// sweep body can be written once per mode.
struct Lane {
  int p;
  bool member;
  double tx, ty, tz;
  float fx, fy, fz;
  int status;
  float R;          // search radius (search phase)
  float hR2, h_inv; // histogram range of the current search sweep
  // select
  double lo, hi, scale, emin, emax;
  float lo_f, hi_f;
  int c_below, n_in;
  // density
  double d2k, hh, norm_h3, accd;
  float d2k_f, inv_h, accf;
  // sweep
  bool in_sweep;    // this lane takes part in the current sweep
  float rad;        // its radius in the current sweep
};

template <bool F32>
struct Smem {
  typename Stage<F32>::T *stage;
  int *sidx, *spfx, *srsm;
  unsigned *hist;   // [NB_HIST][32]
  double *band;     // [BAND_CAP][32]
  unsigned *bh;     // [NB_BAND][32]
};

// One sweep over the cells reachable from the task's lanes in the sweep.
// Source: a tree walk (optionally recording the touched cells) or the list
// recorded by an earlier walk.
template <int SW, bool F32>
__device__ __forceinline__ void sweep(const FusedArgs &a, Lane &L, const Smem<F32> &sm, bool from_list,
                                      bool record, int *cell_list, int &n_cells, bool &list_ok,
                                      unsigned long long &tests, unsigned long long &accepted) {
  using StageT = typename Stage<F32>::T;
  const int lane = threadIdx.x & 31;
  const StageT *__restrict__ pos = reinterpret_cast<const StageT *>(a.pos);
  const float4 *__restrict__ nlo = a.nlo;
  const float4 *__restrict__ nhi = a.nhi;
  const int n_nodes = a.n_nodes;
  const int n = a.n;
  const unsigned smask = __ballot_sync(FULL, L.in_sweep);
  if (!smask) return;
  const int n_mem = __popc(smask);

  // group box and radius
  const bool in = L.in_sweep;
  float bx0 = in ? (F32 ? L.fx : __double2float_rd(L.tx)) : INFINITY;
  float by0 = in ? (F32 ? L.fy : __double2float_rd(L.ty)) : INFINITY;
  float bz0 = in ? (F32 ? L.fz : __double2float_rd(L.tz)) : INFINITY;
  float bx1 = in ? (F32 ? L.fx : __double2float_ru(L.tx)) : -INFINITY;
  float by1 = in ? (F32 ? L.fy : __double2float_ru(L.ty)) : -INFINITY;
  float bz1 = in ? (F32 ? L.fz : __double2float_ru(L.tz)) : -INFINITY;
  bx0 = warp_min(bx0); by0 = warp_min(by0); bz0 = warp_min(bz0);
  bx1 = warp_max(bx1); by1 = warp_max(by1); bz1 = warp_max(bz1);
  const float Rb = warp_max(in ? L.rad : 0.f);
  const float R2b = Rb * Rb * (1.0f + 4.0f * kEps) + 1e-37f;
  const float my_r2 = in ? L.rad * L.rad * (1.0f + 4.0f * kEps) + 1e-37f : -1.f;

  // effective thresholds (non-participants: none)
  const float h_r2 = in ? L.hR2 : -1.f;
  const float h_inv = L.h_inv;
  const double h_r2d = (double)h_r2, h_invd = (double)h_inv;
  const float e_lo_f = in ? L.lo_f : -1.f, e_hi_f = in ? L.hi_f : -2.f;
  const float e_d2k_f = in ? L.d2k_f : -1.f;
  const double e_d2k = in ? L.d2k : -1.0;

  const float boxf = (float)a.box;
  int rs = 0, re = 0, nr = 0, last_e = -1;
  int cur_shift = -1;
  // shift-dependent values (recomputed when the shift changes)
  bool shifted = false;
  float csx = 0.f, csy = 0.f, csz = 0.f, tfx = L.fx, tfy = L.fy, tfz = L.fz;
  double dsx = 0.0, dsy = 0.0, dsz = 0.0;
  float pqx = L.fx, pqy = L.fy, pqz = L.fz, pslack = 0.f;
  auto set_shift = [&](int sidx) {
    cur_shift = sidx;
    const int sx = a.periodic ? sidx / 9 - 1 : 0;
    const int sy = a.periodic ? (sidx / 3) % 3 - 1 : 0;
    const int sz = a.periodic ? sidx % 3 - 1 : 0;
    shifted = (sx | sy | sz) != 0;
    csx = sx < 0 ? -boxf : 0.f; csy = sy < 0 ? -boxf : 0.f; csz = sz < 0 ? -boxf : 0.f;
    tfx = sx > 0 ? L.fx - boxf : L.fx; tfy = sy > 0 ? L.fy - boxf : L.fy; tfz = sz > 0 ? L.fz - boxf : L.fz;
    dsx = sx * a.box; dsy = sy * a.box; dsz = sz * a.box;
    pqx = shifted ? (float)(L.tx - dsx) : L.fx;
    pqy = shifted ? (float)(L.ty - dsy) : L.fy;
    pqz = shifted ? (float)(L.tz - dsz) : L.fz;
    pslack = shifted ? boxf * 4.8e-7f
                     : (F32 ? 0.f : fmaxf(fabsf(L.fx), fmaxf(fabsf(L.fy), fabsf(L.fz))) * 1.2e-7f);
  };

  // stream the batched ranges through shared memory and test every lane
  auto flush = [&]() {
    const int len = lane < nr ? re - rs : 0;
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    sm.spfx[lane] = incl;
    sm.srsm[lane] = rs - (incl - len);
    __syncwarp();
    auto cand_of = [&](int s) -> int {
      int r = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1)
        if (sm.spfx[r + step - 1] <= s) r += step;
      return sm.srsm[r] + s;
    };
    int my_ci = lane < total ? cand_of(lane) : 0;
    StageT v_cur;
    if (lane < total) v_cur = pos[my_ci];
    for (int c0 = 0; c0 < total; c0 += 32) {
      StageT *stb = sm.stage + ((c0 >> 5) & 1) * 32;
      int *sti = sm.sidx + ((c0 >> 5) & 1) * 32;
      const int nc = min(32, total - c0);
      if (lane < nc) { stb[lane] = v_cur; sti[lane] = my_ci; }
      __syncwarp();
      if (c0 + 32 + lane < total) {
        my_ci = cand_of(c0 + 32 + lane);
        v_cur = pos[my_ci];
      }
      tests += (unsigned long long)nc * n_mem;
#pragma unroll 4
      for (int j = 0; j < nc; ++j) {
        const StageT c = stb[j];
        const int cidx = sti[j];
        float af = 0.f;
        double ad = 0.0;
        if constexpr (F32) {
          float dx, dy, dz;
          if (shifted) {
            dx = (c.x + csx) - tfx; dy = (c.y + csy) - tfy; dz = (c.z + csz) - tfz;
          } else {
            dx = c.x - L.fx; dy = c.y - L.fy; dz = c.z - L.fz;
          }
          af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        } else {
          double cx = c.x, cy = c.y, cz = c.z;
          if (shifted) { cx = __dadd_rn(cx, dsx); cy = __dadd_rn(cy, dsy); cz = __dadd_rn(cz, dsz); }
          ad = exact_d2(__dsub_rn(cx, L.tx), __dsub_rn(cy, L.ty), __dsub_rn(cz, L.tz));
        }
#define SPH_EXACT() exact_image_d2((double)c.x, (double)c.y, (double)c.z, shifted, dsx, dsy, dsz, L.tx, L.ty, L.tz)
        if constexpr (SW == SW_HIST) {
          bool inr;
          float x;
          if constexpr (F32) { inr = af <= h_r2; x = af * h_inv; }
          else { inr = ad <= h_r2d; x = (float)(ad * h_invd); }
          if (inr) sm.hist[hist_bin(x) * 32 + lane] += 1u;
        } else if constexpr (SW == SW_BAND) {
          const bool is_self = (cidx == L.p) && !shifted;
          if (!is_self) {
            double e = -1.0;
            if constexpr (F32) {
              if (af < e_lo_f) ++L.c_below;
              else if (af <= e_hi_f) e = SPH_EXACT();
            } else {
              e = in ? ad : -1.0;
            }
            if (e >= 0.0) {
              if (e < L.lo) ++L.c_below;
              else if (e <= L.hi) {
                if (L.n_in < BAND_CAP) sm.band[L.n_in * 32 + lane] = e;
                ++L.n_in;
                L.emin = fmin(L.emin, e);
                L.emax = fmax(L.emax, e);
                const int bin = min(max((int)((e - L.lo) * L.scale), 0), NB_BAND - 1);
                sm.bh[bin * 32 + lane] += 1u;
              }
            }
          }
        } else {  // SW_DENS
          if constexpr (F32) {
            if (af < e_d2k_f) {
              if (a.dens64) {
                const double e = SPH_EXACT();
                if (e < L.d2k) {
                  const double r_ = __dsqrt_rn(e);
                  double w;
                  if (a.kernel_kind == 0) {
                    w = wc6_lowered(r_, L.hh, L.norm_h3);
                  } else {
                    const double q = __ddiv_rn(r_, L.hh);
                    w = q < 1.0 ? L.norm_h3 * m4_profile(q) : 0.0;
                  }
                  L.accd = __dadd_rn(L.accd, __dmul_rn(a.mass64[cidx], w));
                }
              } else {
                const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
                const float q = rr * L.inv_h;
                const float w = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
                if (q < 1.f) L.accf = fmaf(c.w, w, L.accf);
              }
              ++accepted;
            }
          } else {
            if (ad < e_d2k) {
              const double r_ = __dsqrt_rn(ad);
              double w;
              if (a.kernel_kind == 0) {
                w = wc6_lowered(r_, L.hh, L.norm_h3);
              } else {
                const double q = __ddiv_rn(r_, L.hh);
                w = q < 1.0 ? L.norm_h3 * m4_profile(q) : 0.0;
              }
              L.accd = __dadd_rn(L.accd, __dmul_rn(c.m, w));
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
  };

  // classify one cell (box from lane `src` registers) and count / batch it
  auto visit_cell = [&](int node, float4 l4, float4 h4, int src, int s0, int e0) {
    const float cx0 = __shfl_sync(FULL, l4.x, src), cy0 = __shfl_sync(FULL, l4.y, src),
                cz0 = __shfl_sync(FULL, l4.z, src), cx1 = __shfl_sync(FULL, h4.x, src),
                cy1 = __shfl_sync(FULL, h4.y, src), cz1 = __shfl_sync(FULL, h4.z, src);
    const float gx = fmaxf(fmaxf(cx0 - pqx, pqx - cx1) - pslack, 0.f);
    const float gy = fmaxf(fmaxf(cy0 - pqy, pqy - cy1) - pslack, 0.f);
    const float gz = fmaxf(fmaxf(cz0 - pqz, pqz - cz1) - pslack, 0.f);
    const float gap2 = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps);
    const bool touch = gap2 <= my_r2;
    if (!__any_sync(FULL, touch)) return;
    if (record) {
      if (n_cells < kCellList) {
        if (lane == 0) cell_list[n_cells] = (int)((unsigned)node | ((unsigned)cur_shift << 27));
        ++n_cells;
      } else {
        list_ok = false;
      }
    }
    const float fxa = fmaxf(pqx - cx0, cx1 - pqx) + pslack;
    const float fya = fmaxf(pqy - cy0, cy1 - pqy) + pslack;
    const float fza = fmaxf(pqz - cz0, cz1 - pqz) + pslack;
    const float dmax2 = (fxa * fxa + fya * fya + fza * fza) * (1.0f + 4.0f * kEps);
    const int ncell = e0 - s0;
    const int self_in = (!shifted && s0 <= L.p && L.p < e0) ? 1 : 0;
    bool need = false;
    int sc = -1;
    if constexpr (SW == SW_HIST) {
      if (gap2 <= h_r2) {
        const int b0 = hist_bin(gap2 * h_inv), b1 = hist_bin(dmax2 * h_inv);
        if (dmax2 <= h_r2 && b0 == b1) sc = b0; else need = true;
      }
    } else if constexpr (SW == SW_BAND) {
      if (!(gap2 > e_hi_f)) {
        if (dmax2 < e_lo_f) sc = ncell - self_in; else need = true;
      }
    } else {
      need = gap2 < e_d2k_f;
    }
    if (!__any_sync(FULL, need)) {
      if constexpr (SW == SW_HIST) {
        if (sc >= 0) sm.hist[sc * 32 + lane] += (unsigned)ncell;
      } else if constexpr (SW == SW_BAND) {
        if (sc > 0) L.c_below += sc;
      }
      return;
    }
    if (s0 == last_e) {
      if (lane == nr - 1) re = e0;
    } else {
      if (nr == 32) flush();
      if (lane == nr) { rs = s0; re = e0; }
      ++nr;
    }
    last_e = e0;
  };

  if (from_list) {
    for (int c0 = 0; c0 < n_cells; c0 += 32) {
      const int nc = min(32, n_cells - c0);
      int my_code = 0, my_start = n, my_end = n;
      float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
      if (lane < nc) {
        my_code = cell_list[c0 + lane];
        const int node = my_code & ((1 << 27) - 1);
        l4 = nlo[node];
        h4 = nhi[node];
        my_start = __float_as_int(h4.w);
        my_end = node + 1 < n_nodes ? __float_as_int(nhi[node + 1].w) : n;
      }
      for (int j = 0; j < nc; ++j) {
        const int code = __shfl_sync(FULL, my_code, j);
        const int sidx = (int)((unsigned)code >> 27);
        if (sidx != cur_shift) {
          if (nr) flush();
          set_shift(sidx);
        }
        visit_cell(code & ((1 << 27) - 1), l4, h4, j, __shfl_sync(FULL, my_start, j), __shfl_sync(FULL, my_end, j));
      }
    }
    if (nr) flush();
    return;
  }

  if (record) { n_cells = 0; list_ok = n_nodes < (1 << 27); }
  const int n_shift = a.periodic ? 27 : 1;
  for (int s = 0; s < n_shift; ++s) {
    const int sidx = a.periodic ? s : 0;
    const int sx = a.periodic ? sidx / 9 - 1 : 0;
    const int sy = a.periodic ? (sidx / 3) % 3 - 1 : 0;
    const int sz = a.periodic ? sidx % 3 - 1 : 0;
    float qlx = bx0, qly = by0, qlz = bz0, qhx = bx1, qhy = by1, qhz = bz1;
    if (sx | sy | sz) {
      const double bxs = a.box;
      qlx = __double2float_rd((double)bx0 - sx * bxs); qhx = __double2float_ru((double)bx1 - sx * bxs);
      qly = __double2float_rd((double)by0 - sy * bxs); qhy = __double2float_ru((double)by1 - sy * bxs);
      qlz = __double2float_rd((double)bz0 - sz * bxs); qhz = __double2float_ru((double)bz1 - sz * bxs);
      if (box_gap2(nlo[0], nhi[0], qlx, qly, qlz, qhx, qhy, qhz) > R2b) continue;
    }
    if (nr) flush();
    set_shift(sidx);
    int kk = 0;
    while (kk < n_nodes) {
      const int w = kk;
      const int my = w + lane;
      bool hit = false;
      int my_skip = n_nodes, my_start = n;
      float4 l4 = make_float4(0.f, 0.f, 0.f, 0.f), h4 = l4;
      if (my < n_nodes) {
        l4 = nlo[my];
        h4 = nhi[my];
        my_skip = __float_as_int(l4.w);
        my_start = __float_as_int(h4.w);
        hit = box_gap2(l4, h4, qlx, qly, qlz, qhx, qhy, qhz) <= R2b;
      }
      const unsigned hitm = __ballot_sync(FULL, hit);
      int next_start = __shfl_down_sync(FULL, my_start, 1);
      if (lane == 31) next_start = (w + 32 < n_nodes) ? __float_as_int(nhi[w + 32].w) : n;
      while (kk < w + 32 && kk < n_nodes) {
        const int bb = kk - w;
        const int skp = __shfl_sync(FULL, my_skip, bb);
        if ((hitm >> bb) & 1u) {
          if (skp == kk + 1)
            visit_cell(kk, l4, h4, bb, __shfl_sync(FULL, my_start, bb), __shfl_sync(FULL, next_start, bb));
          ++kk;
        } else {
          kk = skp;
        }
      }
    }
  }
  if (nr) flush();
}

template <bool F32>
__global__ void __launch_bounds__(kWarps * 32) k_fused(const FusedArgs a) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  using StageT = typename Stage<F32>::T;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  unsigned char *wbase = smem_raw + wib * warp_smem<F32>();
  Smem<F32> sm;
  sm.stage = reinterpret_cast<StageT *>(wbase);
  sm.sidx = reinterpret_cast<int *>(wbase + 2 * 32 * sizeof(StageT));
  sm.spfx = sm.sidx + 64;
  sm.srsm = sm.spfx + 32;
  unsigned char *tbase = wbase + stage_bytes<F32>();
  sm.hist = reinterpret_cast<unsigned *>(tbase);
  sm.band = reinterpret_cast<double *>(tbase);
  sm.bh = reinterpret_cast<unsigned *>(tbase + BAND_CAP * 32 * 8);
  const int gwarp = blockIdx.x * kWarps + wib;
  int *cell_list = a.cell_lists + (size_t)gwarp * kCellList;
  const int K = a.k;
  unsigned long long tests = 0, accepted = 0, tests_search = 0;
  unsigned long long cyc_search = 0, cyc_select = 0, cyc_dens = 0;

  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(a.work_counter, 1);
    b = __shfl_sync(FULL, b, 0);
    if (b >= *a.task_count) break;
    const int2 task = a.tasks[b];
    const long long dbg_t0 = a.dbg ? clock64() : 0;
    const unsigned long long dbg_tests0 = tests;

    Lane L;
    L.member = lane < task.y;
    L.p = (int)a.members[task.x + (L.member ? lane : 0)];
    if constexpr (F32) {
      const float4 v = reinterpret_cast<const float4 *>(a.pos)[L.p];
      L.fx = v.x; L.fy = v.y; L.fz = v.z;
      L.tx = v.x; L.ty = v.y; L.tz = v.z;
    } else {
      const D4 v = reinterpret_cast<const D4 *>(a.pos)[L.p];
      L.tx = v.x; L.ty = v.y; L.tz = v.z;
      L.fx = (float)v.x; L.fy = (float)v.y; L.fz = (float)v.z;
    }
    L.status = L.member ? L_HIST : L_NONE;
    L.R = L.member ? a.r0[L.p] : 0.f;
    L.hR2 = 0.f; L.h_inv = 0.f;
    L.lo = 0.0; L.hi = -1.0; L.scale = 0.0; L.emin = INFINITY; L.emax = -INFINITY;
    L.lo_f = -1.f; L.hi_f = -2.f; L.c_below = 0; L.n_in = 0;
    L.d2k = 0.0; L.hh = 0.0; L.norm_h3 = 0.0; L.accd = 0.0; L.d2k_f = -1.f; L.inv_h = 0.f; L.accf = 0.f;
    L.in_sweep = false; L.rad = 0.f;
    int n_cells = 0;
    bool list_ok = false;
    int search_rounds = 0, band_rounds = 0;

    // ---------------- search ----------------
    long long tc0 = clock64();
    for (int round = 0; round < kMaxSearchRounds; ++round) {
      L.in_sweep = L.status == L_HIST;
      if (!__any_sync(FULL, L.in_sweep)) break;
      ++search_rounds;
#pragma unroll
      for (int bb = 0; bb < NB_HIST; ++bb) sm.hist[bb * 32 + lane] = 0u;
      if (L.in_sweep) {
        L.rad = L.R;
        L.hR2 = L.R * L.R;
        L.h_inv = 1.0f / L.hR2;
      }
      const unsigned long long t0 = tests;
      sweep<SW_HIST, F32>(a, L, sm, false, false, cell_list, n_cells, list_ok, tests, accepted);
      tests_search += tests - t0;
      if (L.in_sweep) {
        unsigned total = 0;
#pragma unroll
        for (int bb = 0; bb < NB_HIST; ++bb) total += sm.hist[bb * 32 + lane];
        total -= 1u;  // the target itself (d2 = 0, bin 0)
        if ((int)total < K) {
          if (L.R >= a.rmax) {
            L.status = L_UNREACH;
          } else {
            float f = total > 0 ? cbrtf((float)(K + 8) / (float)total) * 1.15f : 2.f;
            f = fminf(fmaxf(f, 1.26f), 2.5f);
            L.R = fminf(L.R * f, a.rmax);
          }
        } else {
          int cum = 0, bb = 0;
          for (; bb < NB_HIST; ++bb) {
            const int hcount = (int)sm.hist[bb * 32 + lane] - (bb == 0 ? 1 : 0);
            if (cum + hcount >= K) break;
            cum += hcount;
          }
          const double R2d = (double)L.hR2;
          if (bb == 0) {
            L.lo = 0.0;
            L.hi = (double)__int_as_float(kHistBase << 21) * R2d * (1.0 + 8.0 * kEpsD);
          } else if (bb >= NB_HIST - 1) {
            L.lo = R2d * (1.0 - 8.0 * kEpsD);
            L.hi = R2d * (1.0 + 8.0 * kEpsD);
          } else {
            L.lo = (double)__int_as_float((kHistBase + bb - 1) << 21) * R2d * (1.0 - 8.0 * kEpsD);
            L.hi = (double)__int_as_float((kHistBase + bb) << 21) * R2d * (1.0 + 8.0 * kEpsD);
          }
          L.status = L_BAND;
        }
      }
    }
    if (L.status == L_HIST) L.status = L_UNREACH;  // round limit: treated as no K-th neighbour

    long long tc1 = clock64();
    cyc_search += (unsigned long long)(tc1 - tc0);
    // ---------------- select ----------------
    float cover = -1.f;  // radius the recorded cell list covers for this lane
    for (int round = 0; round < kMaxBandRounds; ++round) {
      L.in_sweep = L.status == L_BAND;
      if (!__any_sync(FULL, L.in_sweep)) break;
      ++band_rounds;
#pragma unroll
      for (int bb = 0; bb < NB_BAND; ++bb) sm.bh[bb * 32 + lane] = 0u;
      if (L.in_sweep) {
        L.scale = L.hi > L.lo ? (double)NB_BAND / (L.hi - L.lo) : 0.0;
        L.lo_f = __double2float_rd(L.lo * (1.0 - kEpsD)) - 1e-37f;
        L.hi_f = __double2float_ru(L.hi * (1.0 + kEpsD)) + 1e-37f;
        L.rad = __double2float_ru(sqrt(L.hi) * (1.0 + kEpsD)) + 1e-30f;
        L.c_below = 0; L.n_in = 0; L.emin = INFINITY; L.emax = -INFINITY;
      }
      const bool covered = __all_sync(FULL, !L.in_sweep || L.rad <= cover);
      const bool use_list = covered && list_ok;
      if (!use_list) cover = L.in_sweep ? L.rad : -1.f;  // the re-recorded list covers only this sweep
      sweep<SW_BAND, F32>(a, L, sm, use_list, !use_list, cell_list, n_cells, list_ok, tests, accepted);
      if (L.in_sweep) {
        const int r = K - L.c_below;  // 1-based rank inside the bracket
        if (r <= 0) {
          L.hi = nextafter(L.lo, -INFINITY);
          L.lo = 0.0;
        } else if (r > L.n_in) {
          L.lo = nextafter(L.hi, INFINITY);
          L.hi = (double)L.R * (double)L.R * (1.0 + 16.0 * kEpsD);
        } else if (L.n_in <= BAND_CAP) {
          double v = 0.0;
          for (int i = 0; i < L.n_in; ++i) {
            const double ei = sm.band[i * 32 + lane];
            int less = 0, eq = 0;
            for (int j2 = 0; j2 < L.n_in; ++j2) {
              const double ej = sm.band[j2 * 32 + lane];
              less += ej < ei;
              eq += ej == ei;
            }
            if (less < r && r <= less + eq) { v = ei; break; }
          }
          L.d2k = v;
          L.status = L_DONE;
        } else if (L.emin == L.emax) {
          L.d2k = L.emin;
          L.status = L_DONE;
        } else {
          int cum = 0, bb = 0;
          for (; bb < NB_BAND; ++bb) {
            const int hcount = (int)sm.bh[bb * 32 + lane];
            if (cum + hcount >= r) break;
            cum += hcount;
          }
          bb = min(bb, NB_BAND - 1);
          const double width = L.hi - L.lo;
          double nl = bb == 0 ? L.lo : L.lo + (double)bb / L.scale - width * 1e-12;
          double nh = bb == NB_BAND - 1 ? L.hi : L.lo + (double)(bb + 1) / L.scale + width * 1e-12;
          nl = fmax(nextafter(nl, -INFINITY), fmax(L.lo, L.emin));
          nh = fmin(nextafter(nh, INFINITY), fmin(L.hi, L.emax));
          L.lo = nl;
          L.hi = nh;
        }
      }
    }
    const bool unsettled = L.status == L_BAND;  // internal failure, reported by the host

    tc0 = clock64();
    cyc_select += (unsigned long long)(tc0 - tc1);
    // ---------------- density ----------------
    L.in_sweep = L.status == L_DONE;
    if (L.in_sweep) {
      L.hh = __dsqrt_rn(L.d2k);
      L.norm_h3 = __ddiv_rn(a.kernel_kind == 0 ? kWc6Norm : kM4Norm, __dmul_rn(__dmul_rn(L.hh, L.hh), L.hh));
      L.d2k_f = __double2float_ru(L.d2k * (1.0 + kEpsD));
      L.inv_h = (float)(1.0 / L.hh);
      L.rad = __double2float_ru(L.hh * (1.0 + kEpsD)) + 1e-30f;
    }
    {
      const bool covered = __all_sync(FULL, !L.in_sweep || L.rad <= cover);
      sweep<SW_DENS, F32>(a, L, sm, covered && list_ok, false, cell_list, n_cells, list_ok, tests, accepted);
    }

    cyc_dens += (unsigned long long)(clock64() - tc0);
    if (L.member) {
      if (L.status == L_DONE) {
        a.d2k[L.p] = L.d2k;
        a.rho[L.p] = (F32 && !a.dens64) ? __dmul_rn(L.norm_h3, (double)L.accf) : L.accd;
        a.state[L.p] = ST_DONE;
      } else {
        a.d2k[L.p] = INFINITY;
        a.state[L.p] = unsettled ? ST_FAILED : ST_UNREACHABLE;
        if (unsettled) atomicAdd(&a.stats[4], 1ull);
      }
    }
    if (a.dbg && lane == 0) {
      unsigned long long *d = a.dbg + 4ull * b;
      d[0] = (unsigned long long)(clock64() - dbg_t0);
      d[1] = tests - dbg_tests0;
      d[2] = ((unsigned long long)(unsigned)L.p << 32) | ((unsigned)task.y << 16) | ((unsigned)search_rounds << 8) |
             (unsigned)band_rounds;
      d[3] = (unsigned long long)__float_as_uint(warp_max(L.member ? L.R : 0.f));
    }
  }
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
    atomicAdd(&a.stats[3], tests_search);
    atomicAdd(&a.stats[5], cyc_search);
    atomicAdd(&a.stats[6], cyc_select);
    atomicAdd(&a.stats[7], cyc_dens);
  }
}

template <bool F32>
int fused_blocks(int num_sms) {
  static int bps = 0;
  if (!bps) {
    cudaFuncSetAttribute(k_fused<F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWarps * warp_smem<F32>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_fused<F32>, kWarps * 32, kWarps * warp_smem<F32>());
    if (bps < 1) bps = 1;
  }
  return num_sms * bps;
}

}  // namespace

int fused_warps(int f32, int num_sms) {
  return (f32 ? fused_blocks<true>(num_sms) : fused_blocks<false>(num_sms)) * kWarps;
}
size_t fused_cell_list_ints(int f32, int num_sms) { return (size_t)fused_warps(f32, num_sms) * kCellList; }

void launch_fused(cudaStream_t s, int f32, const FusedArgs &a, int num_sms) {
  cudaMemsetAsync(a.work_counter, 0, sizeof(int), s);
  if (f32)
    k_fused<true><<<fused_blocks<true>(num_sms), kWarps * 32, kWarps * warp_smem<true>(), s>>>(a);
  else
    k_fused<false><<<fused_blocks<false>(num_sms), kWarps * 32, kWarps * warp_smem<false>(), s>>>(a);
}

}  // namespace sph
