// Bundle pass: one warp serves 32 consecutive sorted targets (a spatially
// coherent bundle, one target per lane) whose search radius is already known
// to within ~10% (the seeds' converged h, k_seed_radius in sph_api.cu).
//
// The reference searches each target on its own (density.py:193-212,
// octree.py:179-227); here the warp walks the tree ONCE for the bundle (the
// box holding every lane's search sphere) and every candidate it streams is
// tested by all 32 lanes against their own targets from a shared-memory tile:
//
//   pass 1  count   d2 (fp32) of every candidate of the bundle's cells; each
//                   lane bins the ones within its R into its own column of a
//                   d2/R^2 histogram (16 bins per octave); candidates within R
//                   of some lane are kept in a per-bundle list
//   bracket         each lane finds the bin holding its K-th neighbour
//   pass 2  select  over the kept list: exact unfused fp64 d2 (octree.py:211-214
//                   arithmetic) for the candidates whose fp32 d2 may fall in the
//                   bracket, count below + rank inside -> the exact d2_K
//                   (h = sqrt(d2_K), density.py:226-245)
//   pass 3  density rho = sum over the kept list within h of m_j W(r/h)
//                   (density.py:160-171, 249-261; kernel.py:30-45)
//
// A lane whose radius holds fewer than K others, whose bracket is too crowded
// or misses, keeps its target in ST_NEED_HIST for the per-target kernel
// (sph_warp.cu); so does a whole bundle whose cell or candidate list overflows.
// fp32 positions only (BASELINE configs 2-5); the fp64 path uses k_target.
#include "sph_internal.cuh"
#include <algorithm>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kBW = 4;  // warps per block
#ifndef SPH_BUNDLE_BPO_LOG2
#define SPH_BUNDLE_BPO_LOG2 4
#endif
#ifndef SPH_BUNDLE_OCT
#define SPH_BUNDLE_OCT 4
#endif
constexpr int kBOct = SPH_BUNDLE_OCT;                 // octaves of d2 / R^2 the histogram resolves
constexpr int kBBits = SPH_BUNDLE_BPO_LOG2;           // log2 bins per octave
constexpr int kBBase = (127 - kBOct) << kBBits;
constexpr int kBNB = (kBOct << kBBits) + 2;           // bin 0: below 2^-kBOct; last bin: x >= 1
constexpr int kBNBp = (kBNB + 3) & ~3;
constexpr int kBShift = 23 - kBBits;
#ifndef SPH_BUNDLE_CELLS
#define SPH_BUNDLE_CELLS 192
#endif
#ifndef SPH_BUNDLE_LIST
#define SPH_BUNDLE_LIST 768
#endif
constexpr int kBCells = SPH_BUNDLE_CELLS;  // cells per bundle and image
constexpr int kBList = SPH_BUNDLE_LIST;    // kept candidates per bundle
constexpr int kBStack = 160;               // traversal stack (node ids)
constexpr int kBBuf = (kBNBp * 2) / 8 < 24 ? (kBNBp * 2) / 8 : 24;  // in-bracket fp64 values per lane (alias the histogram)
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard (as sph_warp.cu)
constexpr double kEpsD = 9.5367431640625e-07;

struct alignas(16) BundleSmem {
  uint16_t hist[kBNBp * 32];  // [bin][lane]; pass 2 reuses it as double buf[kBBuf][32]
  uint32_t list[kBList];      // kept candidates: sorted position | image shift << 27
  int2 cells[kBCells];        // traversal: child-record index; after culling: (start, end)
  float4 tgt[32];             // the lanes' targets (x, y, z, R^2; R^2 < 0: inactive)
  union {
    int stk[kBStack];
    struct {
      float4 tile[32];        // the candidate chunk every lane tests
      uint32_t tidx[32];      // its list entries
    } t;
  } u;
  int seg_list[28];           // first list entry of each image segment
  int seg_sidx[28];
};

__device__ __forceinline__ int bbin(float x) {  // x = d2 / R^2 <= 1 (+ rounding)
  return max((__float_as_int(x) >> kBShift) - kBBase + 1, 0);
}

// fp32 image arithmetic of k_target (sph_warp.cu): x_j - box for a -box shift,
// the target moves instead (x_i - box) for a +box shift
struct Img {
  float csx, csy, csz, tfx, tfy, tfz;
};
__device__ __forceinline__ Img make_img(int sidx, bool periodic, float boxf, float fx, float fy, float fz) {
  const int sx = periodic ? sidx / 9 - 1 : 0, sy = periodic ? (sidx / 3) % 3 - 1 : 0, sz = periodic ? sidx % 3 - 1 : 0;
  Img m;
  m.csx = sx < 0 ? -boxf : 0.f;
  m.csy = sy < 0 ? -boxf : 0.f;
  m.csz = sz < 0 ? -boxf : 0.f;
  m.tfx = sx > 0 ? fx - boxf : fx;
  m.tfy = sy > 0 ? fy - boxf : fy;
  m.tfz = sz > 0 ? fz - boxf : fz;
  return m;
}
__device__ __forceinline__ float img_d2(const float4 &c, const Img &m) {
  const float dx = (c.x + m.csx) - m.tfx, dy = (c.y + m.csy) - m.tfy, dz = (c.z + m.csz) - m.tfz;
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
__device__ __forceinline__ float own_d2(const float4 &c, float fx, float fy, float fz) {
  const float dx = c.x - fx, dy = c.y - fy, dz = c.z - fz;
  return fmaf(dx, dx, fmaf(dy, dy, dz * dz));
}
// the reference's fp64 d2 of an image candidate (octree.py:211-214, image
// position fl(x + s*box) as in the image-augmented oracle)
__device__ __forceinline__ double exact_img_d2(const float4 &c, int sidx, bool periodic, double box, double tx,
                                               double ty, double tz) {
  double cx = c.x, cy = c.y, cz = c.z;
  if (periodic && sidx != 13) {
    const int sx = sidx / 9 - 1, sy = (sidx / 3) % 3 - 1, sz = sidx % 3 - 1;
    cx = __dadd_rn(cx, sx * box);
    cy = __dadd_rn(cy, sy * box);
    cz = __dadd_rn(cz, sz * box);
  }
  return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
}

// one pass-1 chunk: every lane tests the tile's ne candidates against its target
template <bool SHIFTED>
__device__ __forceinline__ unsigned count_chunk(BundleSmem &S, int ne, int lane, const Img &im, float fx, float fy,
                                                float fz, float R2, float invR2) {
  unsigned mine = 0u;
  auto one = [&](int e) {
    const float4 c = S.u.t.tile[e];
    const float af = SHIFTED ? img_d2(c, im) : own_d2(c, fx, fy, fz);
    if (af <= R2) {
      ++S.hist[bbin(af * invR2) * 32 + lane];
      mine |= 1u << e;
    }
  };
  if (ne == 32) {
#pragma unroll 8
    for (int e = 0; e < 32; ++e) one(e);
  } else {
    for (int e = 0; e < ne; ++e) one(e);
  }
  return mine;
}

__global__ void __launch_bounds__(kBW * 32) k_bundle(const PassArgs a, int nbundles, int *counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BundleSmem &S = reinterpret_cast<BundleSmem *>(smem_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const float4 *__restrict__ pos = reinterpret_cast<const float4 *>(a.pos);
  const int n = a.n, K = a.k;
  const bool periodic = a.periodic != 0;
  const int center = periodic ? 13 : 0;
  const float boxf = (float)a.box;
  const double norm = a.kernel_kind == 0 ? kWc6Norm : kM4Norm;
  const float4 root_lo = a.tree.nlo[0], root_hi = a.tree.nhi[0];
  double *buf = reinterpret_cast<double *>(S.hist);
  unsigned long long tests = 0, accepted = 0;
  int n_bundle_fail = 0, n_lane_fail = 0, n_done = 0;

  int b_next = 0;
  if (lane == 0) b_next = atomicAdd(a.work_counter, 1);
  for (;;) {
    const int b = __shfl_sync(FULL, b_next, 0);
    if (b >= nbundles) break;
    if (lane == 0) b_next = atomicAdd(a.work_counter, 1);
    const int p = b * 32 + lane;
    bool act0 = p < n && a.state[p] == ST_NEED_HIST;
    const float R = act0 ? a.radius[p] : 0.f;
    if (!(R > 0.f) || !(R < a.rmax)) act0 = false;
    if (!__any_sync(FULL, act0)) continue;
    const float4 t4 = act0 ? pos[p] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float fx = t4.x, fy = t4.y, fz = t4.z;
    const double tx = fx, ty = fy, tz = fz;

    // the whole bundle first; a bundle whose cells or kept candidates overflow
    // is retried as 2, then 4 sub-bundles of consecutive lanes
    for (int parts = 1; parts <= 4; parts *= 2) {
      bool part_failed = false;
      for (int part = 0; part < parts; ++part) {
        const bool act = act0 && (lane * parts) / 32 == part;
        const unsigned amask = __ballot_sync(FULL, act);
        if (!amask) continue;
        const float R2 = act ? R * R : -1.f;
        const float invR2 = act ? 1.0f / R2 : 0.f;
        S.tgt[lane] = make_float4(fx, fy, fz, R2);

        // ---- query box: every active lane's search sphere (tree frame) ----
        const float ext = R * (1.0f + 16.0f * kEps);
        float qlx = act ? fx - ext : INFINITY, qly = act ? fy - ext : INFINITY, qlz = act ? fz - ext : INFINITY;
        float qhx = act ? fx + ext : -INFINITY, qhy = act ? fy + ext : -INFINITY, qhz = act ? fz + ext : -INFINITY;
        for (int o = 16; o; o >>= 1) {
          qlx = fminf(qlx, __shfl_xor_sync(FULL, qlx, o));
          qly = fminf(qly, __shfl_xor_sync(FULL, qly, o));
          qlz = fminf(qlz, __shfl_xor_sync(FULL, qlz, o));
          qhx = fmaxf(qhx, __shfl_xor_sync(FULL, qhx, o));
          qhy = fmaxf(qhy, __shfl_xor_sync(FULL, qhy, o));
          qhz = fmaxf(qhz, __shfl_xor_sync(FULL, qhz, o));
        }
        {  // rounding slack of the box arithmetic (and of the shifted frames)
          const float m = fmaxf(fmaxf(fmaxf(fabsf(qlx), fabsf(qhx)), fmaxf(fabsf(qly), fabsf(qhy))),
                                fmaxf(fabsf(qlz), fabsf(qhz)));
          const float sl = (m + (periodic ? boxf : 0.f)) * 4.8e-7f;
          qlx -= sl; qly -= sl; qlz -= sl;
          qhx += sl; qhy += sl; qhz += sl;
        }
        // images to search: the unshifted one plus every shift whose query box
        // meets the root box (one shift per lane)
        unsigned shifts = 1u << center;
        if (periodic) {
          bool want = false;
          if (lane < 27 && lane != 13) {
            const float sx = (float)(lane / 9 - 1) * boxf, sy = (float)((lane / 3) % 3 - 1) * boxf,
                        sz = (float)(lane % 3 - 1) * boxf;
            // tree-frame query box of image s: Q - s*box (candidates x_j + s*box near the targets)
            want = root_lo.x <= qhx - sx && root_hi.x >= qlx - sx && root_lo.y <= qhy - sy &&
                   root_hi.y >= qly - sy && root_lo.z <= qhz - sz && root_hi.z >= qlz - sz;
          }
          shifts |= __ballot_sync(FULL, want);
        }

        // ---- pass 1: walk once per image, cull cells per target, count into the histograms ----
        {
          uint4 *h4 = reinterpret_cast<uint4 *>(S.hist);
          for (int i = lane; i < (kBNBp * 32 * 2) / 16; i += 32) h4[i] = make_uint4(0u, 0u, 0u, 0u);
        }
        int nlist = 0, nseg = 0, cnt = 0;
        bool fail = false;
        __syncwarp();
        for (unsigned sm = shifts; sm && !fail;) {
          const int sidx = (sm >> center) & 1u ? center : __ffs(sm) - 1;  // the unshifted image first
          sm &= ~(1u << sidx);
          const bool shifted = sidx != center;
          const int isx = periodic ? sidx / 9 - 1 : 0, isy = periodic ? (sidx / 3) % 3 - 1 : 0,
                    isz = periodic ? sidx % 3 - 1 : 0;
          const float ox = isx * boxf, oy = isy * boxf, oz = isz * boxf;
          const float Lx = qlx - ox, Ly = qly - oy, Lz = qlz - oz, Hx = qhx - ox, Hy = qhy - oy, Hz = qhz - oz;
          // start below the root when an ancestor of the first target's cell holds the whole query box
          int start = a.tree.root_start;
          if (!shifted) {
            const int cell = a.tree.cellof[b * 32 + __ffs(amask) - 1];
            const int4 an = a.tree.anc4[cell];
            const int my = lane == 0 ? an.x : lane == 1 ? an.y : lane == 2 ? an.z : lane == 3 ? an.w : -1;
            bool holds = false;
            if (my >= 0) {
              const float4 l4 = a.tree.nlo[my], h4 = a.tree.nhi[my];
              holds = l4.x <= Lx && Hx <= h4.x && l4.y <= Ly && Hy <= h4.y && l4.z <= Lz && Hz <= h4.z;
            }
            const unsigned hm = __ballot_sync(FULL, holds);
            if (hm) start = __shfl_sync(FULL, my, __ffs(hm) - 1);
          }
          if (lane == 0) {
            S.u.stk[0] = start;
            S.seg_list[nseg] = nlist;
            S.seg_sidx[nseg] = sidx;
          }
          ++nseg;
          int top = 1, ncell = 0;
          __syncwarp();
          while (top > 0) {
            const int np = min(top, 4);
            top -= np;
            const int pi = lane >> 3;
            const int par = pi < np ? S.u.stk[top + pi] : -1;
            __syncwarp();
            bool hit = false, is_cell = false;
            int code = 0;
            if (par >= 0) {
              const float4 *rec = a.tree.crec + 16 * (size_t)par + 2 * (lane & 7);
              const float4 l4 = rec[0], h4 = rec[1];
              code = __float_as_int(l4.w);
              is_cell = code < 0;
              hit = l4.x <= Hx && h4.x >= Lx && l4.y <= Hy && h4.y >= Ly && l4.z <= Hz && h4.z >= Lz;
            }
            const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
            const unsigned cm = __ballot_sync(FULL, hit && is_cell);
            if (top + __popc(pm) > kBStack || ncell + __popc(cm) > kBCells) { fail = true; break; }
            if (hit && !is_cell) S.u.stk[top + __popc(pm & lt)] = code;
            if (hit && is_cell) S.cells[ncell + __popc(cm & lt)].x = par * 8 + (lane & 7);
            top += __popc(pm);
            ncell += __popc(cm);
            __syncwarp();
          }
          if (fail) break;

          // per-target cull (k_target's sphere-box test, sph_warp.cu): keep a
          // cell only if it lies within R of some active target; compact to (start, end)
          {
            const float pslack = shifted ? boxf * 4.8e-7f : 0.f;
            int w = 0;
            for (int g0 = 0; g0 < ncell; g0 += 32) {
              const int ci = g0 + lane;
              float4 l4 = make_float4(INFINITY, INFINITY, INFINITY, 0.f), h4 = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
              if (ci < ncell) {
                const float4 *rec = a.tree.crec + 2 * (size_t)S.cells[ci].x;
                l4 = rec[0];
                h4 = rec[1];
              }
              bool keep = false;
              for (unsigned am = amask; am && ci < ncell; am &= am - 1u) {
                const float4 t = S.tgt[__ffs(am) - 1];
                // the target in the tree frame of this image: x_i - s*box
                const float px = shifted ? (float)((double)t.x - (double)isx * a.box) : t.x;
                const float py = shifted ? (float)((double)t.y - (double)isy * a.box) : t.y;
                const float pz = shifted ? (float)((double)t.z - (double)isz * a.box) : t.z;
                const float gx = fmaxf(fmaxf(l4.x - px, px - h4.x) - pslack, 0.f);
                const float gy = fmaxf(fmaxf(l4.y - py, py - h4.y) - pslack, 0.f);
                const float gz = fmaxf(fmaxf(l4.z - pz, pz - h4.z) - pslack, 0.f);
                if ((gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= t.w) { keep = true; break; }
              }
              const unsigned km = __ballot_sync(FULL, keep);
              __syncwarp();
              if (keep) S.cells[w + __popc(km & lt)] = make_int2(~__float_as_int(l4.w), __float_as_int(h4.w));
              w += __popc(km);
              __syncwarp();
            }
            ncell = w;
          }
          const Img im = make_img(sidx, periodic, boxf, fx, fy, fz);

          // stream the kept cells, 32 at a time; 32 candidates per chunk
          for (int g0 = 0; g0 < ncell && !fail; g0 += 32) {
            const int ci = g0 + lane;
            int len = 0, cst = 0;
            if (ci < ncell) {
              const int2 ce = S.cells[ci];
              cst = ce.x;
              len = ce.y - ce.x;
            }
            int incl = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(FULL, incl, o);
              if (lane >= o) incl += v;
            }
            const int total = __shfl_sync(FULL, incl, 31);
            const int cend = ci < ncell ? incl : 0x7fffffff;
            const int cb = cst - (incl - len);  // j = cb(owner) + stream slot
            for (int c0 = 0; c0 < total; c0 += 32) {
              const int s = c0 + lane;
              const unsigned ev = (cend > c0 && cend <= c0 + 31) ? 1u << (cend - c0 - 1) : 0u;
              const unsigned emask = __reduce_or_sync(FULL, ev);
              const int owner = __popc(__ballot_sync(FULL, cend <= c0)) + __popc(emask & lt);
              const int cbo = __shfl_sync(FULL, cb, owner & 31);
              const int j = s < total ? cbo + s : -1;
              float4 c = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
              if (j >= 0) c = pos[j];
              S.u.t.tile[lane] = c;
              __syncwarp();
              const int ne = min(32, total - c0);
              const unsigned mine = shifted ? count_chunk<true>(S, ne, lane, im, fx, fy, fz, R2, invR2)
                                            : count_chunk<false>(S, ne, lane, im, fx, fy, fz, R2, invR2);
              cnt += __popc(mine);
              tests += (unsigned)ne;
              const bool keep = (__reduce_or_sync(FULL, mine) >> lane) & 1u;
              const unsigned km = __ballot_sync(FULL, keep);
              if (nlist + __popc(km) > kBList) { fail = true; break; }
              if (keep) S.list[nlist + __popc(km & lt)] = (uint32_t)j | ((uint32_t)sidx << 27);
              nlist += __popc(km);
              __syncwarp();
            }
          }
        }
        if (fail) {
          part_failed = true;
          break;  // retry with smaller sub-bundles
        }
        if (lane == 0) S.seg_list[nseg] = nlist;
        __syncwarp();

        // ---- per lane: enough others within R? bracket of the K-th ----
        bool ok = act;
        double tl = 0.0, th = 0.0;
        if (act) {
          const int others = cnt - 1;
          if (others < K) {
            float f = others > 0 ? cbrtf((float)(K + 8) / (float)others) * 1.15f : 2.f;
            f = fminf(fmaxf(f, 1.26f), 2.5f);
            a.radius[p] = fminf(R * f, a.rmax);
            ok = false;
          } else {
            int cum = -1, bb = kBNB - 1;  // the target itself sits in bin 0
            for (int q = 0; q < kBNB; ++q) {
              cum += S.hist[q * 32 + lane];
              if (cum >= K) { bb = q; break; }
            }
            const double R2d = (double)R2;
            if (bb == 0) {
              tl = 0.0;
              th = (double)__int_as_float(kBBase << kBShift) * R2d * (1.0 + 8.0 * kEpsD);
            } else if (bb >= kBNB - 1) {
              tl = R2d * (1.0 - 8.0 * kEpsD);
              th = R2d * (1.0 + 8.0 * kEpsD);
            } else {
              tl = (double)__int_as_float((kBBase + bb - 1) << kBShift) * R2d * (1.0 - 8.0 * kEpsD);
              th = (double)__int_as_float((kBBase + bb) << kBShift) * R2d * (1.0 + 8.0 * kEpsD);
            }
            // the kept list holds every candidate with exact d2 <= R^2 (1 - 4 eps)
            th = fmin(th, R2d * (1.0 - 4.0 * kEpsD));
            if (th < tl) ok = false;
          }
        }
        __syncwarp();  // histogram reads done: the region becomes the in-bracket buffer

        // ---- pass 2: exact count below the bracket, the bracket's values ----
        const float lo_f = ok ? __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f : -1.f;
        const float hi_f = ok ? __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f : -2.f;
        int below = 0, n_in = 0;
        for (int sg = 0; sg < nseg; ++sg) {
          const int sidx = S.seg_sidx[sg];
          const int e0 = S.seg_list[sg], e1 = S.seg_list[sg + 1];
          const Img im = make_img(sidx, periodic, boxf, fx, fy, fz);
          for (int c0 = e0; c0 < e1; c0 += 32) {
            const int i = c0 + lane;
            if (i < e1) {
              const uint32_t ent = S.list[i];
              S.u.t.tile[lane] = pos[ent & ((1u << 27) - 1u)];
              S.u.t.tidx[lane] = ent;
            }
            __syncwarp();
            const int ne = min(32, e1 - c0);
            tests += (unsigned)ne;
            if (ok) {
              for (int e = 0; e < ne; ++e) {
                const float4 c = S.u.t.tile[e];
                const float af = sidx == center ? own_d2(c, fx, fy, fz) : img_d2(c, im);
                if (af < lo_f) {
                  ++below;
                } else if (af <= hi_f) {
                  const int j = (int)(S.u.t.tidx[e] & ((1u << 27) - 1u));
                  if (!(j == p && sidx == center)) {
                    const double ex = exact_img_d2(c, sidx, periodic, a.box, tx, ty, tz);
                    if (ex < tl) {
                      ++below;
                    } else if (ex <= th) {
                      if (n_in < kBBuf) buf[n_in * 32 + lane] = ex;
                      ++n_in;
                    }
                  }
                }
              }
            }
            __syncwarp();
          }
        }
        double d2k = 0.0;
        if (ok) {
          if (tl > 0.0) --below;  // the target itself (d2 = 0 < lo_f); with tl == 0 it was skipped
          const int r = K - below;
          if (r < 1 || r > n_in || n_in > kBBuf) {
            ok = false;
          } else {
            double v = INFINITY;
            for (int i = 0; i < n_in; ++i) {
              const double ei = buf[i * 32 + lane];
              int less = 0, eq = 0;
              for (int jj = 0; jj < n_in; ++jj) {
                const double ej = buf[jj * 32 + lane];
                less += ej < ei;
                eq += ej == ei;
              }
              if (less < r && r <= less + eq) v = ei;
            }
            d2k = v;
            if (!(d2k > 0.0)) ok = false;  // coincident K-th: the per-target kernel reports it
          }
        }
        if (act && !ok) ++n_lane_fail;

        // ---- pass 3: density over the kept list within h ----
        const bool f32sum = !a.dens64;
        const double hh = ok ? __dsqrt_rn(d2k) : 1.0;
        const double norm_h3 = __ddiv_rn(norm, __dmul_rn(__dmul_rn(hh, hh), hh));
        const float d2k_f = ok ? __double2float_ru(d2k * (1.0 + kEpsD)) : -1.f;
        const float inv_h = (float)(1.0 / hh);
        float accf = 0.f;
        double accd = 0.0;
        const bool any_ok = __any_sync(FULL, ok);
        for (int sg = 0; sg < nseg && any_ok; ++sg) {
          const int sidx = S.seg_sidx[sg];
          const int e0 = S.seg_list[sg], e1 = S.seg_list[sg + 1];
          const Img im = make_img(sidx, periodic, boxf, fx, fy, fz);
          for (int c0 = e0; c0 < e1; c0 += 32) {
            const int i = c0 + lane;
            if (i < e1) {
              const uint32_t ent = S.list[i];
              S.u.t.tile[lane] = pos[ent & ((1u << 27) - 1u)];
              S.u.t.tidx[lane] = ent;
            }
            __syncwarp();
            const int ne = min(32, e1 - c0);
            tests += (unsigned)ne;
            if (f32sum) {
              for (int e = 0; e < ne; ++e) {
                const float4 c = S.u.t.tile[e];
                const float af = sidx == center ? own_d2(c, fx, fy, fz) : img_d2(c, im);
                if (af < d2k_f) {
                  const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
                  const float q = rr * inv_h;
                  const float wv = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
                  if (q < 1.f) {
                    accf = fmaf(c.w, wv, accf);
                    ++accepted;
                  }
                }
              }
            } else if (ok) {
              for (int e = 0; e < ne; ++e) {
                const float4 c = S.u.t.tile[e];
                const float af = sidx == center ? own_d2(c, fx, fy, fz) : img_d2(c, im);
                if (af < d2k_f) {
                  const double ex = exact_img_d2(c, sidx, periodic, a.box, tx, ty, tz);
                  if (ex < d2k) {
                    const double r_ = __dsqrt_rn(ex);
                    double wv;
                    if (a.kernel_kind == 0) {
                      wv = wc6_lowered(r_, hh, norm_h3);
                    } else {
                      const double q = __ddiv_rn(r_, hh);
                      wv = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
                    }
                    const int j = (int)(S.u.t.tidx[e] & ((1u << 27) - 1u));
                    accd = __dadd_rn(accd, __dmul_rn(a.mass64[j], wv));
                    ++accepted;
                  }
                }
              }
            }
            __syncwarp();
          }
        }
        if (ok) {
          a.d2k[p] = d2k;
          a.rho[p] = f32sum ? __dmul_rn(norm_h3, (double)accf) : accd;
          a.state[p] = ST_FINAL;
          ++n_done;
        }
      }
      if (!part_failed) break;
      if (parts == 4) ++n_bundle_fail;  // every lane to the per-target kernel
    }
  }
  // statistics: pair tests per lane-candidate of every pass
  for (int o = 16; o; o >>= 1) {
    accepted += __shfl_xor_sync(FULL, accepted, o);
    n_lane_fail += __shfl_xor_sync(FULL, n_lane_fail, o);
    n_done += __shfl_xor_sync(FULL, n_done, o);
  }
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests * 32ull);
    atomicAdd(&a.stats[1], accepted);
    if (counters) {
      if (n_bundle_fail) atomicAdd(counters, n_bundle_fail);
      if (n_lane_fail) atomicAdd(counters + 1, n_lane_fail);
      if (n_done) atomicAdd(counters + 2, n_done);
    }
  }
}

}  // namespace

void launch_bundle(cudaStream_t s, const PassArgs &a, int *counters, int num_sms) {
  const int nb = (a.n + 31) / 32;
  const int smem = kBW * (int)sizeof(BundleSmem);
  int bps = 0;
  cudaFuncSetAttribute(k_bundle, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_bundle, kBW * 32, smem);
  const int grid = std::min(num_sms * std::max(bps, 1), (nb + kBW - 1) / kBW);
  k_bundle<<<std::max(grid, 1), kBW * 32, smem, s>>>(a, nb, counters);
}

}  // namespace sph
