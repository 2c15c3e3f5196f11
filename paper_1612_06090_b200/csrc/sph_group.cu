// sph_group.cu -- the main pass: one warp per search cell (<= 32 consecutive
// sorted particles), its targets served in groups of up to G, so the tree
// walk and the candidate stream are paid once per group instead of once per
// target.
//
// For a group of targets t with radii R_t (reference compute_density_pass,
// density.py:286-413: the todo loop is replaced by a radius that bounds the
// K-th neighbour; the reference's todo trace is rebuilt from h0 and d2_K in
// k_finalize):
//   walk    the search tree from the lowest ancestor of the cell whose box
//           holds the group's region (box of the targets grown by max R),
//           4 parents x 8 child records per step (one record per lane);
//           every hit cell gets a G-bit mask of the target spheres it meets.
//           Periodic boxes: the walk is repeated for each image shift whose
//           region meets the root box, the records tagged with the shift;
//   stage   the hit cells' particles -- contiguous runs of the sorted
//           (x, y, z, index) array -- form one candidate stream, copied
//           global -> shared 32 at a time with cp.async (16 B per lane) into
//           a kRing-deep ring, kRing - 1 chunks ahead of the one in use;
//   list    each staged candidate (one per lane) is tested in fp32 against
//           every group target its cell's mask names (image chunks: the
//           image offset is added in fp64, x_j + s*box - x_i, as the image-
//           augmented reference does) and appended to that target's
//           shared-memory list {index | image << 27, fp32 d2} when d2 <= R_t^2;
//   select  per target, warp-wide over its list: a 32-bin histogram of
//           (d2/R^2)^1.5 finds the bin of the K-th other, the fp32 K-th is
//           ranked inside it, list entries within a relative 2^-20 guard of
//           the band around it get the exact unfused fp64 d2 (octree.py:211-214)
//           and the exact K-th is counted and ranked (density.py:226-245);
//   sum     rho = sum over list entries within h of m_j W(r/h), self included
//           (density.py:160-171, 249-261; kernel.py:30-45), fp32 per pair or
//           fp64 term-for-term (dens64);
//   retry   a target with fewer than K others within R, more than the list
//           holds, or its K-th at the list edge gets a new radius from its
//           exact count inside R (bracketed between the radii already tried)
//           and joins a later group of the same cell.  The first group starts
//           from the tree estimate R0 (k_r0); later groups from margin x the
//           largest h already converged in the cell.
// Targets this kernel cannot finish (a walk beyond its record capacity, a
// crowded bin or band, a radius window that closed, images with n > 2^27)
// are appended to a list for the general per-target kernel (k_target,
// sph_warp.cu).
#include "sph_internal.cuh"

#include <algorithm>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kGWarps = 4;
#ifndef SPH_GROUP_MINB
#define SPH_GROUP_MINB 4
#endif
constexpr int kRing = 4;                      // cp.async ring depth (chunks of 32 candidates)
#ifndef SPH_GROUP_CHITS
#define SPH_GROUP_CHITS 224
#endif
#ifndef SPH_GROUP_GHITS
#define SPH_GROUP_GHITS 160
#endif
#ifndef SPH_GROUP_DEBUG
#define SPH_GROUP_DEBUG 0
#endif
constexpr int kCHits = SPH_GROUP_CHITS;       // hit cells of a cell walk
constexpr int kGHits = SPH_GROUP_GHITS;       // hit cells of a group
constexpr int kGStack = 96;                   // walk stack (internal nodes) per warp
constexpr int kMaxTries = 6;                  // radius retries per target
constexpr int kCenter = 13;                   // the unshifted image (shift index sx*9 + sy*3 + sz + 13)
constexpr unsigned kIdxMask = (1u << 27) - 1u;
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard (fp32 d2 vs exact)
constexpr double kEpsD = 9.5367431640625e-07;

template <int G>
struct alignas(16) GroupSmem {
  float4 ring[kRing][32];
  unsigned meta[kRing][32];  // per staged candidate: target mask | image shift << 8 (0: empty slot)
  float4 tgt[G];             // (x, y, z, R^2) per group target
  float ir2[G];              // 1 / R^2
  int tp[G];                 // sorted position per group target
  int ne[G];                 // entries within R per group target (may exceed the list capacity)
  int res[G];                // outcome per group target
  float rnew[G];             // retry radius per group target (0: the lane's own rule)
  double d2k[G];
  unsigned hist[G][32];      // per target: entries within R in 32 bins of (d2/R^2)^1.5
  unsigned crec_i[kCHits];   // the cell walk's hit cells: child-record index | image shift << 27
  int2 hrec[kGHits];         // the group's hit cells: (first sorted position, stream offset)
  unsigned short hmeta[kGHits];  // target mask | image shift << 8
  int stk[kGStack];
  unsigned binv[32];
  double band[32];
};

enum : int { R_DONE = 0, R_FEW = 1, R_FULL = 2, R_EDGE = 3, R_FALL = 4 };

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async16s(unsigned dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void sts_v2(unsigned addr, unsigned a, unsigned b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts_u16(unsigned addr, unsigned v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void atoms_inc(unsigned addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}
// histogram bin of x = d2 / R^2 in [0, 1]: 32 bins of equal volume.  Only
// its consistency matters (the stream and the select compute it the same way).
__device__ __forceinline__ int vbin(float x) { return min(31, __float2int_rz(32.0f * x * sqrt_approx(x))); }

// exact reference d2 of list entry e (index | image code << 27) from target t:
// the image position fl(x_j + s*box) (image-augmented reference), then
// octree.py:211-214 arithmetic
__device__ __forceinline__ double entry_exact_d2(const PassArgs &a, unsigned e, double tx, double ty, double tz) {
  const float4 c = a.posj[e & kIdxMask];
  double cx = c.x, cy = c.y, cz = c.z;
  const unsigned code = e >> 27;
  if (code) {
    const int s = (int)code - 1;
    cx = __dadd_rn(cx, (s / 9 - 1) * a.box);
    cy = __dadd_rn(cy, ((s / 3) % 3 - 1) * a.box);
    cz = __dadd_rn(cz, (s % 3 - 1) * a.box);
  }
  return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
}

// sorted index | image code << 27 of the candidate in stream slot `slot` of
// the group (its cell: the last hit cell starting at or before the slot)
__device__ __forceinline__ unsigned slot_index(const int2 *hrec, const unsigned short *hmeta, int nh, int slot) {
  int lo = 0, hi = nh - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (hrec[mid].y <= slot) lo = mid;
    else hi = mid - 1;
  }
  const int2 h = hrec[lo];
  const unsigned sidx = hmeta[lo] >> 8;
  return (unsigned)(h.x + (slot - h.y)) | (sidx != kCenter ? (sidx + 1u) << 27 : 0u);
}

// Exact K-th other and density of target p from its list (every entry with
// fp32 d2 <= R^2, the target itself included, as the (K+1)-th smallest
// counts it) and the list's histogram.  Returns R_DONE (d2k, rho written) or
// the reason it could not finish.
template <bool DENS64>
__device__ __forceinline__ int select_density(const PassArgs &a, const uint2 *list, const unsigned short *lslot,
                                              int ne, const unsigned *hist, const int2 *hrec,
                                              const unsigned short *hmeta, int nh, int p, float fx, float fy,
                                              float fz, float R2, float invR2, unsigned *binv, double *band,
                                              unsigned long long &accepted, double &d2k_out) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int K1 = a.k + 1;  // the target itself (d2 = 0) is the smallest entry
  // ---- bin of the (K+1)-th entry ----
  const unsigned hc = hist[lane];
  unsigned hin = hc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(FULL, hin, o);
    if (lane >= o) hin += v;
  }
  const int B = __ffs(__ballot_sync(FULL, (int)hin >= K1)) - 1;  // ne >= K1: exists
  const int rr = K1 - (int)__shfl_sync(FULL, hin - hc, B);       // rank inside bin B (1-based)
  int m = 0;
  for (int i0 = 0; i0 < ne; i0 += 32) {
    const int i = i0 + lane;
    bool mine = false;
    unsigned v = 0;
    if (i < ne) {
      v = list[i].x;
      mine = vbin(__uint_as_float(v) * invR2) == B;
    }
    const unsigned mm = __ballot_sync(FULL, mine);
    if (mine && m + __popc(mm & lt) < 32) binv[m + __popc(mm & lt)] = v;
    m += __popc(mm);
  }
  __syncwarp();
  if (m > 32) return R_FALL;
  unsigned vKb;
  {
    const unsigned v = lane < m ? binv[lane] : 0xffffffffu;
    int rank = 0;
    for (int l = 0; l < m; ++l) {
      const unsigned u = __shfl_sync(FULL, v, l);
      rank += (u < v) || (u == v && l < lane);
    }
    const unsigned sel = __ballot_sync(FULL, lane < m && rank == rr - 1);
    vKb = __shfl_sync(FULL, v, __ffs(sel) - 1);
  }
  // ---- exact K-th: count below the band, rank inside it; the fp32 path sums
  // the density in the same pass with h from the fp32 K-th (terms at the
  // support edge vanish as (1-q)^8, so the band does not move rho) ----
  const double vK = (double)__uint_as_float(vKb);
  const double tl = vK * (1.0 - 3.0 * kEpsD), th = vK * (1.0 + 3.0 * kEpsD);
  const float lo_f = __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f;
  const float hi_f = __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f;
  const double tx = fx, ty = fy, tz = fz;
  const float4 *__restrict__ pos = reinterpret_cast<const float4 *>(a.pos);
  const float vKf = __uint_as_float(vKb);
  const float inv_hf = vKf > 0.f ? rsqrtf(vKf) : 0.f;
  const bool wc6 = a.kernel_kind == 0;
  float accf = 0.f;
  int below = 0, nin = 0;
  for (int i0 = 0; i0 < ne; i0 += 32) {
    const int i = i0 + lane;
    bool inb = false;
    double ex = 0.0;
    if (i < ne) {
      const uint2 e = list[i];
      const float af = __uint_as_float(e.x);
      if (af < lo_f) {
        ++below;
      } else if (af <= hi_f) {
        ex = entry_exact_d2(a, slot_index(hrec, hmeta, nh, lslot[i]), tx, ty, tz);
        if (ex < tl) ++below;
        else if (ex <= th) inb = true;
      }
      if constexpr (!DENS64) {
        if (af < vKf) {
          const float q = af * rsqrtf(fmaxf(af, 1e-37f)) * inv_hf;
          const float wv = wc6 ? wc6_profile_f(q) : m4_profile_f(q);
          if (q < 1.f) accf = fmaf(__uint_as_float(e.y), wv, accf);
          ++accepted;
        }
      }
    }
    const unsigned bmk = __ballot_sync(FULL, inb);
    if (inb && nin + __popc(bmk & lt) < 32) band[nin + __popc(bmk & lt)] = ex;
    nin += __popc(bmk);
  }
  __syncwarp();
  below = (int)__reduce_add_sync(FULL, (unsigned)below);
  const int r = K1 - below;
  if (nin > 32 || r < 1 || r > nin) return R_FALL;
  double d2k;
  {
    const double v = lane < nin ? band[lane] : INFINITY;
    int less = 0, eq = 0;
    for (int l = 0; l < nin; ++l) {
      const double u = __shfl_sync(FULL, v, l);
      less += u < v;
      eq += u == v;
    }
    const unsigned sel = __ballot_sync(FULL, lane < nin && less < r && r <= less + eq);
    d2k = __shfl_sync(FULL, v, __ffs(sel) - 1);
  }
  // everything within the K-th must be in the list: d2_K clear of R^2
  if (!(d2k * (1.0 + 4.0 * kEpsD) < (double)R2)) return R_EDGE;
  double rho = 0.0;
  if (d2k > 0.0) {
    const double norm = wc6 ? kWc6Norm : kM4Norm;
    const double hh = __dsqrt_rn(d2k);
    const double norm_h3 = __ddiv_rn(norm, __dmul_rn(__dmul_rn(hh, hh), hh));
    if constexpr (DENS64) {
      // fp64 term for term over the entries within h (density.py:160-171)
      const float d2k_f = __double2float_ru(d2k * (1.0 + kEpsD));
      double accd = 0.0;
      for (int i = lane; i < ne; i += 32) {
        const uint2 e = list[i];
        if (!(__uint_as_float(e.x) < d2k_f)) continue;
        const unsigned jc = slot_index(hrec, hmeta, nh, lslot[i]);
        const double ex = entry_exact_d2(a, jc, tx, ty, tz);
        if (ex < d2k) {
          ++accepted;
          const double r_ = __dsqrt_rn(ex);
          double wv;
          if (wc6) {
            wv = wc6_lowered(r_, hh, norm_h3);
          } else {
            const double qq = __ddiv_rn(r_, hh);
            wv = qq < 1.0 ? norm_h3 * m4_profile(qq) : 0.0;
          }
          accd = __dadd_rn(accd, __dmul_rn(a.mass64[jc & kIdxMask], wv));
        }
      }
      for (int o = 16; o; o >>= 1) accd += __shfl_xor_sync(FULL, accd, o);
      rho = accd;
    } else {
      for (int o = 16; o; o >>= 1) accf += __shfl_xor_sync(FULL, accf, o);
      rho = __dmul_rn(norm_h3, (double)accf);
    }
  }
  if (lane == 0) {
    a.d2k[p] = d2k;
    a.rho[p] = rho;
    a.state[p] = ST_FINAL;
  }
  d2k_out = d2k;
  return R_DONE;
}

template <int G, bool DENS64>
__global__ void __launch_bounds__(kGWarps * 32, SPH_GROUP_MINB) k_cell(const PassArgs a, const int *__restrict__ cellnode,
                                                       const int *__restrict__ ncells, int lcap, float margin,
                                                       float r0f, int first_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  GroupSmem<G> &S = reinterpret_cast<GroupSmem<G> *>(smem_raw)[wib];
  uint2 *lists = reinterpret_cast<uint2 *>(smem_raw + kGWarps * sizeof(GroupSmem<G>)) + (size_t)wib * G * lcap;
  const unsigned lists_s = smem_u32(lists);
  unsigned short *lslots = reinterpret_cast<unsigned short *>(smem_raw + kGWarps * sizeof(GroupSmem<G>) +
                                                              (size_t)kGWarps * G * lcap * sizeof(uint2)) +
                           (size_t)wib * G * lcap;
  const unsigned lslots_s = smem_u32(lslots);
  const float4 *__restrict__ pos4 = reinterpret_cast<const float4 *>(a.pos);
  const float4 *__restrict__ posj = a.posj;
  const float4 *__restrict__ crec = a.tree.crec;
  const unsigned lt = (1u << lane) - 1u;
  const int nc = *ncells;
  const int n_nodes = a.tree.n_nodes;
  const int K = a.k;
  const bool img_ok = a.n <= (1 << 27);  // list entries carry the image shift in the index's top bits
  const float sl = (float)a.box * 4.8e-7f;  // slack for an image frame rounded to fp32
  unsigned tests = 0;
  unsigned long long accepted = 0;
  int nfb_walk = 0, nfb_sel = 0, nfb_tries = 0, nretry = 0;
#if SPH_GROUP_DEBUG
  unsigned dbg_tc = 0, dbg_chunks = 0, dbg_groups = 0;  // (target, chunk) pairs, chunks, groups
#endif

  for (;;) {
    int ci = 0;
    if (lane == 0) ci = atomicAdd(a.work_counter, 1);
    ci = __shfl_sync(FULL, ci, 0);
    if (ci >= nc) break;
    const int node = cellnode[ci];
    const int s0 = __float_as_int(a.tree.nhi[node].w);
    const int e0 = node + 1 < n_nodes ? __float_as_int(a.tree.nhi[node + 1].w) : a.n;
    const int q = s0 + lane;
    const bool is_t = q < e0 && a.state[q] == ST_NEED_HIST;
    unsigned pend = __ballot_sync(FULL, is_t);
    // a cell of more than 32 particles (a run of identical keys): the rest go
    // to the general kernel
    for (int r = s0 + 32 + lane; r < e0; r += 32)
      if (a.state[r] == ST_NEED_HIST) a.fb_list[atomicAdd(a.fb_count, 1)] = (uint32_t)r;
    if (!pend) continue;
    // per-lane target state (lane = particle of the cell)
    float4 myq = make_float4(0.f, 0.f, 0.f, 0.f);
    float myR = 0.f, Rlo = 0.f, Rhi = INFINITY;
    int tries = 0;
    if (is_t) {
      myq = posj[q];
      myR = fminf(a.radius[q] * r0f, a.rmax);
    }
    float hmax = 0.f;    // largest converged h in the cell so far
    float Dw = -1.f;     // radius the cell's hit list covers (< 0: no walk yet)
    int nch = 0;         // hit cells of the cell walk
    bool cover = false;  // the cell walk overflowed its capacity
    const float4 cbl = a.tree.nlo[node], cbh = a.tree.nhi[node];  // the cell's (tight) box
    const int4 an = a.tree.anc4[node];
    while (pend) {
      // ---- the group: the next (up to) G pending targets; the first group of
      // a cell (no h known yet) is smaller, with longer lists ----
      const int gmax = hmax > 0.f ? G : first_g;
      const int capg = (G * lcap) / gmax;
      unsigned gm = 0;
      int gc = 0;
      {
        unsigned t = pend;
        while (t && gc < gmax) {
          gm |= t & (0u - t);
          t &= t - 1u;
          ++gc;
        }
      }
      const bool in_g = (gm >> lane) & 1u;
      const int slot = __popc(gm & lt);
      const int kind = tries > 0 ? 2 : hmax > 0.f ? 1 : 0;  // debug: retry, from the cell's h, from R0
      if (in_g && tries == 0 && hmax > 0.f) myR = fminf(fmaxf(margin * hmax, Rlo * 1.03f), a.rmax);
      if (in_g) {
        S.tgt[slot] = make_float4(myq.x, myq.y, myq.z, myR * myR);
        S.ir2[slot] = 1.0f / (myR * myR);
        S.tp[slot] = q;
        S.ne[slot] = 0;
        S.rnew[slot] = 0.f;
      }
#pragma unroll
      for (int t = 0; t < G; ++t) S.hist[t][lane] = 0u;
      float gR = in_g ? myR : 0.f;
      for (int o = 16; o; o >>= 1) gR = fmaxf(gR, __shfl_xor_sync(FULL, gR, o));
      __syncwarp();
      // ---- the cell walk: every cell within D of the cell box, for each image
      // shift whose region meets the root box (D = the largest pending radius;
      // walked again only when a group needs more) ----
      if (!(gR <= Dw)) {
        float D = is_t && ((pend >> lane) & 1u) ? myR : 0.f;
        for (int o = 16; o; o >>= 1) D = fmaxf(D, __shfl_xor_sync(FULL, D, o));
        D = fmaxf(D, gR);
        const float D2 = D * D * (1.0f + 16.0f * kEps);
        unsigned shifts = 1u << kCenter;
        if (a.periodic) {
          bool want = false;
          if (lane < 27 && lane != kCenter) {
            const double sx = lane / 9 - 1, sy = (lane / 3) % 3 - 1, sz = lane % 3 - 1;
            const float4 l4 = a.tree.nlo[0], h4 = a.tree.nhi[0];
            const float lx = (float)((double)cbl.x - sx * a.box), hx = (float)((double)cbh.x - sx * a.box);
            const float ly = (float)((double)cbl.y - sy * a.box), hy = (float)((double)cbh.y - sy * a.box);
            const float lz = (float)((double)cbl.z - sz * a.box), hz = (float)((double)cbh.z - sz * a.box);
            const float gx = fmaxf(fmaxf(l4.x - hx, lx - h4.x) - sl, 0.f);
            const float gy = fmaxf(fmaxf(l4.y - hy, ly - h4.y) - sl, 0.f);
            const float gz = fmaxf(fmaxf(l4.z - hz, lz - h4.z) - sl, 0.f);
            want = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= D2;
          }
          shifts |= __ballot_sync(FULL, want);
        }
        nch = 0;
        cover = shifts != (1u << kCenter) && !img_ok;
        for (unsigned sm = shifts; sm && !cover;) {
          const int sidx = (sm >> kCenter) & 1u ? kCenter : __ffs(sm) - 1;  // the unshifted image first
          sm &= ~(1u << sidx);
          const bool shifted = sidx != kCenter;
          float rlx = cbl.x, rly = cbl.y, rlz = cbl.z, rhx = cbh.x, rhy = cbh.y, rhz = cbh.z, slk = 0.f;
          if (shifted) {
            const double dsx = (sidx / 9 - 1) * a.box, dsy = ((sidx / 3) % 3 - 1) * a.box,
                         dsz = (sidx % 3 - 1) * a.box;
            rlx = (float)((double)cbl.x - dsx); rhx = (float)((double)cbh.x - dsx);
            rly = (float)((double)cbl.y - dsy); rhy = (float)((double)cbh.y - dsy);
            rlz = (float)((double)cbl.z - dsz); rhz = (float)((double)cbh.z - dsz);
            slk = sl;
          }
          // start: the lowest of the cell's first four ancestors holding the region
          int start = a.tree.root_start;
          if (!shifted) {
            const float Dm = D * (1.0f + 8.0f * kEps);
            const int my_anc = lane == 0 ? an.x : lane == 1 ? an.y : lane == 2 ? an.z : lane == 3 ? an.w : -1;
            bool holds = false;
            if (my_anc >= 0) {
              const float4 l4 = a.tree.nlo[my_anc], h4 = a.tree.nhi[my_anc];
              holds = l4.x <= rlx - Dm && rhx + Dm <= h4.x && l4.y <= rly - Dm && rhy + Dm <= h4.y &&
                      l4.z <= rlz - Dm && rhz + Dm <= h4.z;
            }
            const unsigned hm = __ballot_sync(FULL, holds);
            if (hm) start = __shfl_sync(FULL, my_anc, __ffs(hm) - 1);
          }
          if (lane == 0) S.stk[0] = start;
          int top = 1;
          __syncwarp();
          while (top > 0) {
            const int np = min(top, 4);
            top -= np;
            const int pi = lane >> 3;
            const int par = pi < np ? S.stk[top + pi] : -1;
            __syncwarp();
            bool hit = false;
            int cid = 0;
            if (par >= 0) {
              const float4 *rec = crec + 16 * (size_t)par + 2 * (lane & 7);
              const float4 l4 = rec[0], h4 = rec[1];
              const float gx = fmaxf(fmaxf(l4.x - rhx, rlx - h4.x) - slk, 0.f);
              const float gy = fmaxf(fmaxf(l4.y - rhy, rly - h4.y) - slk, 0.f);
              const float gz = fmaxf(fmaxf(l4.z - rhz, rlz - h4.z) - slk, 0.f);
              hit = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= D2;
              cid = __float_as_int(l4.w);
            }
            const bool is_cell = cid < 0;
            const unsigned pm = __ballot_sync(FULL, hit && !is_cell);
            if (top + __popc(pm) > kGStack) { cover = true; break; }
            if (hit && !is_cell) S.stk[top + __popc(pm & lt)] = cid;
            top += __popc(pm);
            const unsigned cm = __ballot_sync(FULL, hit && is_cell);
            if (nch + __popc(cm) > kCHits) { cover = true; break; }
            if (hit && is_cell)
              S.crec_i[nch + __popc(cm & lt)] = ((unsigned)par * 8u + (unsigned)(lane & 7)) | ((unsigned)sidx << 27);
            nch += __popc(cm);
            __syncwarp();
          }
        }
        Dw = D;
        __syncwarp();
      }
      // ---- the group's cells: the cell walk's hits culled by the target spheres,
      // with their offsets in the candidate stream ----
      int nh = 0, tot = 0;
      bool over = cover;
      for (int e0r = 0; e0r < nch && !over; e0r += 32) {
        const int e = e0r + lane;
        unsigned mk = 0;
        int cs = 0, cl = 0, sidx = kCenter;
        if (e < nch) {
          const unsigned ri = S.crec_i[e];
          sidx = (int)(ri >> 27);
          const float4 *rec = crec + 2 * (size_t)(ri & kIdxMask);
          const float4 l4 = rec[0], h4 = rec[1];
          if (sidx == kCenter) {
#pragma unroll
            for (int t = 0; t < G; ++t) {
              if (t < gc) {
                const float4 T = S.tgt[t];
                const float tx = fmaxf(fmaxf(l4.x - T.x, T.x - h4.x), 0.f);
                const float ty = fmaxf(fmaxf(l4.y - T.y, T.y - h4.y), 0.f);
                const float tz = fmaxf(fmaxf(l4.z - T.z, T.z - h4.z), 0.f);
                if ((tx * tx + ty * ty + tz * tz) * (1.0f - 4.0f * kEps) <= T.w) mk |= 1u << t;
              }
            }
          } else {
            const double dsx = (sidx / 9 - 1) * a.box, dsy = ((sidx / 3) % 3 - 1) * a.box,
                         dsz = (sidx % 3 - 1) * a.box;
#pragma unroll
            for (int t = 0; t < G; ++t) {
              if (t < gc) {
                const float4 T = S.tgt[t];
                const float qx = (float)((double)T.x - dsx), qy = (float)((double)T.y - dsy),
                            qz = (float)((double)T.z - dsz);
                const float tx = fmaxf(fmaxf(l4.x - qx, qx - h4.x) - sl, 0.f);
                const float ty = fmaxf(fmaxf(l4.y - qy, qy - h4.y) - sl, 0.f);
                const float tz = fmaxf(fmaxf(l4.z - qz, qz - h4.z) - sl, 0.f);
                if ((tx * tx + ty * ty + tz * tz) * (1.0f - 4.0f * kEps) <= T.w) mk |= 1u << t;
              }
            }
          }
          if (mk) {
            cs = ~__float_as_int(l4.w);
            cl = __float_as_int(h4.w) - cs;
          }
        }
        const bool ch = cl > 0;
        const unsigned cm = __ballot_sync(FULL, ch);
        if (nh + __popc(cm) > kGHits) { over = true; break; }
        int incl = cl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += v;
        }
        if (ch) {
          const int w = nh + __popc(cm & lt);
          S.hrec[w] = make_int2(cs, tot + incl - cl);
          S.hmeta[w] = (unsigned short)(mk | ((unsigned)sidx << 8));
        }
        nh += __popc(cm);
        tot += __shfl_sync(FULL, incl, 31);
      }
      __syncwarp();
      if (lane < gc) S.res[lane] = R_FALL;
      if (!over) {
        // ---- stream: cp.async ring of 32-slot chunks, kRing - 1 ahead; a slot's
        // cell from the cells starting inside its chunk (one OR-reduced mask) ----
        const int nchunk = (tot + 31) >> 5;
#if SPH_GROUP_DEBUG
        dbg_chunks += nchunk;
        ++dbg_groups;
#endif
        const unsigned ring_s = smem_u32(&S.ring[0][lane]);
        const unsigned lemask = (2u << lane) - 1u;
        int ra = 0;  // hit cell holding the first slot of the next chunk to issue
        auto issue = [&](int qi) {
          if (qi < nchunk) {
            const int c0 = qi << 5;
            const int r = ra + lane;
            const int off = r < nh ? S.hrec[r].y : 0x7fffffff;
            const unsigned d = (unsigned)(off - c0 - 1);
            const unsigned M = __reduce_or_sync(FULL, d < 31u ? 2u << d : 0u);  // cells starting in (c0, c0 + 32)
            const int owner = ra + __popc(M & lemask);
            const int slc = c0 + lane;
            const int rs = qi & (kRing - 1);
            unsigned mt = 0;
            if (slc < tot) {
              const int2 h = S.hrec[owner];
              mt = S.hmeta[owner];
              cp_async16s(ring_s + (unsigned)rs * 512u, pos4 + h.x + (slc - h.y));
            }
            S.meta[rs][lane] = mt;
            // the cell holding slot c0 + 32
            const int pm = __popc(M);
            int step = pm + (__any_sync(FULL, off == c0 + 32) ? 1 : 0);
            if (pm == 31 && ra + 32 < nh && S.hrec[ra + 32].y == c0 + 32) step = 32;
            ra += step;
          }
          cp_async_commit();
        };
#pragma unroll 1
        for (int i = 0; i < kRing - 1; ++i) issue(i);
        int ne[G];
#pragma unroll
        for (int t = 0; t < G; ++t) ne[t] = 0;
        const unsigned hist_s = smem_u32(&S.hist[0][0]);
#pragma unroll 1
        for (int qc = 0; qc < nchunk; ++qc) {
          issue(qc + kRing - 1);
          cp_async_wait<kRing - 1>();
          const int rs = qc & (kRing - 1);
          const float4 c = S.ring[rs][lane];
          const unsigned mt = S.meta[rs][lane];
          const unsigned mk = mt & 0xffu;
          tests += __popc(mk);
          const unsigned om = __reduce_or_sync(FULL, mk);
#if SPH_GROUP_DEBUG
          dbg_tc += __popc(om);
#endif
          const int sidx = (int)(mt >> 8);
          const bool img = mk != 0 && sidx != kCenter;
          float cx = c.x, cy = c.y, cz = c.z;
          double dcx = 0.0, dcy = 0.0, dcz = 0.0;
          const bool any_img = __any_sync(FULL, img);
          if (any_img) {
            // image chunk: x_j + s*box - x_i in fp64 (the reference's image
            // arithmetic), rounded once to fp32
            const int sx = img ? sidx / 9 - 1 : 0, sy = img ? (sidx / 3) % 3 - 1 : 0, sz = img ? sidx % 3 - 1 : 0;
            dcx = __dadd_rn((double)c.x, sx * a.box);
            dcy = __dadd_rn((double)c.y, sy * a.box);
            dcz = __dadd_rn((double)c.z, sz * a.box);
          }
#pragma unroll
          for (int t = 0; t < G; ++t) {
            if ((om >> t) & 1u) {
              const float4 T = S.tgt[t];
              float dx, dy, dz;
              if (!any_img) {
                dx = cx - T.x; dy = cy - T.y; dz = cz - T.z;
              } else {
                dx = (float)__dsub_rn(dcx, (double)T.x);
                dy = (float)__dsub_rn(dcy, (double)T.y);
                dz = (float)__dsub_rn(dcz, (double)T.z);
              }
              const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
              const bool in = ((mk >> t) & 1u) && d2 <= T.w;
              const unsigned b = __ballot_sync(FULL, in);
              if (in) {
                const int w = ne[t] + __popc(b & lt);
                if (w < capg) {
                  sts_v2(lists_s + (unsigned)(t * capg + w) * 8u, __float_as_uint(d2), __float_as_uint(c.w));
                  sts_u16(lslots_s + (unsigned)(t * capg + w) * 2u, (unsigned)((qc << 5) + lane));
                }
                else atoms_inc(hist_s + (unsigned)(t * 32 + vbin(d2 * S.ir2[t])) * 4u);  // beyond the list: count only
              }
              ne[t] += __popc(b);
            }
          }
        }
        cp_async_wait<0>();
        if (lane == 0) {
#pragma unroll
          for (int t = 0; t < G; ++t)
            if (t < gc) S.ne[t] = ne[t];
        }
        __syncwarp();
        // ---- per target: histogram of its list, exact select and density ----
        for (int t = 0; t < gc; ++t) {
          const int nt = S.ne[t];
          const float4 T = S.tgt[t];
          const float ir2 = S.ir2[t];
          int res;
          double d2k = 0.0;
          float rnew = 0.f;
          if (nt < K + 1) {
            res = R_FEW;  // the target itself is in the list
          } else {
            const uint2 *lt_list = lists + t * capg;
            const int nl = min(nt, capg);
            for (int i = lane; i < nl; i += 32)
              atoms_inc(hist_s + (unsigned)(t * 32 + vbin(__uint_as_float(lt_list[i].x) * ir2)) * 4u);
            __syncwarp();
            if (nt > capg) {
              res = R_FULL;
              // the histogram holds every entry within R: a radius whose count
              // fits the list and holds the (K+1)-th surely exists when the bin
              // after the (K+1)-th's still fits
              const unsigned hc = S.hist[t][lane];
              unsigned hin = hc;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const unsigned v = __shfl_up_sync(FULL, hin, o);
                if (lane >= o) hin += v;
              }
              const int B = __ffs(__ballot_sync(FULL, (int)hin >= K + 1)) - 1;
              if (B >= 0 && B < 31 && (int)__shfl_sync(FULL, hin, B + 1) <= capg) {
                const float e = ((float)B + 1.5f) * (1.0f / 32.0f);  // mid bin B+1 in (d2/R^2)^1.5
                rnew = sqrtf(T.w * cbrtf(e * e));
              }
            } else {
              res = select_density<DENS64>(a, lt_list, lslots + t * capg, nt, S.hist[t], S.hrec, S.hmeta, nh,
                                           S.tp[t], T.x, T.y, T.z, T.w, ir2, S.binv, S.band, accepted, d2k);
            }
          }
          if (lane == 0) {
            S.res[t] = res;
            S.d2k[t] = d2k;
            S.rnew[t] = rnew;
          }
          __syncwarp();
        }
      } else {
        ++nfb_walk;
      }
      __syncwarp();
      // ---- outcomes: done, fallback, or a new radius for a later group ----
      bool fall = false, done = false;
      if (in_g) {
        const int res = S.res[slot];
        const int others = S.ne[slot] - 1;
        if (res == R_DONE) {
          done = true;
          hmax = fmaxf(hmax, (float)sqrt(S.d2k[slot]));
        } else if (res == R_FALL) {
          fall = true;
          if (!over) ++nfb_sel;
        } else {
          if (a.kn_counters && kind < 2) atomicAdd(a.kn_counters + 12 + 3 * kind + res, 1);
          ++tries;
          ++nretry;
          float Rn;
          if (res == R_FEW) {
            Rlo = fmaxf(Rlo, myR);
            Rn = myR * fminf(fmaxf(cbrtf(1.3f * (float)(K + 1) / (float)max(others, 1)), 1.15f), 4.0f);
          } else if (res == R_FULL) {
            Rhi = fminf(Rhi, myR);
            const float rn = S.rnew[slot];
            Rn = rn > 0.f ? rn : myR * fminf(fmaxf(cbrtf(1.25f * (float)(K + 1) / (float)others), 0.4f), 0.95f);
          } else {  // the K-th at the list edge
            Rlo = fmaxf(Rlo, myR * 0.999f);
            Rn = myR * 1.08f;
          }
          Rn = fminf(Rn, a.rmax);
          if (Rhi < INFINITY) Rn = fminf(Rn, Rhi * 0.97f);
          Rn = fmaxf(Rn, Rlo * 1.03f);
          if (tries > kMaxTries || !(Rn < Rhi) || !(Rn > Rlo) || (res != R_FULL && myR >= a.rmax)) {
            fall = true;
            ++nfb_tries;
          } else {
            myR = Rn;
          }
        }
        if (fall) a.fb_list[atomicAdd(a.fb_count, 1)] = (uint32_t)q;
      }
      for (int o = 16; o; o >>= 1) hmax = fmaxf(hmax, __shfl_xor_sync(FULL, hmax, o));
      pend &= ~__ballot_sync(FULL, done || fall);
    }
  }
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  tests = __reduce_add_sync(FULL, tests);
  // the walk counter is per warp; the others per lane
  const int nsel = (int)__reduce_add_sync(FULL, (unsigned)nfb_sel);
  const int ntries = (int)__reduce_add_sync(FULL, (unsigned)nfb_tries);
  const int nret = (int)__reduce_add_sync(FULL, (unsigned)nretry);
  if (lane == 0) {
    atomicAdd(&a.stats[0], (unsigned long long)tests);
    atomicAdd(&a.stats[1], accepted);
    if (a.kn_counters) {
      if (nfb_walk) atomicAdd(a.kn_counters + 0, nfb_walk);
      if (nret) atomicAdd(a.kn_counters + 1, nret);
      if (ntries) atomicAdd(a.kn_counters + 2, ntries);
      if (nsel) atomicAdd(a.kn_counters + 3, nsel);
#if SPH_GROUP_DEBUG
      atomicAdd(a.kn_counters + 19, dbg_tc);
      atomicAdd(a.kn_counters + 20, dbg_chunks);
      atomicAdd(a.kn_counters + 21, dbg_groups);
#endif
    }
  }
}

template <int G>
size_t cell_smem(int lcap) {
  return kGWarps * (sizeof(GroupSmem<G>) + (size_t)G * lcap * (sizeof(uint2) + sizeof(unsigned short)));
}

template <int G, bool D64>
void launch_c(cudaStream_t s, const PassArgs &a, const int *cellnode, const int *ncells, int lcap, float margin,
              float r0f, int first_g, int num_sms) {
  const size_t smem = cell_smem<G>(lcap);
  int bps = 0;
  cudaFuncSetAttribute(k_cell<G, D64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_cell<G, D64>, kGWarps * 32, smem);
  k_cell<G, D64><<<num_sms * std::max(bps, 1), kGWarps * 32, smem, s>>>(a, cellnode, ncells, lcap, margin, r0f,
                                                                              std::min(std::max(first_g, 1), G));
}

}  // namespace

int group_list_cap(int k) { return std::min(std::max(5 * k / 2, 96), 512); }

void launch_group(cudaStream_t s, const PassArgs &a, const int *cellnode, const int *ncells, int lcap, float margin,
                  float r0f, int first_g, int num_sms, int g) {
  if (g == 4) {
    if (a.dens64) launch_c<4, true>(s, a, cellnode, ncells, lcap, margin, r0f, first_g, num_sms);
    else launch_c<4, false>(s, a, cellnode, ncells, lcap, margin, r0f, first_g, num_sms);
  } else {
    if (a.dens64) launch_c<8, true>(s, a, cellnode, ncells, lcap, margin, r0f, first_g, num_sms);
    else launch_c<8, false>(s, a, cellnode, ncells, lcap, margin, r0f, first_g, num_sms);
  }
}

}  // namespace sph
