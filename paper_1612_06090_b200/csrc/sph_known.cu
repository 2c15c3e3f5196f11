// sph_known.cu -- the pass for targets whose search radius is already known
// to be close: every non-seed target, whose radius R is 1.1 x the converged
// h of the seeds around it in sorted (= spatial) order.  This is the bulk of
// the work (11 of every 12 targets).
//
// For target i (reference compute_density_pass, density.py:286-413: the
// todo loop is replaced by a radius that bounds the K-th neighbour; the
// reference's todo trace is rebuilt from h0 and d2_K in k_finalize):
//   cull    the cell list of i's cell (every cell within D >= R of the cell
//           box, k_cell_lists) against the sphere (i, R): one record per
//           lane, hits compacted with their stream offsets (one warp scan);
//   stage   the hit cells -- contiguous runs of the sorted float4 array --
//           are copied global -> shared with cp.async.bulk (one bulk copy per
//           cell, issued by the lane that found it) completing on a per-warp
//           mbarrier; batches of up to kStage candidates;
//   list    each staged candidate is tested in fp32 (lanes over candidates,
//           LDS reads) and appended to the target's shared-memory list
//           {sorted index, fp32 d2} when d2 <= R^2 (ballot + popc);
//   select  a 32-bin histogram of (d2/R^2)^1.5 (equal expected counts per
//           bin) finds the bin of the K-th other; the fp32 K-th is ranked
//           inside it; then every list entry within a relative 2^-20 guard
//           of the band [v(1-3e), v(1+3e)] around it gets the exact unfused
//           fp64 d2 (octree.py:211-214 arithmetic) and the exact K-th is
//           counted and ranked (density.py:226-245: h = sqrt(d2_K));
//   sum     rho = sum over list entries within h of m_j W(r/h), self
//           included (density.py:160-171, 249-261; kernel.py:30-45), fp32
//           per pair or fp64 term-for-term (dens64).
// Targets this kernel cannot finish (a periodic image within R, fewer than
// K others or more than the list holds within R, the K-th at the list edge,
// a crowded bin or band) are appended to a list for the general per-target
// kernel (k_target, sph_warp.cu), which grows its own radius.
#include "sph_internal.cuh"

#include <algorithm>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kKWarps = 4;
constexpr float kEps = 9.5367431640625e-07f;  // 2^-20 relative guard (fp32 d2 vs exact)
constexpr double kEpsD = 9.5367431640625e-07;
#ifndef SPH_KNOWN_STAGE
#define SPH_KNOWN_STAGE 512
#endif
constexpr int kStage = SPH_KNOWN_STAGE;  // staged candidates per batch (16 B each)
constexpr int kHits = 192;               // hit cells per target (>= the cell-list capacity)

// per-warp shared memory
struct alignas(16) KnownSmem {
  float4 stage[kStage];
  int2 hits[kHits];     // (first sorted position, stream offset) of each hit cell
  unsigned hist[32];
  unsigned binv[32];    // fp32 d2 bits of the K-th's bin members
  double band[32];      // exact d2 of the band around the K-th
  unsigned long long mbar;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <bool DENS64>
__global__ void __launch_bounds__(kKWarps * 32) k_known(const PassArgs a, int lcap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  KnownSmem &S = reinterpret_cast<KnownSmem *>(smem_raw)[wib];
  uint2 *list = reinterpret_cast<uint2 *>(smem_raw + kKWarps * sizeof(KnownSmem)) + (size_t)wib * lcap;
  const float4 *__restrict__ posj = a.posj;
  const float4 *__restrict__ pos = reinterpret_cast<const float4 *>(a.pos);
  const unsigned lt = (1u << lane) - 1u;
  const int K = a.k;
  const double norm = a.kernel_kind == 0 ? kWc6Norm : kM4Norm;
  if (lane == 0) mbar_init(&S.mbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned phase = 0;
  unsigned long long tests = 0, accepted = 0;
  int nfb0 = 0, nfb1 = 0, nfb2 = 0, nfb3 = 0;  // fallback reasons

  const int count = a.list ? *a.list_count : a.static_count;
  int t_pref = 0;
  if (lane == 0) t_pref = atomicAdd(a.work_counter, 32);
  for (;;) {
    const int t0 = __shfl_sync(FULL, t_pref, 0);
    if (t0 >= count) break;
    if (lane == 0) t_pref = atomicAdd(a.work_counter, 32);
    const int q = t0 + lane;
    int pq = -1;
    if (q < count) {
      pq = a.list ? (int)a.list[q] : q;
      if (a.state[pq] != ST_NEED_HIST) pq = -1;
    }
    unsigned pend = __ballot_sync(FULL, pq >= 0);
    while (pend) {
      const int src = __ffs(pend) - 1;
      pend &= pend - 1u;
      const int p = __shfl_sync(FULL, pq, src);
      int why = -1;  // fallback reason, -1: done here
      const float4 tq = posj[p];
      const float fx = tq.x, fy = tq.y, fz = tq.z;
      const float R = a.radius[p];
      const float R2 = R * R;
      do {
        // ---- a periodic image within R: the general kernel walks images ----
        if (a.periodic) {
          bool img = false;
          if (lane < 27 && lane != 13) {
            const int sx = lane / 9 - 1, sy = (lane / 3) % 3 - 1, sz = lane % 3 - 1;
            const float4 l4 = a.tree.nlo[0], h4 = a.tree.nhi[0];
            const float qx = (float)((double)fx - sx * a.box), qy = (float)((double)fy - sy * a.box),
                        qz = (float)((double)fz - sz * a.box);
            const float sl = (float)a.box * 4.8e-7f;
            const float gx = fmaxf(fmaxf(l4.x - qx, qx - h4.x) - sl, 0.f);
            const float gy = fmaxf(fmaxf(l4.y - qy, qy - h4.y) - sl, 0.f);
            const float gz = fmaxf(fmaxf(l4.z - qz, qz - h4.z) - sl, 0.f);
            img = (gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= R2;
          }
          if (__ballot_sync(FULL, img)) { why = 0; break; }
        }
        // ---- the cell list of the target's cell ----
        const int ci = a.cellidx[a.tree.cellof[p]];
        int llen = ci >= 0 ? a.clen[ci] : -1;
        if (llen < 0 || !(R2 <= a.crad2[ci])) { why = 0; break; }
        const int lnear = a.cnear[ci];
        const int lfar_off = a.clcap - llen;
        if (R2 <= a.near_frac2 * a.crad2[ci] * (1.0f - 16.0f * kEps)) llen = lnear;
        const unsigned *cl = a.clist + (size_t)ci * a.clcap;
        // ---- cull: hit cells with their stream offsets ----
        int nh = 0, tot = 0;
        for (int e0 = 0; e0 < llen; e0 += 32) {
          const int e = e0 + lane;
          int st = 0, ln = 0;
          if (e < llen) {
            const float4 *rec = a.tree.crec + 2 * (size_t)cl[e < lnear ? e : e + lfar_off];
            const float4 l4 = rec[0], h4 = rec[1];
            const float gx = fmaxf(fmaxf(l4.x - fx, fx - h4.x), 0.f);
            const float gy = fmaxf(fmaxf(l4.y - fy, fy - h4.y), 0.f);
            const float gz = fmaxf(fmaxf(l4.z - fz, fz - h4.z), 0.f);
            if ((gx * gx + gy * gy + gz * gz) * (1.0f - 4.0f * kEps) <= R2) {
              st = ~__float_as_int(l4.w);
              ln = __float_as_int(h4.w) - st;
            }
          }
          int incl = ln;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
          }
          const unsigned hm = __ballot_sync(FULL, ln > 0);
          if (ln > 0) S.hits[nh + __popc(hm & lt)] = make_int2(st, tot + incl - ln);
          nh += __popc(hm);
          tot += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
        // ---- stage (cp.async.bulk) and list, batch by batch ----
        int ne = 0;
        bool over = false;
        for (int bh = 0; bh < nh;) {
          const int boff = S.hits[bh].y;
          // the batch: the hits (at most 32) whose runs end within kStage of boff
          const int i = bh + lane;
          const int iend = i < nh ? (i + 1 < nh ? S.hits[i + 1].y : tot) : 0x7fffffff;
          const unsigned bm = __ballot_sync(FULL, iend - boff <= kStage);
          const int nbh = __popc(bm);  // a prefix: the ends grow with i
          const int bend = __shfl_sync(FULL, iend, nbh - 1);
          const int nb = bend - boff;
          if (lane == 0) mbar_arrive_expect_tx(&S.mbar, (unsigned)nb * 16u);
          __syncwarp();
          if (lane < nbh) {
            const int2 h = S.hits[i];
            fence_proxy_async();
            bulk_g2s(&S.stage[h.y - boff], posj + h.x, (unsigned)(iend - h.y) * 16u, &S.mbar);
          }
          while (!mbar_try_wait(&S.mbar, phase)) {
          }
          phase ^= 1u;
          tests += (unsigned)nb;
          for (int s0 = 0; s0 < nb; s0 += 32) {
            const int s = s0 + lane;
            bool in = false;
            float d2 = 0.f;
            unsigned j = 0;
            if (s < nb) {
              const float4 c = S.stage[s];
              const float dx = c.x - fx, dy = c.y - fy, dz = c.z - fz;
              d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
              in = d2 <= R2;
              j = __float_as_uint(c.w);
            }
            const unsigned m = __ballot_sync(FULL, in);
            if (ne + __popc(m) > lcap) { over = true; break; }
            if (in) list[ne + __popc(m & lt)] = make_uint2(j, __float_as_uint(d2));
            ne += __popc(m);
          }
          __syncwarp();
          if (over) break;
          bh += nbh;
        }
        if (over) { why = 1; break; }
        if (ne - 1 < K) { why = 2; break; }  // the target itself is in the list
        // ---- select: bin of the K-th other in (d2/R^2)^1.5 ----
        const float invR2 = 1.0f / R2;
        S.hist[lane] = 0u;
        __syncwarp();
        for (int i = lane; i < ne; i += 32) {
          const uint2 e = list[i];
          if (e.x != (unsigned)p) {
            const float x = __uint_as_float(e.y) * invR2;
            atomicAdd(&S.hist[min(31, (int)(32.0f * x * sqrtf(x)))], 1u);
          }
        }
        __syncwarp();
        const unsigned hc = S.hist[lane];
        unsigned hin = hc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(FULL, hin, o);
          if (lane >= o) hin += v;
        }
        const int B = __ffs(__ballot_sync(FULL, (int)hin >= K)) - 1;  // ne - 1 >= K: exists
        const int rr = K - (int)__shfl_sync(FULL, hin - hc, B);       // rank inside bin B (1-based)
        // the bin's members (fp32 d2 bits)
        int m = 0;
        for (int i0 = 0; i0 < ne; i0 += 32) {
          const int i = i0 + lane;
          bool mine = false;
          unsigned v = 0;
          if (i < ne) {
            const uint2 e = list[i];
            if (e.x != (unsigned)p) {
              const float x = __uint_as_float(e.y) * invR2;
              mine = min(31, (int)(32.0f * x * sqrtf(x))) == B;
              v = e.y;
            }
          }
          const unsigned mm = __ballot_sync(FULL, mine);
          if (mine && m + __popc(mm & lt) < 32) S.binv[m + __popc(mm & lt)] = v;
          m += __popc(mm);
        }
        __syncwarp();
        if (m > 32) { why = 3; break; }
        unsigned vKb;
        {
          const unsigned v = lane < m ? S.binv[lane] : 0xffffffffu;
          int rank = 0;
          for (int l = 0; l < m; ++l) {
            const unsigned u = __shfl_sync(FULL, v, l);
            rank += (u < v) || (u == v && l < lane);
          }
          const unsigned sel = __ballot_sync(FULL, lane < m && rank == rr - 1);
          vKb = __shfl_sync(FULL, v, __ffs(sel) - 1);
        }
        // ---- exact K-th: count below the band, rank inside it ----
        const double vK = (double)__uint_as_float(vKb);
        const double tl = vK * (1.0 - 3.0 * kEpsD), th = vK * (1.0 + 3.0 * kEpsD);
        const float lo_f = __double2float_rd(tl * (1.0 - kEpsD)) - 1e-37f;
        const float hi_f = __double2float_ru(th * (1.0 + kEpsD)) + 1e-37f;
        const double tx = fx, ty = fy, tz = fz;
        int below = 0, nin = 0;
        for (int i0 = 0; i0 < ne; i0 += 32) {
          const int i = i0 + lane;
          bool inb = false;
          double ex = 0.0;
          if (i < ne) {
            const uint2 e = list[i];
            const float af = __uint_as_float(e.y);
            if (e.x != (unsigned)p) {
              if (af < lo_f) {
                ++below;
              } else if (af <= hi_f) {
                const float4 c = posj[e.x];
                ex = exact_d2(__dsub_rn((double)c.x, tx), __dsub_rn((double)c.y, ty), __dsub_rn((double)c.z, tz));
                if (ex < tl) ++below;
                else if (ex <= th) inb = true;
              }
            }
          }
          const unsigned bmk = __ballot_sync(FULL, inb);
          if (inb && nin + __popc(bmk & lt) < 32) S.band[nin + __popc(bmk & lt)] = ex;
          nin += __popc(bmk);
        }
        __syncwarp();
        below = (int)__reduce_add_sync(FULL, (unsigned)below);
        const int r = K - below;
        if (nin > 32 || r < 1 || r > nin) { why = 3; break; }
        double d2k;
        {
          const double v = lane < nin ? S.band[lane] : INFINITY;
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
        if (!(d2k * (1.0 + 4.0 * kEpsD) < (double)R2)) { why = 4; break; }
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
            const uint2 e = list[i];
            const float af = __uint_as_float(e.y);
            if (!(af < d2k_f)) continue;
            ++accepted;
            if constexpr (!DENS64) {
              const float rr_ = af > 0.f ? af * rsqrtf(af) : 0.f;
              const float q = rr_ * inv_h;
              const float wv = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
              if (q < 1.f) accf = fmaf(pos[e.x].w, wv, accf);
            } else {
              const float4 c = posj[e.x];
              const double ex = exact_d2(__dsub_rn((double)c.x, tx), __dsub_rn((double)c.y, ty),
                                         __dsub_rn((double)c.z, tz));
              if (ex < d2k) {
                const double r_ = __dsqrt_rn(ex);
                double wv;
                if (a.kernel_kind == 0) {
                  wv = wc6_lowered(r_, hh, norm_h3);
                } else {
                  const double qq = __ddiv_rn(r_, hh);
                  wv = qq < 1.0 ? norm_h3 * m4_profile(qq) : 0.0;
                }
                accd = __dadd_rn(accd, __dmul_rn(a.mass64[e.x], wv));
              }
            }
          }
          for (int o = 16; o; o >>= 1) {
            accd += __shfl_xor_sync(FULL, accd, o);
            accf += __shfl_xor_sync(FULL, accf, o);
          }
          rho = DENS64 ? accd : __dmul_rn(norm_h3, (double)accf);
        }
        if (lane == 0) {
          a.d2k[p] = d2k;
          a.rho[p] = rho;
          a.state[p] = ST_FINAL;
        }
      } while (false);
      if (why >= 0) {
        if (why == 0) ++nfb0;
        else if (why == 1) ++nfb1;
        else if (why == 2) ++nfb2;
        else ++nfb3;
        if (lane == 0) a.fb_list[atomicAdd(a.fb_count, 1)] = (uint32_t)p;
      }
      __syncwarp();
    }
  }
  for (int o = 16; o; o >>= 1) accepted += __shfl_xor_sync(FULL, accepted, o);
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
    if (a.kn_counters) {
      if (nfb0) atomicAdd(a.kn_counters + 0, nfb0);
      if (nfb1) atomicAdd(a.kn_counters + 1, nfb1);
      if (nfb2) atomicAdd(a.kn_counters + 2, nfb2);
      if (nfb3) atomicAdd(a.kn_counters + 3, nfb3);
    }
  }
}

}  // namespace

int known_max_cells() { return kHits; }

int known_list_cap(int k) { return std::min(std::max(4 * k, 128), 512); }

size_t known_smem_bytes(int lcap) { return kKWarps * (sizeof(KnownSmem) + (size_t)lcap * sizeof(uint2)); }

void launch_known(cudaStream_t s, const PassArgs &a, int lcap, int num_sms) {
  const size_t smem = known_smem_bytes(lcap);
  int bps = 0;
  if (a.dens64) {
    cudaFuncSetAttribute(k_known<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_known<true>, kKWarps * 32, smem);
    k_known<true><<<num_sms * std::max(bps, 1), kKWarps * 32, smem, s>>>(a, lcap);
  } else {
    cudaFuncSetAttribute(k_known<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_known<false>, kKWarps * 32, smem);
    k_known<false><<<num_sms * std::max(bps, 1), kKWarps * 32, smem, s>>>(a, lcap);
  }
}

}  // namespace sph
