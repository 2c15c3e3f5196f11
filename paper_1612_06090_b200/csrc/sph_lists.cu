// Exact K-th selection and density from the neighbour lists the histogram
// pass recorded (one warp per target).
//
// The histogram pass (sph_pass.cu, MODE_HIST with PassArgs::nlists) leaves,
// per target p, a bracket [t_lo, t_hi] holding the K-th other-neighbour d2
// (the reference's select, density.py:215-246) and a list of every candidate
// it accepted -- all j with fp32 d2 <= its final acceptance radius, which
// covers t_hi by construction -- as particle entries or whole-cell entries.
// This kernel replaces the re-walking select (MODE_BAND) and density
// (MODE_DENS) passes for those targets:
//   1. exact fp64 d2 (octree.py:211-214 arithmetic) for entries whose fp32 d2
//      may lie in the bracket; count the ones below t_lo, collect the ones in it;
//   2. rank selection inside the bracket -> d2_K (h = sqrt(d2_K), density.py:226-245);
//   3. density = sum over entries within h of m_j W(r/h), self term included
//      (density.py:160-171, 249-261; kernel.py:30-45), with the density pass's
//      per-pair arithmetic (fp32, or fp64 term-for-term when dens64).
// The list is held in registers (EPL entries per lane); the fp32 d2 decides
// every entry except the few near the bracket, so only those and the density
// terms gather positions.
// A target whose list overflowed, or whose bracket does not hold the K-th
// (fp32 histogram edge cases), stays in ST_NEED_BAND for the walking passes.
#include "sph_internal.cuh"
#include <cstdio>

namespace sph {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned kCellTag = 0xff000000u;
constexpr double kEpsD = 9.5367431640625e-07;  // 2^-20, as sph_pass.cu
constexpr int kInCap = 256;                    // in-bracket entries per target
constexpr int kWarps = 4;

struct alignas(32) D4 { double x, y, z, m; };
template <bool F32> struct Pos;
template <> struct Pos<true> { using T = float4; };
template <> struct Pos<false> { using T = D4; };

template <bool F32, int EPL>
__global__ void __launch_bounds__(kWarps * 32, 5) k_lists(const PassArgs a, int *fallbacks) {
  using PT = typename Pos<F32>::T;
  __shared__ double s_in[kWarps][kInCap];
  __shared__ int s_nin[kWarps];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  double *inb = s_in[wib];
  const PT *__restrict__ pos = reinterpret_cast<const PT *>(a.pos);
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int center = a.periodic ? 13 : 0;
  const float boxf = (float)a.box;
  const double norm = a.kernel_kind == 0 ? kWc6Norm : kM4Norm;
  const bool f32sum = F32 && !a.dens64;
  unsigned long long tests = 0, accepted = 0;
  int fb = 0, fb_r = 0, fb_in = 0;

  // targets in chunks of 32 (one lane loads each target's scalars), then one
  // warp per target of the chunk
  for (int base = gw * 32; base < a.n; base += nw * 32) {
    const int pl = base + lane;
    int m_l = 0;
    double lo_l = 0.0, hi_l = 0.0;
    PT t_l{};
    bool want = false;
    if (pl < a.n && a.state[pl] == ST_NEED_BAND) {
      m_l = a.ncount[pl];
      if (m_l > a.ncap || m_l > 32 * EPL) {
        ++fb;
        if (m_l <= 0x7ffffffd) a.ncount[pl] = 0x7fffffff;  // overflowed: the collect pass (sph_warp.cu)
      } else {
        want = true;
        lo_l = a.t_lo[pl];
        hi_l = a.t_hi[pl];
        t_l = pos[pl];
      }
    }
    unsigned todo = __ballot_sync(FULL, want);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1u;
      const int p = base + src;
      const int m = __shfl_sync(FULL, m_l, src);
      const uint2 *__restrict__ L = a.nlists + (size_t)p * a.ncap;
      // the list, EPL entries per lane (lane + 32u); absent slots carry a NaN d2
      uint2 ev[EPL];
      bool cell = false;
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int i = lane + 32 * u;
        ev[u] = i < m ? L[i] : make_uint2(0u, 0x7fc00000u);
        cell = cell || (ev[u].y >= kCellTag);
      }
      const double tx = __shfl_sync(FULL, (double)t_l.x, src), ty = __shfl_sync(FULL, (double)t_l.y, src),
                   tz = __shfl_sync(FULL, (double)t_l.z, src);
      const float fx = (float)tx, fy = (float)ty, fz = (float)tz;
      const double lo = __shfl_sync(FULL, lo_l, src), hi = __shfl_sync(FULL, hi_l, src);
      const float lo_f = __double2float_rd(lo * (1.0 - kEpsD)) - 1e-37f;
      const float hi_f = __double2float_ru(hi * (1.0 + kEpsD)) + 1e-37f;
      // exact image d2 (octree.py:211-214 arithmetic)
      auto image_d2 = [&](const PT &c, int sidx) {
        double cx = c.x, cy = c.y, cz = c.z;
        if (a.periodic && sidx != 13) {
          const int sx = sidx / 9 - 1, sy = (sidx / 3) % 3 - 1, sz = sidx % 3 - 1;
          cx = __dadd_rn(cx, sx * a.box); cy = __dadd_rn(cy, sy * a.box); cz = __dadd_rn(cz, sz * a.box);
        }
        return exact_d2(__dsub_rn(cx, tx), __dsub_rn(cy, ty), __dsub_rn(cz, tz));
      };
      auto mass_of = [&](const PT &c, int j) -> double {
        if constexpr (F32) return a.dens64 ? a.mass64[j] : (double)c.w;
        else return c.m;
      };
      const bool slow = __any_sync(FULL, cell);  // whole-cell entries: expanded one by one

      // generic walk over the entries, expanding cells; fn(self, af, c, j, sidx)
      auto for_entries = [&](auto &&fn) {
#pragma unroll 1
        for (int u = 0; u < EPL; ++u) {
          const uint2 e = ev[u];
          if (e.y == 0x7fc00000u) continue;
          const int j0 = (int)(e.x & ((1u << 27) - 1u));
          const int sidx = (int)(e.x >> 27);
          const bool is_cell = e.y >= kCellTag;
          const int cnt = is_cell ? (int)(e.y & 0xffffffu) : 1;
          const int sx = a.periodic ? sidx / 9 - 1 : 0;
          const int sy = a.periodic ? (sidx / 3) % 3 - 1 : 0;
          const int sz = a.periodic ? sidx % 3 - 1 : 0;
          for (int j = j0; j < j0 + cnt; ++j) {
            const PT c = pos[j];
            float af = __uint_as_float(e.y);
            if (is_cell) {
              if constexpr (F32) {
                const float csx = sx < 0 ? -boxf : 0.f, csy = sy < 0 ? -boxf : 0.f, csz = sz < 0 ? -boxf : 0.f;
                const float tfx = sx > 0 ? fx - boxf : fx, tfy = sy > 0 ? fy - boxf : fy,
                            tfz = sz > 0 ? fz - boxf : fz;
                const float dx = (c.x + csx) - tfx, dy = (c.y + csy) - tfy, dz = (c.z + csz) - tfz;
                af = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
              } else {
                af = (float)image_d2(c, sidx);
              }
            }
            fn(j == p && sidx == center, af, c, j, sidx);
          }
        }
      };

      // ---- 1. count below the bracket, collect the bracket ----
      if (lane == 0) s_nin[wib] = 0;
      __syncwarp();
      int below = 0;
      auto classify = [&](bool self, double e, float af) {
        if (self) return;
        if (af < lo_f || e < lo) {
          ++below;
        } else if (e <= hi) {
          const int slot = atomicAdd(&s_nin[wib], 1);
          if (slot < kInCap) inb[slot] = e;
        }
      };
      float mw[EPL];  // fp32 sums: the entry's mass (gathered once)
      if (slow) {
        for_entries([&](bool self, float af, const PT &c, int, int sidx) {
          ++tests;
          if (!(af <= hi_f)) return;
          classify(self, (!self && !(af < lo_f)) ? image_d2(c, sidx) : 0.0, af);
        });
      } else {
        // fp32 d2 decides all but the entries near the bracket (exact fp64
        // there); the fp32 sums gather each candidate mass here, once
        const float *__restrict__ posf = reinterpret_cast<const float *>(a.pos);
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const float af = __uint_as_float(ev[u].y);
          tests += af == af;
          mw[u] = 0.f;
          if (f32sum && af <= hi_f) mw[u] = posf[4 * (size_t)(ev[u].x & ((1u << 27) - 1u)) + 3];
        }
#pragma unroll
        for (int u = 0; u < EPL; ++u) {
          const float af = __uint_as_float(ev[u].y);
          if (af <= hi_f) {
            const int j = (int)(ev[u].x & ((1u << 27) - 1u));
            const int sidx = (int)(ev[u].x >> 27);
            const bool self = j == p && sidx == center;
            const bool near = !self && !(af < lo_f);
            classify(self, near ? image_d2(pos[j], sidx) : 0.0, af);
          }
        }
      }
      __syncwarp();
      below = (int)__reduce_add_sync(FULL, (unsigned)below);
      const int n_in = s_nin[wib];
      const int r = a.k - below;  // 1-based rank of the K-th inside the bracket
      if (n_in > kInCap) { ++fb_in; continue; }
      if (r < 1 || r > n_in) {
        ++fb_r;
        if (lane == 0 && a.dbg && atomicAdd(fallbacks + 3, 1) < 8)
          printf("[lists miss] p=%d m=%d K=%d below=%d n_in=%d lo=%.9g hi=%.9g\n", p, m, a.k, below, n_in, lo, hi);
        continue;
      }

      // ---- 2. the r-th smallest of the bracket ----
      double v = INFINITY;
      for (int i = lane; i < n_in; i += 32) {
        const double ei = inb[i];
        int less = 0, eq = 0;
        for (int j = 0; j < n_in; ++j) {
          const double ej = inb[j];
          less += ej < ei;
          eq += ej == ei;
        }
        if (less < r && r <= less + eq) v = ei;
      }
      for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
      const double d2k = v;

      // ---- 3. density over the entries within h ----
      double rho = 0.0;
      if (d2k > 0.0) {
        double accd = 0.0;
        float accf = 0.f;
        const double hh = __dsqrt_rn(d2k);
        const double norm_h3 = __ddiv_rn(norm, __dmul_rn(__dmul_rn(hh, hh), hh));
        const float d2k_f = __double2float_ru(d2k * (1.0 + kEpsD));
        const float inv_h = (float)(1.0 / hh);
        // one pair term: fp32 (the density pass's arithmetic) or fp64 term-for-term
        auto term = [&](float af, double e, double mj) {
          if (f32sum) {
            const float rr = af > 0.f ? af * rsqrtf(af) : 0.f;
            const float q = rr * inv_h;
            const float w = a.kernel_kind == 0 ? wc6_profile_f(q) : m4_profile_f(q);
            if (q < 1.f) accf = fmaf((float)mj, w, accf);
          } else if (e < d2k) {
            const double r_ = __dsqrt_rn(e);
            double w;
            if (a.kernel_kind == 0) {
              w = wc6_lowered(r_, hh, norm_h3);
            } else {
              const double q = __ddiv_rn(r_, hh);
              w = q < 1.0 ? norm_h3 * m4_profile(q) : 0.0;
            }
            accd = __dadd_rn(accd, __dmul_rn(mj, w));
          }
        };
        if (slow) {
          for_entries([&](bool, float af, const PT &c, int j, int sidx) {
            if (!(af < d2k_f)) return;
            ++accepted;
            term(af, f32sum ? 0.0 : image_d2(c, sidx), mass_of(c, j));
          });
        } else {
#pragma unroll
          for (int u = 0; u < EPL; ++u) {
            const float af = __uint_as_float(ev[u].y);
            if (af < d2k_f) {
              ++accepted;
              if (f32sum) {
                term(af, 0.0, mw[u]);
              } else {
                const int j = (int)(ev[u].x & ((1u << 27) - 1u));
                const PT c = pos[j];
                term(af, image_d2(c, (int)(ev[u].x >> 27)), mass_of(c, j));
              }
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
        a.state[p] = ST_FINAL;
      }
    }
  }
  // statistics
  for (int o = 16; o; o >>= 1) {
    tests += __shfl_xor_sync(FULL, tests, o);
    accepted += __shfl_xor_sync(FULL, accepted, o);
    fb += __shfl_xor_sync(FULL, fb, o);
  }
  if (lane == 0) {
    atomicAdd(&a.stats[0], tests);
    atomicAdd(&a.stats[1], accepted);
    if (fb) atomicAdd(fallbacks, fb);
    if (fb_r) atomicAdd(fallbacks + 1, fb_r);
    if (fb_in) atomicAdd(fallbacks + 2, fb_in);
  }
}

}  // namespace

int lists_max_cap() { return 32 * 16; }

void launch_lists(cudaStream_t s, int f32, const PassArgs &a, int *fallbacks, int num_sms) {
  const int blocks = num_sms * (2048 / (kWarps * 32));
  if (a.ncap <= 256) {
    if (f32) k_lists<true, 8><<<blocks, kWarps * 32, 0, s>>>(a, fallbacks);
    else k_lists<false, 8><<<blocks, kWarps * 32, 0, s>>>(a, fallbacks);
  } else {
    if (f32) k_lists<true, 16><<<blocks, kWarps * 32, 0, s>>>(a, fallbacks);
    else k_lists<false, 16><<<blocks, kWarps * 32, 0, s>>>(a, fallbacks);
  }
}

}  // namespace sph
