// sph_workload.cu -- the clustered generator of BASELINE configs 2-5 on the
// device (SURVEY 8d inputs, 8f "on-device input path").
//
// The reference has no clustered generator; its only generator is
// the counter-based UniformBox stream (workload.py:42-84), and this follows
// the same pattern: every random draw is a pure function of (seed, counter),
// draw t of the stream = splitmix64(seed + (t+1) * GAMMA) >> 11 scaled by
// 2^-53 (workload.py:42-60), so particle i needs no state from particle i-1
// and the whole set is generated in one pass over HBM.
//
// Particle i uses draws t = 8i + j:
//   halo member (i < halo_start[n_halos], halo h = the run holding i):
//     j = 0  NFW radius by inverse CDF: m(x) = ln(1+x) - x/(1+x) inverted by
//            60 bisection steps on [0, x_max], r = x * r_vir / c
//     j = 1  cos(theta) = 2u - 1;  j = 2  phi = 2 pi u   (isotropic)
//   background: j = 0, 1, 2 -> u * box per axis
//   velocities (generated, never read by the pass): Box-Muller from j = 3..6
//     times sigma_h (halo) or 1 (background)
// Positions wrap into [0, box) with numpy's mod semantics and are rounded to
// fp32; an fp32 value that lands on box clamps to nextafter(box, 0).
#include "sph_internal.cuh"

namespace sph {
namespace {

__device__ __forceinline__ double u01(uint64_t seed, uint64_t t) {
  uint64_t s = seed + (t + 1ull) * 0x9E3779B97F4A7C15ull;
  s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ull;
  s = (s ^ (s >> 27)) * 0x94D049BB133111EBull;
  s = s ^ (s >> 31);
  return __dmul_rn(__ull2double_rn(s >> 11), 0x1p-53);
}

__device__ __forceinline__ double nfw_m(double x) { return log1p(x) - x / (1.0 + x); }

// numpy's floor-mod for a positive divisor (npy_divmod)
__device__ __forceinline__ double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) {
    if (m < 0.0) m += b;
  } else {
    m = 0.0;
  }
  return m;
}

__global__ void k_nfw_positions(int64_t n, int64_t n_halos, const int64_t *__restrict__ start,
                                const double *__restrict__ halo, double conc, double x_max, uint64_t seed,
                                double box, float *__restrict__ xo, float *__restrict__ yo, float *__restrict__ zo,
                                float *__restrict__ vel) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t t0 = 8ull * (uint64_t)i;
  const int64_t n_in_halos = start[n_halos];
  double p[3];
  double sigma = 1.0;
  if (i < n_in_halos) {
    int64_t lo = 0, hi = n_halos;  // last h with start[h] <= i
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (start[mid] <= i) lo = mid; else hi = mid;
    }
    const double *hp = halo + 5 * lo;
    const double um = u01(seed, t0) * nfw_m(x_max);
    double a = 0.0, b = x_max;
    for (int it = 0; it < 60; ++it) {
      const double mid = 0.5 * (a + b);
      if (nfw_m(mid) < um) a = mid; else b = mid;
    }
    const double r = 0.5 * (a + b) * (hp[3] / conc);
    const double mu = 2.0 * u01(seed, t0 + 1) - 1.0;
    const double phi = 6.283185307179586 * u01(seed, t0 + 2);
    const double s = sqrt(fmax(0.0, 1.0 - mu * mu));
    double sp, cp;
    sincos(phi, &sp, &cp);
    p[0] = hp[0] + r * (s * cp);
    p[1] = hp[1] + r * (s * sp);
    p[2] = hp[2] + r * mu;
    sigma = hp[4];
  } else {
    p[0] = u01(seed, t0) * box;
    p[1] = u01(seed, t0 + 1) * box;
    p[2] = u01(seed, t0 + 2) * box;
  }
  const float bf = (float)box;
  const float top = nextafterf(bf, 0.0f);
  float f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    f[a] = (float)py_mod(p[a], box);
    if ((double)f[a] >= box) f[a] = top;
  }
  xo[i] = f[0];
  yo[i] = f[1];
  zo[i] = f[2];
  if (vel) {
    const double r1 = sqrt(-2.0 * log(1.0 - u01(seed, t0 + 3)));
    const double r2 = sqrt(-2.0 * log(1.0 - u01(seed, t0 + 5)));
    double s1, c1, s2, c2;
    sincos(6.283185307179586 * u01(seed, t0 + 4), &s1, &c1);
    sincos(6.283185307179586 * u01(seed, t0 + 6), &s2, &c2);
    vel[3 * i + 0] = (float)(sigma * r1 * c1);
    vel[3 * i + 1] = (float)(sigma * r1 * s1);
    vel[3 * i + 2] = (float)(sigma * r2 * c2);
  }
}

}  // namespace

void launch_nfw_positions(cudaStream_t s, int64_t n, int64_t n_halos, const int64_t *start, const double *halo,
                          double conc, double x_max, uint64_t seed, double box, float *x, float *y, float *z,
                          float *vel) {
  if (n <= 0) return;
  k_nfw_positions<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, n_halos, start, halo, conc, x_max, seed, box, x, y,
                                                               z, vel);
}

}  // namespace sph
