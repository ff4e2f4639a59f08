// survey.cu -- on-device pulse generation (NEXT f2): platform + deflector ->
// per-pulse origin / direction / time, written into the chunk's pulse arrays
// right before K6 (helios_simulate_survey).  Reading R30 (DESIGN.md s.3):
//
//   pulse g of a survey is emitted at t = t0 + g / PRF            (P:177 PRF)
//   deflector, u = frac(f t), A = scan angle (Fig. 5):
//     polygon mirror   theta = -A + 2 A u                (parallel lines)
//     fibre optics     theta = -A + 2 A (k + 1/2) / n, k = min(n-1, floor(u n))
//     oscillating      theta = A sin(2 pi f t)           (zig-zag, dense extrema)
//     Palmer           cone of half-angle A off nadir, azimuth 2 pi u
//   scanner frame      s = (0, -sin theta, -cos theta)   (theta > 0: starboard)
//                      Palmer: (sin A cos phi, sin A sin phi, -cos A)
//   head rotation      h = Rz(omega t) s;  mount  m = M h
//   platform   Static (one waypoint) or LinearPath: constant speed
//                      from waypoint to waypoint, yaw towards the next one:
//                      (cos, sin) = (dx, dy) / hypot(dx, dy) of the leg
//   world              d = Rz(yaw) m,  o = P + Rz(yaw) offset   (fp64 -> fp32)
//
// Every fp64 expression uses explicit round-to-nearest intrinsics in the
// operation order of the definition (no FMA contraction).
#include <math.h>

#include "internal.cuh"

namespace helios {
namespace {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ void rot_cs(double c, double s, const double v[3], double out[3]) {
  out[0] = sub(mul(c, v[0]), mul(s, v[1]));
  out[1] = add(mul(s, v[0]), mul(c, v[1]));
  out[2] = v[2];
}

__device__ __forceinline__ void heading(const double d[3], double* c, double* s) {
  const double rho = __dsqrt_rn(add(mul(d[0], d[0]), mul(d[1], d[1])));
  if (rho > 0.0) {
    *c = dvd(d[0], rho);
    *s = dvd(d[1], rho);
  } else {
    *c = 1.0;
    *s = 0.0;
  }
}

__global__ void k_generate(const SurveyArgs a, uint64_t first, uint64_t n, float* __restrict__ o,
                           float* __restrict__ dir, double* __restrict__ time) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g = first + i;
  const double tau = dvd((double)g, a.prf);
  const double t = add(a.t0, tau);
  // deflector
  const double ft = mul(a.f, t);
  const double u = sub(ft, floor(ft));
  const double A = a.A;
  double s[3];
  if (a.deflector == HELIOS_DEFLECTOR_PALMER) {
    const double phi = mul(2.0 * kPi, u);
    s[0] = mul(sin(A), cos(phi));
    s[1] = mul(sin(A), sin(phi));
    s[2] = -cos(A);
  } else {
    double theta;
    if (a.deflector == HELIOS_DEFLECTOR_POLYGON) {
      theta = add(-A, mul(mul(2.0, A), u));
    } else if (a.deflector == HELIOS_DEFLECTOR_FIBRE) {
      const double nf = (double)a.n_fibres;
      const double k = fmin(sub(nf, 1.0), floor(mul(u, nf)));
      theta = add(-A, dvd(mul(mul(2.0, A), add(k, 0.5)), nf));
    } else {
      theta = mul(A, sin(mul(mul(2.0 * kPi, a.f), t)));
    }
    s[0] = 0.0;
    s[1] = -sin(theta);
    s[2] = -cos(theta);
  }
  double h[3], m[3];
  const double ha = mul(a.head, t);
  rot_cs(cos(ha), sin(ha), s, h);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    m[r] = add(add(mul(a.mount[3 * r], h[0]), mul(a.mount[3 * r + 1], h[1])),
               mul(a.mount[3 * r + 2], h[2]));
  // platform
  const double* W = a.waypoints;
  double P[3] = {W[0], W[1], W[2]};
  double yc = 1.0, ys = 0.0;
  if (a.n_waypoints > 1) {
    double T = 0.0;
    bool placed = false;
    int last_leg = -1;
    for (uint32_t k = 0; k + 1 < a.n_waypoints; ++k) {
      const double* p0 = W + 3 * k;
      const double* p1 = p0 + 3;
      const double d[3] = {sub(p1[0], p0[0]), sub(p1[1], p0[1]), sub(p1[2], p0[2])};
      const double len = __dsqrt_rn(add(add(mul(d[0], d[0]), mul(d[1], d[1])), mul(d[2], d[2])));
      if (!(len > 0.0)) continue;
      last_leg = (int)k;
      const double dur = dvd(len, a.speed);
      if (tau < add(T, dur) || k + 2 == a.n_waypoints) {
        const double w = mul(fmin(sub(tau, T), dur), a.speed);
        const double along = fmax(0.0, w);
#pragma unroll
        for (int c = 0; c < 3; ++c) P[c] = add(p0[c], mul(along, dvd(d[c], len)));
        heading(d, &yc, &ys);
        placed = true;
        break;
      }
      T = add(T, dur);
    }
    if (!placed && last_leg >= 0) {
      const double* p0 = W + 3 * last_leg;
      const double* p1 = p0 + 3;
      const double d[3] = {sub(p1[0], p0[0]), sub(p1[1], p0[1]), sub(p1[2], p0[2])};
#pragma unroll
      for (int c = 0; c < 3; ++c) P[c] = p1[c];
      heading(d, &yc, &ys);
    }
  }
  double dw[3], ow[3];
  rot_cs(yc, ys, m, dw);
  rot_cs(yc, ys, a.offset, ow);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    o[3 * i + c] = (float)add(P[c], ow[c]);
    dir[3 * i + c] = (float)dw[c];
  }
  time[i] = t;
}

}  // namespace

cudaError_t launch_generate(const SurveyArgs& a, uint64_t first, uint64_t n, float* origin,
                            float* direction, double* time, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned T = 128;
  k_generate<<<(unsigned)((n + T - 1) / T), T, 0, s>>>(a, first, n, origin, direction, time);
  return cudaGetLastError();
}

}  // namespace helios
