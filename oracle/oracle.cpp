/*
 * oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation (C++17, IEEE double)
 * of the HELIOS++ virtual-laser-scanning hot path (arXiv 2101.09154):
 * subray fan-out -> nearest hit (brute force over every triangle) ->
 * transmissive-voxel segments -> radiometry -> full-waveform sum -> peaks.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2101_09154_b200/) never does, and this file shares no code, header,
 * table or constant generator with it.
 *
 * Citations: "P:n" = PAPER.md line n (section / equation named in prose);
 * "R<k>" = the reading with that id in DESIGN.md section 3 (the ambiguity
 * register).  Every function follows the paper's order and notation; where
 * the paper defines a result plainly (a nearest hit, a sum, a local maximum)
 * the function is that definition written out (minimum over ALL triangles,
 * direct sums, a predicate applied to every bin).
 *
 * Parity pins: every exported function is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py against closed forms, printed values, brute force or
 * an independent library (curand's host Philox generator); see DESIGN.md s.4.
 */
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace {

const double kPi = 3.14159265358979323846;
const double kC = 299792458.0;  // speed of light, m/s (Sec. 3.4)
const double kInf = std::numeric_limits<double>::infinity();
const double kNaN = std::numeric_limits<double>::quiet_NaN();
// C-4 exports: at most kMaxCand triangle candidates per subray, kMaxAttr
// attribution candidates per return
const int32_t kMaxCand = 8;
const int32_t kMaxAttr = 4;
// Decision margins below which the CUDA path may legitimately decide the
// other way (C-4; DESIGN.md s.4): it bins the fp32-rounded amplitudes
// (relative error <= 2^-24 = 6e-8 per term, all terms >= 0, so every bin and
// every contribution is within 6e-8 relative of the oracle's), so a
// comparison of two such values can flip only within 1.2e-7 relative;
// 2.5e-7 leaves a factor 2.
const double kDecisionEps = 2.5e-7;

struct V3 {
  double x, y, z;
};
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
double norm(V3 a) { return std::sqrt(dot(a, a)); }

}  // namespace

extern "C" {

/* ------------------------------------------------------------------------
 * Subray pattern (Fig. 6 caption P:204; readings R1, R2, R4).
 * ring i = 1..q carries floor(2*pi*i) subrays; a central subray is
 * always added.  R1: counts reachable by that rule select it; the hexagonal
 * counts 1 + 3q(q+1) select n_i = 6i.  Returns q (>= 0), or -1 if the count
 * is reachable by neither rule.  *rule = 0 paper rule, 1 hexagonal.
 * ---------------------------------------------------------------------- */
int oracle_resolve_subrays(uint32_t count, int* rule) {
  for (int q = 0; q <= 64; ++q) {
    uint64_t n = 1;
    for (int i = 1; i <= q; ++i) n += (uint64_t)std::floor(2.0 * kPi * i);
    if (n == count) {
      if (rule) *rule = 0;
      return q;
    }
  }
  for (int q = 0; q <= 64; ++q) {
    uint64_t n = 1 + 3ull * q * (q + 1);
    if (n == count) {
      if (rule) *rule = 1;
      return q;
    }
  }
  return -1;
}

/* Ring size n_i under the given rule (P:199 / R1). */
static int ring_size(int rule, int i) {
  if (rule == 0) return (int)std::floor(2.0 * kPi * i);
  return 6 * i;
}

/* Per-subray ring index i(s), slot j(s), ring size n_i and angles
 * theta_i = (i/q) * beta (R2), phi = 2*pi*j/n_i (R4).  Order: centre, then
 * rings outward, slots by j (R4).  Returns 0, or -1 on a bad count. */
int oracle_subray_pattern(uint32_t count, double beta, int* ring, int* slot,
                          int* ring_n, double* theta, double* phi) {
  int rule = 0;
  int q = oracle_resolve_subrays(count, &rule);
  if (q < 0) return -1;
  uint32_t s = 0;
  ring[s] = 0;
  slot[s] = 0;
  ring_n[s] = 1;
  theta[s] = 0.0;
  phi[s] = 0.0;
  ++s;
  for (int i = 1; i <= q; ++i) {
    int n = ring_size(rule, i);
    for (int j = 0; j < n; ++j) {
      ring[s] = i;
      slot[s] = j;
      ring_n[s] = n;
      theta[s] = ((double)i / (double)q) * beta;
      phi[s] = 2.0 * kPi * (double)j / (double)n;
      ++s;
    }
  }
  return 0;
}

/* Subray direction ("sampled in a regular pattern around the central
 * ray"; R4 frame): d = pulse direction normalised; a = z unless |d_z| > 0.9,
 * then x; u = normalize(a x d); v = d x u;
 * d_s = cos(theta) d + sin(theta) (cos(phi) u + sin(phi) v). */
void oracle_subray_direction(const double d_in[3], double theta, double phi,
                             double out[3]) {
  V3 d = {d_in[0], d_in[1], d_in[2]};
  d = scale(d, 1.0 / norm(d));
  V3 a = std::fabs(d.z) > 0.9 ? V3{1.0, 0.0, 0.0} : V3{0.0, 0.0, 1.0};
  V3 u = cross(a, d);
  u = scale(u, 1.0 / norm(u));
  V3 v = cross(d, u);
  V3 ring = add(scale(u, std::cos(phi)), scale(v, std::sin(phi)));
  V3 ds = add(scale(d, std::cos(theta)), scale(ring, std::sin(theta)));
  out[0] = ds.x;
  out[1] = ds.y;
  out[2] = ds.z;
}

/* ------------------------------------------------------------------------
 * Eq. 1: I = I0 exp(-2 r^2 / w^2).
 * Eq. 2: w = w0 sqrt(omega0^2 + omega^2), omega = lambda R/(pi w0^2),
 *                omega0 = lambda R0/(pi w0^2).  lambda given in nm.
 * ---------------------------------------------------------------------- */
double oracle_eq1_intensity(double I0, double r, double w) {
  return I0 * std::exp(-2.0 * r * r / (w * w));
}

double oracle_eq2_beam_width(double w0, double lambda_nm, double R, double R0) {
  double lambda = lambda_nm * 1e-9;
  double omega = lambda * R / (kPi * w0 * w0);
  double omega0 = lambda * R0 / (kPi * w0 * w0);
  return w0 * std::sqrt(omega0 * omega0 + omega * omega);
}

/* Subray base intensity I_s at hit range R (R5): r = R sin(theta_i); w from
 * Eq. 2 when w0 > 0, else the far-field specialisation w = R tan(beta). */
double oracle_subray_intensity(double I0, double theta, double beta, double R,
                               double w0, double lambda_nm, double R0) {
  double r = R * std::sin(theta);
  double w = (w0 > 0.0) ? oracle_eq2_beam_width(w0, lambda_nm, R, R0)
                        : R * std::tan(beta);
  if (r == 0.0) return I0;  // beam centre (Eq. 1 with r = 0)
  return oracle_eq1_intensity(I0, r, w);
}

/* Eq. 3: P(t) = I (t/tau)^2 exp(-t/tau), tau = pulse length / 1.75
 * (P:208). */
double oracle_eq3_pulse(double I, double t, double tau) {
  double x = t / tau;
  return I * x * x * std::exp(-x);
}

/* Eq. 7: I = lambda sigma P alpha^2 / (4 pi d^4 beta^2) (R14, R16). */
double oracle_eq7_intensity(double lambda_eff, double sigma, double P,
                            double alpha, double d, double beta) {
  return lambda_eff * sigma * P * alpha * alpha /
         (4.0 * kPi * d * d * d * d * beta * beta);
}

/* ------------------------------------------------------------------------
 * Ray-triangle intersection (triangles have only t0; R21: t > 0,
 * two-sided).  Moller-Trumbore in double on the fp32 vertices promoted to
 * double.  Inclusive edges; |det| <= 1e-12 |e1||e2| is a miss (parallel ray
 * or degenerate triangle).  Returns t, or -1 on a miss; *cos_inc receives
 * |n . d| / |d| (incidence folded to [0, pi/2]).
 * ---------------------------------------------------------------------- */
}  // extern "C"

// The Moller-Trumbore test proper, given the triangle's v0, e1 = v1 - v0,
// e2 = v2 - v0 and cut = 1e-12 |e1| |e2| (computed once per triangle by the
// callers, in oracle_ray_triangle's order: the same values, the same result).
static double ray_triangle_pre(const V3& o, const V3& d, const V3& v0, const V3& e1,
                               const V3& e2, double cut) {
  V3 p = cross(d, e2);
  double det = dot(e1, p);
  if (std::fabs(det) <= cut) return -1.0;
  double inv = 1.0 / det;
  V3 s = sub(o, v0);
  double u = dot(s, p) * inv;
  if (u < 0.0 || u > 1.0) return -1.0;
  V3 q = cross(s, e1);
  double v = dot(d, q) * inv;
  if (v < 0.0 || u + v > 1.0) return -1.0;
  double t = dot(e2, q) * inv;
  if (!(t > 0.0)) return -1.0;
  return t;
}

struct TriPre {
  V3 v0, e1, e2;
  double cut;
};
static TriPre tri_pre(const float* tri9) {
  TriPre r;
  r.v0 = {tri9[0], tri9[1], tri9[2]};
  V3 v1 = {tri9[3], tri9[4], tri9[5]};
  V3 v2 = {tri9[6], tri9[7], tri9[8]};
  r.e1 = sub(v1, r.v0);
  r.e2 = sub(v2, r.v0);
  r.cut = 1e-12 * norm(r.e1) * norm(r.e2);
  return r;
}

extern "C" {

double oracle_ray_triangle(const double o_in[3], const double d_in[3],
                           const float* tri9, double* cos_inc) {
  V3 o = {o_in[0], o_in[1], o_in[2]};
  V3 d = {d_in[0], d_in[1], d_in[2]};
  const TriPre tp = tri_pre(tri9);
  const double t = ray_triangle_pre(o, d, tp.v0, tp.e1, tp.e2, tp.cut);
  if (t < 0.0) return -1.0;
  if (cos_inc) {
    V3 n = cross(tp.e1, tp.e2);
    *cos_inc = std::fabs(dot(n, d)) / (norm(n) * norm(d));
  }
  return t;
}

}  // extern "C"

// Can any ray from o whose direction lies within angle theta of the unit
// vector d hit the triangle?  False only when the triangle's bounding sphere
// (centroid c, radius r = the largest vertex distance) lies entirely outside
// that one-sided cone: with v = c - o, a = v.d, rho = |v - a d|, the
// distance from c to the cone is rho cos(theta) - a sin(theta) when the
// nearest cone point is on its mantle (a cos(theta) + rho sin(theta) >= 0),
// else |v| (the apex).  Used to skip, per pulse, the triangles none of its
// subrays can reach (the brute force then tests every other triangle with
// every subray); theta and r are widened so rounding cannot reject a hit.
static bool cone_may_hit(const V3& o, const V3& d, double cos_t, double sin_t,
                         const TriPre& tp) {
  const V3 v1 = add(tp.v0, tp.e1), v2 = add(tp.v0, tp.e2);
  const V3 c = scale(add(add(tp.v0, v1), v2), 1.0 / 3.0);
  double r2 = dot(sub(tp.v0, c), sub(tp.v0, c));
  r2 = std::max(r2, dot(sub(v1, c), sub(v1, c)));
  r2 = std::max(r2, dot(sub(v2, c), sub(v2, c)));
  const double r = std::sqrt(r2) * (1.0 + 1e-9) + 1e-9;
  const V3 v = sub(c, o);
  const double a = dot(v, d);
  const V3 w = sub(v, scale(d, a));
  const double rho = norm(w);
  if (a * cos_t + rho * sin_t >= 0.0) return rho * cos_t - a * sin_t <= r;
  return norm(v) <= r;
}

typedef std::vector<std::pair<double, uint32_t>> HitList;  // (t, triangle id) of every hit

// The nearest hit and its candidate set from the list of EVERY hit of a ray
// (the definition: minimum of (t, id); C_tri = {t <= t_min + 1e-6 m}).
static int64_t nearest_from_hits(HitList& hits, double* t_out, int32_t* n_cand, double* gap,
                                 uint32_t* cand, int32_t max_cand) {
  std::sort(hits.begin(), hits.end());  // by t, then the lower id (R22)
  const int64_t best_id = hits.empty() ? -1 : (int64_t)hits[0].second;
  const double best = hits.empty() ? kInf : hits[0].first;
  int32_t nc = 0;
  double second = kInf;
  for (const auto& h : hits) {
    if (h.first <= best + 1e-6) {
      if (cand && nc < max_cand) cand[nc] = h.second;
      ++nc;
    }
    if ((int64_t)h.second != best_id) second = std::min(second, h.first);
  }
  if (cand)
    for (int32_t k = nc; k < max_cand; ++k) cand[k] = 0xFFFFFFFFu;
  if (t_out) *t_out = best;
  if (n_cand) *n_cand = nc;
  if (gap) *gap = second - best;
  return best_id;
}

extern "C" {

int64_t oracle_nearest_candidates(const double o[3], const double d[3], const float* tris,
                                  uint32_t n_tris, double* t_out, double* cos_out,
                                  int32_t* n_cand, double* gap, uint32_t* cand,
                                  int32_t max_cand) {
  HitList hits;
  for (uint32_t i = 0; i < n_tris; ++i) {
    double t = oracle_ray_triangle(o, d, tris + 9ull * i, nullptr);
    if (t >= 0.0) hits.push_back({t, i});
  }
  const int64_t id = nearest_from_hits(hits, t_out, n_cand, gap, cand, max_cand);
  double c = 0.0;
  if (id >= 0) oracle_ray_triangle(o, d, tris + 9ull * id, &c);  // the same t, its cos
  if (cos_out) *cos_out = c;
  return id;
}

int oracle_cone_may_hit(const double o[3], const double d[3], double theta, const float* tri9) {
  return cone_may_hit(V3{o[0], o[1], o[2]}, V3{d[0], d[1], d[2]}, std::cos(theta),
                      std::sin(theta), tri_pre(tri9));
}

int64_t oracle_nearest_triangle(const double o[3], const double d[3], const float* tris,
                                uint32_t n_tris, double* t_out, double* cos_out,
                                int32_t* n_cand, double* gap) {
  return oracle_nearest_candidates(o, d, tris, n_tris, t_out, cos_out, n_cand, gap, nullptr, 0);
}

/* Bin of a range (R8, R9): x = 2R / c / Delta (two-way time in bins),
 * k = floor(x); *margin = |x - nearest integer| (C-4: how far the decision
 * floor(x) is from flipping). */
int64_t oracle_bin_of(double R, double delta_ns, double* margin) {
  const double x = 2.0 * R / kC / (delta_ns * 1e-9);
  if (margin) *margin = std::fabs(x - std::nearbyint(x));
  return (int64_t)std::floor(x);
}

/* Transmission decision (Eq. 6; R17): the subray passes the voxel
 * iff u < exp(-sigma L); *margin = |u - exp(-sigma L)| (C-4). */
int oracle_transmits(double u, double sigma, double L, double* margin) {
  const double pass_p = std::exp(-sigma * L);
  if (margin) *margin = std::fabs(u - pass_p);
  return u < pass_p;
}

/* ------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11), written from its published
 * definition (DESIGN.md s.3 R18/R19): rounds (c0..c3) ->
 * (hi(M1 c2) ^ c1 ^ k0, lo(M1 c2), hi(M0 c0) ^ c3 ^ k1, lo(M0 c0)),
 * key bump k0 += 0x9E3779B9, k1 += 0xBB67AE85 between rounds, 10 rounds.
 * ---------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                          uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* Uniform draw R in [0,1) for a transmission decision (R18,
 * R19): key = (seed_lo, seed_hi), ctr = (pulse_lo, pulse_hi, subray, voxel),
 * u = (x0 >> 8) * 2^-24. */
double oracle_transmission_u(uint64_t seed, uint64_t pulse, uint32_t subray,
                             uint32_t voxel) {
  uint32_t ctr[4] = {(uint32_t)pulse, (uint32_t)(pulse >> 32), subray, voxel};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  oracle_philox4x32_10(ctr, key, x);
  return (double)(x[0] >> 8) * (1.0 / 16777216.0);
}

/* Ranging error ("A single distance measurement is attributed with a
 * random ranging error, drawn from a normal distribution"; reading R29):
 * standard normal z for return number j (1-based) of pulse p by Box-Muller on
 * Philox-4x32-10 with key = (seed_lo, seed_hi ^ 1) (stream tag 1; tag 0 is
 * the transmission stream, R19), ctr = (p_lo, p_hi, j, 0):
 * u1 = ((x0 >> 8) + 1) 2^-24 in (0, 1], u2 = (x1 >> 8) 2^-24,
 * z = sqrt(-2 ln u1) cos(2 pi u2).  The return's range is R + sigma z. */
double oracle_range_noise(uint64_t seed, uint64_t pulse, uint32_t return_number) {
  uint32_t ctr[4] = {(uint32_t)pulse, (uint32_t)(pulse >> 32), return_number, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ 1u};
  uint32_t x[4];
  oracle_philox4x32_10(ctr, key, x);
  double u1 = (double)((x[0] >> 8) + 1u) * (1.0 / 16777216.0);
  double u2 = (double)(x[1] >> 8) * (1.0 / 16777216.0);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

/* ------------------------------------------------------------------------
 * Pulse generation (NEXT f2; P:155 platforms, P:177 deflectors; reading R30).
 * Pulse g of a survey is emitted at t = t0 + g / PRF.
 *   deflector (u = frac(f t), A = scan angle):
 *     polygon mirror:  theta = -A + 2 A u              (sawtooth, parallel lines)
 *     fibre optics:    theta = -A + 2 A (k + 1/2) / n, k = min(n-1, floor(u n))
 *     oscillating:     theta = A sin(2 pi f t)         (zig-zag, dense extrema)
 *     Palmer:          cone of half-angle A off nadir, azimuth phi = 2 pi u
 *   scanner frame: s = (0, -sin theta, -cos theta) (theta > 0 to starboard),
 *     Palmer s = (sin A cos phi, sin A sin phi, -cos A);
 *   head rotation about the platform z axis: h = Rz(omega t) s; mount: m = M h;
 *   platform: Static (one waypoint; yaw 0) or LinearPath (constant speed from
 *     waypoint to waypoint, "orientation ... always towards the next waypoint",
 *     P:155): leg k by time tau = t - t0, P = W_k + ((tau - T_k) v) u_k,
 *     yaw rotation (cos, sin) = (dx, dy) / hypot(dx, dy) of the leg (no
 *     trigonometry: an axis-aligned leg rotates exactly), after the last
 *     waypoint: stays there;
 *   world direction = Rz(yaw) m, origin = P + Rz(yaw) offset.
 * Outputs fp32 origin/direction (rounded from fp64) and fp64 time.
 * ---------------------------------------------------------------------- */
typedef struct {
  const double* waypoints;  // [n_waypoints][3]
  uint32_t n_waypoints;
  uint32_t deflector;       // 0 polygon, 1 fibre, 2 oscillating, 3 Palmer
  double speed_m_s;
  double mount[9];          // row-major scanner -> platform rotation
  double mount_offset[3];
  double head_rotation_rad_s;
  double pulse_freq_hz;
  double t0_s;
  double scan_freq_hz;
  double scan_angle_rad;
  uint32_t n_fibres;
  uint32_t pad_;
} oracle_survey;

static void rot_cs(double c, double s, const double v[3], double out[3]) {
  out[0] = c * v[0] - s * v[1];
  out[1] = s * v[0] + c * v[1];
  out[2] = v[2];
}

// yaw towards the leg's horizontal direction: (cos, sin) = (dx, dy) / hypot(dx, dy)
static void heading(const double d[3], double* c, double* s) {
  const double rho = std::sqrt(d[0] * d[0] + d[1] * d[1]);
  if (rho > 0.0) {
    *c = d[0] / rho;
    *s = d[1] / rho;
  } else {
    *c = 1.0;
    *s = 0.0;
  }
}

void oracle_generate_pulses(const oracle_survey* sv, uint64_t first, int64_t n, float* origin,
                            float* direction, double* time) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t g = first + (uint64_t)i;
    const double tau = (double)g / sv->pulse_freq_hz;
    const double t = sv->t0_s + tau;
    // deflector
    const double ft = sv->scan_freq_hz * t;
    const double u = ft - std::floor(ft);
    const double A = sv->scan_angle_rad;
    double s[3];
    if (sv->deflector == 3) {
      const double phi = 2.0 * kPi * u;
      s[0] = std::sin(A) * std::cos(phi);
      s[1] = std::sin(A) * std::sin(phi);
      s[2] = -std::cos(A);
    } else {
      double theta;
      if (sv->deflector == 0) {
        theta = -A + 2.0 * A * u;
      } else if (sv->deflector == 1) {
        const double nf = (double)sv->n_fibres;
        const double k = std::min(nf - 1.0, std::floor(u * nf));
        theta = -A + 2.0 * A * (k + 0.5) / nf;
      } else {
        theta = A * std::sin(2.0 * kPi * sv->scan_freq_hz * t);
      }
      s[0] = 0.0;
      s[1] = -std::sin(theta);
      s[2] = -std::cos(theta);
    }
    double h[3], m[3];
    const double ha = sv->head_rotation_rad_s * t;
    rot_cs(std::cos(ha), std::sin(ha), s, h);
    for (int r = 0; r < 3; ++r)
      m[r] = sv->mount[3 * r] * h[0] + sv->mount[3 * r + 1] * h[1] + sv->mount[3 * r + 2] * h[2];
    // platform
    double P[3] = {sv->waypoints[0], sv->waypoints[1], sv->waypoints[2]};
    double yc = 1.0, ys = 0.0;  // cos / sin of the yaw
    if (sv->n_waypoints > 1) {
      double T = 0.0;  // start time of the current leg
      bool placed = false;
      int last_leg = -1;
      for (uint32_t k = 0; k + 1 < sv->n_waypoints; ++k) {
        const double* a = sv->waypoints + 3 * k;
        const double* b = a + 3;
        const double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        if (!(len > 0.0)) continue;  // zero-length leg: no time, no heading
        last_leg = (int)k;
        const double dur = len / sv->speed_m_s;
        if (tau < T + dur || k + 2 == sv->n_waypoints) {
          const double w = std::min(tau - T, dur) * sv->speed_m_s;  // distance along the leg
          const double along = std::max(0.0, w);
          for (int c = 0; c < 3; ++c) P[c] = a[c] + along * (d[c] / len);
          heading(d, &yc, &ys);
          placed = true;
          break;
        }
        T += dur;
      }
      if (!placed && last_leg >= 0) {  // only zero-length legs after the last real one
        const double* a = sv->waypoints + 3 * last_leg;
        const double* b = a + 3;
        const double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        for (int c = 0; c < 3; ++c) P[c] = b[c];
        heading(d, &yc, &ys);
      }
    }
    double dw[3], ow[3];
    rot_cs(yc, ys, m, dw);
    rot_cs(yc, ys, sv->mount_offset, ow);
    for (int c = 0; c < 3; ++c) {
      origin[3 * i + c] = (float)(P[c] + ow[c]);
      direction[3 * i + c] = (float)dw[c];
    }
    time[i] = t;
  }
}

/* Opaque voxels (reading R31).  Cube of voxel id: side a and
 * minimum corner.  Opaque mode: the voxel itself.  Scaled mode (Eq. 5):
 * a = a0 (min(1, PAD / PAD_max))^alpha centred in the voxel, optionally
 * shifted by (u_k - 1/2)(a0 - a) per axis with u_k = (x_k >> 8) 2^-24 from
 * Philox-4x32-10, key (seed_lo, seed_hi ^ 2) (stream tag 2), counter
 * (voxel id, 0, 0, 0) -- "random but reproducible". */
void oracle_voxel_cube(const uint32_t n[3], const double org[3], double a0, uint32_t id,
                       double PAD, uint32_t mode, double pad_max, double alpha,
                       uint32_t shift, uint64_t seed, double lo[3], double* side) {
  const uint32_t ix = id % n[0], iy = (id / n[0]) % n[1], iz = id / (n[0] * n[1]);
  const uint32_t idx[3] = {ix, iy, iz};
  if (mode != 2) {
    for (int a = 0; a < 3; ++a) lo[a] = org[a] + (double)idx[a] * a0;
    *side = a0;
    return;
  }
  const double a = a0 * std::pow(std::min(1.0, PAD / pad_max), alpha);
  double sh[3] = {0.0, 0.0, 0.0};
  if (shift) {
    uint32_t ctr[4] = {id, 0u, 0u, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32) ^ 2u};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    for (int k = 0; k < 3; ++k)
      sh[k] = ((double)(x[k] >> 8) * (1.0 / 16777216.0) - 0.5) * (a0 - a);
  }
  for (int k = 0; k < 3; ++k) {
    const double centre = org[k] + ((double)idx[k] + 0.5) * a0;
    lo[k] = centre + sh[k] - 0.5 * a;
  }
  *side = a;
}

/* Ray vs axis-aligned cube [lo, lo + side]^3 (slab test, fp64): entry t and
 * the entry axis (largest near-plane time, lowest axis on ties); returns
 * false when the ray misses or the cube does not lie ahead (entry <= 0). */
static bool ray_cube(const double o[3], const double d[3], const double lo[3], double side,
                     double* t_enter, int* axis) {
  double tn = -kInf, tf = kInf;
  int ax = -1;
  for (int a = 0; a < 3; ++a) {
    const double l = lo[a], h = lo[a] + side;
    if (d[a] == 0.0) {
      if (o[a] < l || o[a] > h) return false;
      continue;
    }
    double t0 = (l - o[a]) / d[a], t1 = (h - o[a]) / d[a];
    if (t0 > t1) std::swap(t0, t1);
    if (t0 > tn) {
      tn = t0;
      ax = a;
    }
    tf = std::min(tf, t1);
  }
  if (!(tn <= tf) || !(tn > 0.0) || ax < 0) return false;
  *t_enter = tn;
  *axis = ax;
  return true;
}

/* G(|d_z|) for sigma = PAD * G (R15): LUT over |d_z| in [0,1] at uniform
 * knots, linear interpolation; no LUT -> spherical LAD, G = 0.5. */
double oracle_g_function(const float* lut, uint32_t n_lut, double abs_dz) {
  if (!lut || n_lut == 0) return 0.5;
  double x = abs_dz * (double)(n_lut - 1);
  int64_t k = (int64_t)std::floor(x);
  if (k < 0) k = 0;
  if (k > (int64_t)n_lut - 2) k = (int64_t)n_lut - 2;
  double f = x - (double)k;
  return (double)lut[k] * (1.0 - f) + (double)lut[k + 1] * f;
}

/* ------------------------------------------------------------------------
 * Voxel segments along a ray (P:366 re-entrant rays with eps -> 0, R20).
 * Independent of any incremental DDA: clip the ray to the grid box and to
 * (0, t_max]; enumerate EVERY x-, y- and z-plane crossing parameter inside
 * that interval directly, sort them, and assign each sub-interval to the
 * voxel containing its midpoint; merge runs of the same voxel and drop
 * zero-length pieces.  Writes up to max_seg (t_a, t_b, voxel id) triples in
 * ray order and returns the count (or -(count) if truncated).
 * ---------------------------------------------------------------------- */
int64_t oracle_voxel_segments(const double o_in[3], const double d_in[3],
                              const uint32_t n[3], const double origin[3],
                              double vs, double t_max, double* ta, double* tb,
                              uint32_t* vid, int64_t max_seg) {
  double o[3] = {o_in[0], o_in[1], o_in[2]};
  double d[3] = {d_in[0], d_in[1], d_in[2]};
  // Slab clip against the grid box.
  double t_in = 0.0, t_out = t_max;
  for (int a = 0; a < 3; ++a) {
    double lo = origin[a];
    double hi = origin[a] + (double)n[a] * vs;
    if (d[a] == 0.0) {
      if (o[a] < lo || o[a] > hi) return 0;
      continue;
    }
    double t0 = (lo - o[a]) / d[a];
    double t1 = (hi - o[a]) / d[a];
    if (t0 > t1) std::swap(t0, t1);
    t_in = std::max(t_in, t0);
    t_out = std::min(t_out, t1);
  }
  if (!(t_in < t_out)) return 0;
  // Every plane crossing strictly inside (t_in, t_out).
  std::vector<double> ts;
  ts.push_back(t_in);
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0) continue;
    for (uint32_t k = 0; k <= n[a]; ++k) {
      double plane = origin[a] + (double)k * vs;
      double t = (plane - o[a]) / d[a];
      if (t > t_in && t < t_out) ts.push_back(t);
    }
  }
  ts.push_back(t_out);
  std::sort(ts.begin(), ts.end());
  int64_t cnt = 0;
  bool trunc = false;
  for (size_t i = 0; i + 1 < ts.size(); ++i) {
    double a = ts[i], b = ts[i + 1];
    if (!(b > a)) continue;  // zero-length piece
    double m = 0.5 * (a + b);
    int64_t idx[3];
    for (int ax = 0; ax < 3; ++ax) {
      double c = (o[ax] + m * d[ax] - origin[ax]) / vs;
      int64_t k = (int64_t)std::floor(c);
      if (k < 0) k = 0;
      if (k >= (int64_t)n[ax]) k = (int64_t)n[ax] - 1;
      idx[ax] = k;
    }
    uint32_t id = (uint32_t)(idx[0] + (int64_t)n[0] * (idx[1] + (int64_t)n[1] * idx[2]));
    if (cnt > 0 && vid[cnt - 1] == id && tb[cnt - 1] == a) {
      tb[cnt - 1] = b;  // same voxel continues
      continue;
    }
    if (cnt >= max_seg) {
      trunc = true;
      break;
    }
    ta[cnt] = a;
    tb[cnt] = b;
    vid[cnt] = id;
    ++cnt;
  }
  return trunc ? -cnt : cnt;
}

/* ------------------------------------------------------------------------
 * Echo width ("Optionally, a Gaussian may be fitted to the resulting
 * waveform, to get a measure of echo width (i.e. standard deviation of the
 * Gaussian)"; "non-linear least squares").  Reading R28:
 * window = the echo: the bins around k over which W decreases strictly away
 * from the peak, at most w = ceil(3 pulse_length / Delta) on each side;
 * x_i = (i - k) Delta (ns), y_i = W[i];  g(x) = A exp(-(x - m)^2 / (2 s^2));
 * Levenberg-Marquardt from A = W[k], m = 0, s = pulse_length / (2 sqrt(2 ln 2)),
 * lambda = 1e-3, step (J^T J + lambda diag(J^T J)) d = J^T r, accept iff the
 * sum of squares decreases (lambda /= 10) else lambda *= 10; stop when an
 * accepted step has max_i |d_i| / (|p_i| + 1e-12) < 1e-10, or after 100
 * iterations (then: no width, NaN), or lambda > 1e16 (converged in place).
 * A Gaussian is identifiable from the window only if its centre and width
 * lie inside it: a converged fit with A <= 0, |m| > w Delta or |s| > w Delta
 * (the least-squares optimum running off to a flat, infinitely wide
 * Gaussian on non-peaked data) is reported as no width.
 * Returns |s|, or NaN.
 * ---------------------------------------------------------------------- */
static double sse_gauss(const double* x, const double* y, int n, double A, double m, double s) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    double z = (x[i] - m) / s;
    double r = y[i] - A * std::exp(-0.5 * z * z);
    acc += r * r;
  }
  return acc;
}

double oracle_fit_echo_width(const double* W, int64_t n_bins, int64_t k, double delta_ns,
                             double pulse_length_ns, double* A_out, double* m_out) {
  const int64_t w = (int64_t)std::ceil(3.0 * pulse_length_ns / delta_ns);
  int64_t lo = k, hi = k;  // the echo: W strictly decreasing away from the peak, within k +- w
  while (lo - 1 >= std::max<int64_t>(0, k - w) && W[lo - 1] < W[lo]) --lo;
  while (hi + 1 <= std::min<int64_t>(n_bins - 1, k + w) && W[hi + 1] < W[hi]) ++hi;
  const int n = (int)(hi - lo + 1);
  std::vector<double> x(n), y(n);
  for (int i = 0; i < n; ++i) {
    x[i] = (double)(lo + i - k) * delta_ns;
    y[i] = W[lo + i];
  }
  double A = W[k], m = 0.0, s = pulse_length_ns / (2.0 * std::sqrt(2.0 * std::log(2.0)));
  double lambda = 1e-3;
  double cur = sse_gauss(x.data(), y.data(), n, A, m, s);
  bool converged = false;
  for (int it = 0; it < 100; ++it) {
    // normal equations
    double H[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, g[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) {
      double z = (x[i] - m) / s;
      double e = std::exp(-0.5 * z * z);
      double J[3] = {e, A * e * z / s, A * e * z * z / s};  // d/dA, d/dm, d/ds
      double r = y[i] - A * e;
      for (int a = 0; a < 3; ++a) {
        g[a] += J[a] * r;
        for (int b = 0; b < 3; ++b) H[a][b] += J[a] * J[b];
      }
    }
    double M[3][3];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[a][b] = H[a][b] + (a == b ? lambda * H[a][a] : 0.0);
    // solve M d = g (Cramer's rule on the 3x3 system)
    double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                 M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                 M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    if (!(std::fabs(det) > 0.0) || !std::isfinite(det)) break;
    double d[3];
    for (int c = 0; c < 3; ++c) {
      double T[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) T[a][b] = (b == c) ? g[a] : M[a][b];
      d[c] = (T[0][0] * (T[1][1] * T[2][2] - T[1][2] * T[2][1]) -
              T[0][1] * (T[1][0] * T[2][2] - T[1][2] * T[2][0]) +
              T[0][2] * (T[1][0] * T[2][1] - T[1][1] * T[2][0])) / det;
    }
    double nA = A + d[0], nm = m + d[1], ns = s + d[2];
    double next = sse_gauss(x.data(), y.data(), n, nA, nm, ns);
    if (std::isfinite(next) && next < cur) {
      double rel = std::max({std::fabs(d[0]) / (std::fabs(A) + 1e-12),
                             std::fabs(d[1]) / (std::fabs(m) + 1e-12),
                             std::fabs(d[2]) / (std::fabs(s) + 1e-12)});
      A = nA;
      m = nm;
      s = ns;
      cur = next;
      lambda /= 10.0;
      if (rel < 1e-10) {
        converged = true;
        break;
      }
    } else {
      lambda *= 10.0;
      if (lambda > 1e16) {
        converged = true;  // no further decrease possible: at the minimum
        break;
      }
    }
  }
  if (A_out) *A_out = A;
  if (m_out) *m_out = m;
  if (!converged || !std::isfinite(s)) return kNaN;
  const double span = (double)w * delta_ns;
  if (!(A > 0.0) || std::fabs(m) > span || std::fabs(s) > span) return kNaN;
  return std::fabs(s);
}

/* ------------------------------------------------------------------------
 * Simulation parameters (mirrors DESIGN.md s.2; plain doubles).
 * ---------------------------------------------------------------------- */
typedef struct {
  double divergence_rad;        // beta (R3)
  double pulse_length_ns;       // tau = pulse_length / 1.75
  double bin_width_ns;          // Delta
  double max_fullwave_range_ns; // window
  double detection_threshold;   // thr (R11)
  double peak_power_w;          // I0 (Eq. 1)
  double efficiency;            // lambda of Eq. 7
  double receiver_diameter_m;   // alpha of Eq. 7 (R14)
  double wavelength_nm;         // lambda of Eq. 2
  double beam_waist_m;          // w0 of Eq. 2 (0 -> far field, R5)
  double focus_range_m;         // R0 of Eq. 2
  uint64_t seed;                // Philox key (R19)
  uint32_t subray_count;        // (R1)
  uint32_t max_returns;         // (R11)
  uint32_t fit_echo_width;      // optional Gaussian echo-width fit (R28)
  uint32_t pad_;
  double range_noise_sd_m;      // ranging error sigma (R29), 0 -> none
} oracle_params;

typedef struct {
  const float* tris;     // [n_tris][9]
  const float* refl;     // [n_tris] or NULL -> 0.5
  uint32_t n_tris;
  const float* pad;      // [nz][ny][nx] or NULL
  uint32_t n[3];         // nx, ny, nz
  double origin[3];
  double voxel_size;
  const float* g_lut;
  uint32_t n_lut;
  // voxel interpretation (NEXT f3, reading R31):
  // 0 transmissive, 1 opaque cubes, 2 PAD-scaled opaque cubes (Eq. 5)
  uint32_t voxel_mode;
  double voxel_reflectance;  // rho of opaque / scaled cubes
  double pad_max;            // PAD_max of Eq. 5
  double scale_alpha;        // alpha of Eq. 5
  uint32_t scale_shift;      // 1: reproducible random shift of each scaled cube
  uint32_t pad2_;
} oracle_scene;

typedef struct {
  // per pulse
  int32_t* n_returns;    // [n]
  int64_t* k0;           // [n]
  double* waveform;      // [n][n_bins] or NULL
  double* ret_range;     // [n][max_returns]
  double* ret_time;
  double* ret_intensity;
  uint32_t* ret_prim;
  int32_t* ret_number;
  double* ret_width;     // [n][max_returns] fitted echo width sigma (ns); NaN = no fit
  double* peak_margin;   // [n] min relative margin of every peak decision
  double* attr_margin;   // [n] min relative gap between the top two contributions
  // per subray, [n][N]
  double* sub_range;     // NaN on miss
  double* sub_amp;
  uint32_t* sub_prim;    // UINT32_MAX on miss
  int64_t* sub_k;        // -1 on miss
  int32_t* sub_ncand;
  double* sub_gap;
  double* sub_kmargin;   // |2R/(c Delta) - round(.)|
  double* sub_umargin;   // min |u - exp(-sigma L)| over this subray's decisions
  uint32_t* sub_cand;    // [n][N][kMaxCand] candidate ids (C_tri by (t, id)) or NULL
  uint32_t* ret_cand;    // [n][max_returns][kMaxAttr] attribution candidates or NULL
} oracle_outputs;

uint32_t oracle_waveform_bins(double window_ns, double bin_ns) {
  if (!(bin_ns > 0.0) || !(window_ns >= bin_ns)) return 0;
  return (uint32_t)std::ceil(window_ns / bin_ns);  // R9
}

/* One subray of pulse i: steps O1..O5 of DESIGN.md s.4 (the paper's order).
 * Writes the per-subray outputs (range, amplitude, prim, bin, margins). */
static void simulate_subray(const oracle_scene* sc, const oracle_params* pr,
                            const float* origin, const float* direction, uint64_t pulse_id,
                            int64_t i, uint32_t s, const double* theta, const double* phi,
                            HitList& hits, const oracle_outputs* out) {
  const uint32_t N = pr->subray_count;
  const double beta = pr->divergence_rad;
  const double delta = pr->bin_width_ns;
  const double K = pr->efficiency * pr->receiver_diameter_m *
                   pr->receiver_diameter_m / (4.0 * kPi * beta * beta);  // Eq. 7

  double o[3] = {origin[0], origin[1], origin[2]};
  double d[3] = {direction[0], direction[1], direction[2]};
  double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);

  double Rs_out = kNaN, A_out = 0.0, gap_out = kInf, kmarg_out = kInf, umarg_out = kInf;
  uint32_t prim_out = 0xFFFFFFFFu;
  uint32_t cand_out[kMaxCand];
  for (int32_t c = 0; c < kMaxCand; ++c) cand_out[c] = 0xFFFFFFFFu;
  int64_t k_out = -1;
  int32_t ncand_out = 0;
  if (dn > 0.0) {
    {
      // O1: subray direction.
      double ds[3];
      oracle_subray_direction(d, theta[s], phi[s], ds);
      // O2: nearest triangle, brute force: `hits` holds the ray's hit on EVERY
      // triangle it meets (phase 1 of oracle_simulate)
      double t_tri = kInf, cos_inc = 0.0, gap = kInf;
      int32_t nc = 0;
      uint32_t cand[kMaxCand];
      int64_t tid = nearest_from_hits(hits, &t_tri, &nc, &gap, cand, kMaxCand);
      if (tid >= 0) oracle_ray_triangle(o, ds, sc->tris + 9ull * tid, &cos_inc);
      // O3: transmissive voxels before the triangle.
      bool vox_hit = false;
      double t_vox = 0.0, sigma_vox = 0.0;
      uint32_t vox_id = 0;
      double um = kInf;
      if (sc->pad && sc->voxel_mode != 0) {
        // O3': opaque / scaled cubes (Eq. 5; R31): the first cube
        // the subray enters, before the triangle
        double tmax = tid >= 0 ? t_tri : kInf;
        int64_t cap = (int64_t)sc->n[0] + sc->n[1] + sc->n[2] + 2;
        std::vector<double> ta(cap), tb(cap);
        std::vector<uint32_t> vid(cap);
        int64_t ns = oracle_voxel_segments(o, ds, sc->n, sc->origin, sc->voxel_size,
                                           tmax, ta.data(), tb.data(), vid.data(), cap);
        if (ns < 0) ns = -ns;
        for (int64_t k = 0; k < ns; ++k) {
          double PAD = sc->pad[vid[k]];
          if (!(PAD > 0.0)) continue;
          double lo[3], side, te;
          int ax;
          oracle_voxel_cube(sc->n, sc->origin, sc->voxel_size, vid[k], PAD, sc->voxel_mode,
                            sc->pad_max, sc->scale_alpha, sc->scale_shift, pr->seed, lo, &side);
          if (!ray_cube(o, ds, lo, side, &te, &ax) || !(te < tmax)) continue;
          vox_hit = true;
          t_vox = te;
          sigma_vox = sc->voxel_reflectance * std::fabs(ds[ax]);  // R31: Lambertian face
          vox_id = vid[k];
          break;
        }
      } else if (sc->pad) {
        double tmax = tid >= 0 ? t_tri : kInf;
        int64_t cap = (int64_t)sc->n[0] + sc->n[1] + sc->n[2] + 2;
        std::vector<double> ta(cap), tb(cap);
        std::vector<uint32_t> vid(cap);
        int64_t ns = oracle_voxel_segments(o, ds, sc->n, sc->origin, sc->voxel_size,
                                           tmax, ta.data(), tb.data(), vid.data(), cap);
        if (ns < 0) ns = -ns;
        double G = oracle_g_function(sc->g_lut, sc->n_lut, std::fabs(ds[2]));
        for (int64_t k = 0; k < ns; ++k) {
          double PAD = sc->pad[vid[k]];
          if (!(PAD > 0.0)) continue;  // sigma = 0 lets the ray continue
          double sigma = PAD * G;        // Eq. 4 via the G-LUT (R15)
          double L = tb[k] - ta[k];
          double u = oracle_transmission_u(pr->seed, pulse_id, s, vid[k]);
          double margin = kInf;
          const int pass = oracle_transmits(u, sigma, L, &margin);
          um = std::min(um, margin);
          if (pass) continue;            // s = -ln(u)/sigma > L: transmit (R17)
          vox_hit = true;                 // Eq. 6: echo at distance s into the voxel
          t_vox = ta[k] + (-std::log(u)) / sigma;
          sigma_vox = sigma;
          vox_id = vid[k];
          break;
        }
      }
      // O4/O5: event, range, radiometry.
      double Rs = kNaN, sig_eff = 0.0;
      uint32_t pid = 0xFFFFFFFFu;
      if (vox_hit) {
        Rs = t_vox;
        sig_eff = sigma_vox;                            // R16
        pid = sc->n_tris + vox_id;
      } else if (tid >= 0) {
        Rs = t_tri;
        double rho = sc->refl ? (double)sc->refl[tid] : 0.5;
        sig_eff = rho * cos_inc;                        // R14 (Lambertian)
        pid = (uint32_t)tid;
      }
      if (pid != 0xFFFFFFFFu) {
        double Is = oracle_subray_intensity(pr->peak_power_w, theta[s], beta, Rs,
                                            pr->beam_waist_m, pr->wavelength_nm,
                                            pr->focus_range_m);      // Eq. 1, 2
        A_out = K * sig_eff * Is / (Rs * Rs * Rs * Rs);                // Eq. 7
        Rs_out = Rs;
        prim_out = pid;
        k_out = oracle_bin_of(Rs, delta, &kmarg_out);  // two-way time in bins (R8, R9)
        ncand_out = vox_hit ? 1 : nc;
        gap_out = vox_hit ? kInf : gap;
        if (vox_hit) {
          cand_out[0] = pid;
        } else {
          for (int32_t c = 0; c < kMaxCand; ++c) cand_out[c] = cand[c];
        }
      }
      umarg_out = um;
    }
  }
  int64_t x = i * (int64_t)N + s;
  out->sub_range[x] = Rs_out;
  out->sub_amp[x] = A_out;
  out->sub_prim[x] = prim_out;
  out->sub_k[x] = k_out;
  out->sub_ncand[x] = ncand_out;
  out->sub_gap[x] = gap_out;
  out->sub_kmargin[x] = kmarg_out;
  out->sub_umargin[x] = umarg_out;
  if (out->sub_cand)
    for (int32_t c = 0; c < kMaxCand; ++c) out->sub_cand[x * kMaxCand + c] = cand_out[c];
}

/* Steps O6..O8 for ONE pulse from its subrays' amplitudes A[s], bins ks[s]
 * (-1 = no event) and prims prim[s], s < N: the full waveform (Eq. 3, P:215,
 * P:408), the local-maximum peaks (R11-R13) and the returns.
 * Outputs (per pulse): *n_returns, *k0, W[n_bins] (may be NULL), the return
 * arrays [max_returns] (range, time, intensity, prim, number, width) and
 * ret_cand [max_returns][kMaxAttr] (may be NULL), *peak_margin, *attr_margin.
 *
 * Decision margins (C-4), what the CUDA path's arithmetic could flip:
 *  - peak_margin: min over bins k of the margin of the decision "k is a
 *    peak".  The decision is a > l AND a > r AND a >= thr M (a = W[k]); the
 *    signed relative margins are (a - l)/max(a, l), (a - r)/max(a, r),
 *    (a - thr M)/M.  A true decision flips if ANY conjunct flips: its margin
 *    is the smallest |margin| of the three; a false one only if EVERY false
 *    conjunct flips: its margin is the largest |margin| among them (a
 *    comparison of two zero bins is false by any margin).
 *  - attribution (R13): the prim of the largest contribution A_s p[k - o_s]
 *    (ties -> lowest s); ret_cand lists the distinct prims whose contribution
 *    is >= c_max (1 - kDecisionEps) (by contribution, then s); attr_margin =
 *    min over returns of (c_max - c_other) / c_max, c_other = the largest
 *    contribution of a DIFFERENT prim (+inf if none). */
int oracle_waveform_peaks(const oracle_params* pr, const double* A, const int64_t* ks,
                          const uint32_t* prim, double time_s, uint64_t pulse_id,
                          int32_t* n_returns_out, int64_t* k0_out, double* W_out,
                          double* ret_range, double* ret_time, double* ret_intensity,
                          uint32_t* ret_prim, int32_t* ret_number, double* ret_width,
                          uint32_t* ret_cand, double* peak_margin, double* attr_margin) {
  const uint32_t N = pr->subray_count;
  const double delta = pr->bin_width_ns;
  const double tau = pr->pulse_length_ns / 1.75;
  const uint32_t n_bins = oracle_waveform_bins(pr->max_fullwave_range_ns, delta);
  if (n_bins == 0 || pr->max_returns < 1) return -1;
  const int64_t Lp = (int64_t)std::ceil(20.0 * tau / delta);           // R9
  const uint32_t maxr = pr->max_returns;

  // O6: full waveform (Eq. 3).
  int64_t k0 = -1;
  for (uint32_t s = 0; s < N; ++s)
    if (ks[s] >= 0 && (k0 < 0 || ks[s] < k0)) k0 = ks[s];
  std::vector<double> W(n_bins, 0.0);
  if (k0 >= 0) {
    for (uint32_t s = 0; s < N; ++s) {
      if (ks[s] < 0) continue;
      int64_t off = ks[s] - k0;
      if (off >= (int64_t)n_bins) continue;  // beyond maxFullwaveRange: discarded
      for (int64_t j = 0; j < Lp; ++j) {
        int64_t k = off + j;
        if (k >= (int64_t)n_bins) break;
        double t = ((double)j + 0.5) * delta;  // bin-centre sampling (R9)
        W[k] += oracle_eq3_pulse(A[s], t, tau);
      }
    }
  }
  // j* = argmax of the binned outgoing pulse (R12).
  int64_t jstar = 0;
  {
    double best = -1.0;
    for (int64_t j = 0; j < Lp; ++j) {
      double p = oracle_eq3_pulse(1.0, ((double)j + 0.5) * delta, tau);
      if (p > best) {
        best = p;
        jstar = j;
      }
    }
  }

  // O7: local-maximum peaks (R11-R13).
  double M = 0.0;
  for (uint32_t k = 0; k < n_bins; ++k) M = std::max(M, W[k]);
  double thr = pr->detection_threshold * M;
  int32_t nret = 0;
  double pmarg = kInf, amarg = kInf;
  for (int64_t k = 1; k + 1 < (int64_t)n_bins; ++k) {
    double a = W[k], l = W[k - 1], r = W[k + 1];
    bool peak = a > l && a > r && a >= thr;
    // margin of this decision (see above)
    {
      const bool c[3] = {a > l, a > r, a >= thr};
      const double m[3] = {
          std::max(a, l) > 0.0 ? std::fabs(a - l) / std::max(a, l) : kInf,
          std::max(a, r) > 0.0 ? std::fabs(a - r) / std::max(a, r) : kInf,
          M > 0.0 ? std::fabs(a - thr) / M : kInf};
      double mk;
      if (peak) {
        mk = std::min(m[0], std::min(m[1], m[2]));
      } else {
        mk = 0.0;
        for (int q = 0; q < 3; ++q)
          if (!c[q]) mk = std::max(mk, m[q]);
      }
      pmarg = std::min(pmarg, mk);
    }
    if (!peak) continue;
    if ((uint32_t)nret >= maxr) continue;  // keep the earliest max_returns
    // Attribution (R13): subray with the largest contribution to bin k.
    std::vector<std::pair<double, uint32_t>> contrib;  // (c, s)
    double c1 = -1.0;
    uint32_t who = 0xFFFFFFFFu;
    for (uint32_t s = 0; s < N; ++s) {
      if (ks[s] < 0) continue;
      int64_t off = ks[s] - k0;
      if (off >= (int64_t)n_bins) continue;
      int64_t j = k - off;
      if (j < 0 || j >= Lp) continue;
      double c = oracle_eq3_pulse(A[s], ((double)j + 0.5) * delta, tau);
      contrib.push_back({c, s});
      if (c > c1) {
        c1 = c;
        who = prim[s];
      }
    }
    double c_other = -1.0;
    for (const auto& cs : contrib)
      if (prim[cs.second] != who) c_other = std::max(c_other, cs.first);
    if (c1 > 0.0 && c_other >= 0.0) amarg = std::min(amarg, (c1 - c_other) / c1);
    int64_t slot = nret;
    if (ret_cand) {
      // distinct prims within kDecisionEps of the top, by (contribution desc, s)
      std::sort(contrib.begin(), contrib.end(), [](const std::pair<double, uint32_t>& x,
                                                   const std::pair<double, uint32_t>& y) {
        return x.first > y.first || (x.first == y.first && x.second < y.second);
      });
      int32_t nc = 0;
      for (int32_t q = 0; q < kMaxAttr; ++q) ret_cand[slot * kMaxAttr + q] = 0xFFFFFFFFu;
      for (const auto& cs : contrib) {
        if (!(cs.first >= c1 * (1.0 - kDecisionEps))) break;
        const uint32_t pid = prim[cs.second];
        bool seen = false;
        for (int32_t q = 0; q < nc; ++q) seen |= ret_cand[slot * kMaxAttr + q] == pid;
        if (!seen && nc < kMaxAttr) ret_cand[slot * kMaxAttr + nc++] = pid;
      }
    }
    ret_range[slot] = 0.5 * kC * ((double)(k0 + k - jstar) + 0.5) * delta * 1e-9;  // R12
    if (pr->range_noise_sd_m > 0.0)  // P:288, R29
      ret_range[slot] += pr->range_noise_sd_m *
                         oracle_range_noise(pr->seed, pulse_id, (uint32_t)(nret + 1));
    ret_time[slot] = time_s;
    ret_intensity[slot] = a;
    ret_prim[slot] = who;
    ret_number[slot] = nret + 1;
    ret_width[slot] =
        pr->fit_echo_width
            ? oracle_fit_echo_width(W.data(), n_bins, k, delta, pr->pulse_length_ns, nullptr, nullptr)
            : kNaN;
    ++nret;
  }

  // O8: emit.
  *n_returns_out = nret;
  *k0_out = k0;
  if (W_out)
    for (uint32_t k = 0; k < n_bins; ++k) W_out[k] = W[k];
  *peak_margin = pmarg;
  *attr_margin = amarg;
  return 0;
}

/* Pulse i after all its subrays: steps O6..O8 on the pulse's row of the
 * per-subray outputs. */
static void finish_pulse(const oracle_params* pr, double time_s, uint64_t pulse_id, int64_t i,
                         const oracle_outputs* out) {
  const uint32_t N = pr->subray_count;
  const uint32_t n_bins = oracle_waveform_bins(pr->max_fullwave_range_ns, pr->bin_width_ns);
  const int64_t R = pr->max_returns;
  oracle_waveform_peaks(pr, out->sub_amp + i * (int64_t)N, out->sub_k + i * (int64_t)N,
                        out->sub_prim + i * (int64_t)N, time_s, pulse_id, out->n_returns + i,
                        out->k0 + i, out->waveform ? out->waveform + i * (int64_t)n_bins : nullptr,
                        out->ret_range + i * R, out->ret_time + i * R, out->ret_intensity + i * R,
                        out->ret_prim + i * R, out->ret_number + i * R, out->ret_width + i * R,
                        out->ret_cand ? out->ret_cand + i * R * kMaxAttr : nullptr,
                        out->peak_margin + i, out->attr_margin + i);
}

/* Simulate the listed pulses (a seeded subset or all of them).  pulse_ids
 * are the GLOBAL pulse indices (Philox counter).  Parallel over pulses
 * with a plain thread pool (P:289's pulse-level multithreading); nothing is
 * shared or reduced across threads, so the result is thread-count
 * independent.  Returns 0, or -1 on invalid parameters. */
int oracle_simulate(const oracle_scene* sc, const oracle_params* pr,
                    const float* origins, const float* directions,
                    const double* times, const uint64_t* pulse_ids,
                    int64_t n_pulses, int n_threads, const oracle_outputs* out) {
  const uint32_t N = pr->subray_count;
  std::vector<int> ring(N), slot(N), ring_n(N);
  std::vector<double> theta(N), phi(N);
  if (oracle_subray_pattern(N, pr->divergence_rad, ring.data(), slot.data(),
                            ring_n.data(), theta.data(), phi.data()) != 0)
    return -1;
  if (oracle_waveform_bins(pr->max_fullwave_range_ns, pr->bin_width_ns) == 0) return -1;
  if (pr->max_returns < 1) return -1;
  for (int64_t i = 0; i < n_pulses; ++i) {
    out->n_returns[i] = 0;
    for (uint32_t r = 0; r < pr->max_returns; ++r) {
      int64_t x = i * pr->max_returns + r;
      out->ret_range[x] = 0.0;
      out->ret_time[x] = 0.0;
      out->ret_intensity[x] = 0.0;
      out->ret_prim[x] = 0;
      out->ret_number[x] = 0;
      out->ret_width[x] = kNaN;
      if (out->ret_cand)
        for (int32_t q = 0; q < kMaxAttr; ++q) out->ret_cand[x * kMaxAttr + q] = 0xFFFFFFFFu;
    }
  }
  if (n_threads < 1) n_threads = 1;
  // Every (pulse, subray) pair is independent, then every pulse's
  // waveform and peaks.  Plain thread pool with an atomic work counter;
  // nothing is reduced across threads in a thread-dependent order
  // (thread-count independent).
  auto run_pool = [&](int64_t n_items, auto&& body) {
    std::atomic<int64_t> next(0);
    auto worker = [&]() {
      for (;;) {
        int64_t k = next.fetch_add(1);
        if (k >= n_items) break;
        body(k);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < n_threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
  };
  // Phase 1: the hits of every subray on every triangle.  Work items are
  // (pulse, block of triangles): each triangle of the block is tested
  // against every subray of the pulse (one read of the scene per pulse).  A
  // subray's hits from all blocks are concatenated; the nearest is the
  // minimum of (t, id) over them, whatever their order.
  const uint32_t kBlock = 1u << 18;
  const int64_t nblk = sc->n_tris ? ((int64_t)sc->n_tris + kBlock - 1) / kBlock : 0;
  // A triangle none of a pulse's subrays can reach (its bounding sphere
  // outside the cone of half-angle max theta_i around the pulse axis) is
  // skipped for that pulse (cone_may_hit; widened by 1e-6 relative + 1e-12).
  double th_max = 0.0;
  for (uint32_t s = 0; s < N; ++s) th_max = std::max(th_max, theta[s]);
  th_max = th_max * (1.0 + 1e-6) + 1e-12;
  const double cos_c = std::cos(th_max), sin_c = std::sin(th_max);
  std::vector<double> dirs((size_t)n_pulses * N * 3, 0.0), axis((size_t)n_pulses * 3, 0.0);
  std::vector<char> dir_ok(n_pulses, 0);
  for (int64_t i = 0; i < n_pulses; ++i) {
    const float* dv = directions + 3 * i;
    const double d[3] = {dv[0], dv[1], dv[2]};
    const double dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    dir_ok[i] = dn > 0.0;
    if (!dir_ok[i]) continue;
    for (int c = 0; c < 3; ++c) axis[3 * i + c] = d[c] / dn;
    for (uint32_t s = 0; s < N; ++s)
      oracle_subray_direction(d, theta[s], phi[s], &dirs[((size_t)i * N + s) * 3]);  // O1
  }
  std::vector<HitList> blk_hits((size_t)n_pulses * nblk * N);
  run_pool(n_pulses * nblk, [&](int64_t item) {
    const int64_t i = item / nblk, b = item % nblk;
    if (!dir_ok[i]) return;
    const double o[3] = {origins[3 * i], origins[3 * i + 1], origins[3 * i + 2]};
    const uint32_t t0 = (uint32_t)(b * kBlock);
    const uint32_t t1 = (uint32_t)std::min<int64_t>((int64_t)sc->n_tris, (b + 1) * (int64_t)kBlock);
    HitList* h = &blk_hits[((size_t)i * nblk + b) * N];
    const V3 ov = {o[0], o[1], o[2]};
    const V3 ax = {axis[3 * i], axis[3 * i + 1], axis[3 * i + 2]};
    for (uint32_t t = t0; t < t1; ++t) {
      const TriPre tp = tri_pre(sc->tris + 9ull * t);  // oracle_ray_triangle's first steps
      if (!cone_may_hit(ov, ax, cos_c, sin_c, tp)) continue;
      for (uint32_t s = 0; s < N; ++s) {
        const double* dd = &dirs[((size_t)i * N + s) * 3];
        const double tt = ray_triangle_pre(ov, V3{dd[0], dd[1], dd[2]}, tp.v0, tp.e1, tp.e2,
                                           tp.cut);
        if (tt >= 0.0) h[s].push_back({tt, t});
      }
    }
  });
  // Phase 2: per subray, steps O2 (from its hits) .. O5
  run_pool(n_pulses * (int64_t)N, [&](int64_t k) {
    const int64_t i = k / N;
    const uint32_t s = (uint32_t)(k % N);
    HitList hits;
    for (int64_t b = 0; b < nblk; ++b) {
      HitList& hb = blk_hits[((size_t)i * nblk + b) * N + s];
      hits.insert(hits.end(), hb.begin(), hb.end());
      HitList().swap(hb);
    }
    simulate_subray(sc, pr, origins + 3 * i, directions + 3 * i, pulse_ids[i], i, s,
                    theta.data(), phi.data(), hits, out);
  });
  run_pool(n_pulses, [&](int64_t i) { finish_pulse(pr, times ? times[i] : 0.0, pulse_ids[i], i, out);
  });
  return 0;
}

}  // extern "C"
