// trace.cu -- K6a (beam pre-pass) and K6: subray fan-out + nearest hit +
// transmissive voxels + radiometry.
//
// K6a: one thread per pulse walks the top of the BVH with the cone of all its
// subrays and lists the subtrees K6 must enter (near-first, with a lower bound
// of the entry distance), plus the pulse frame (DESIGN.md s.7.0).
// K6: one thread per (pulse, subray) -- lanes mapped to subrays along a Hilbert
// curve over the footprint, pulses padded to whole warps when that is cheap --
// so the lanes of a warp carry a compact patch of nearly parallel subrays
// and walk the same BVH nodes as a masked packet from K6a's
// entries: coherent float4 node loads served from L1.
//
// Precision contract (DESIGN.md s.3 C-0):
//   * subray directions in fp64 (P:199 pattern, R2/R4 frame);
//   * BVH boxes tested in fp32 with a conservative relative slack, so the
//     fp32 ray never culls a box the fp64 ray enters;
//   * every leaf triangle is decided by fp64 Moller-Trumbore on the fp32
//     vertices (the exact definition the oracle uses), nearest by fp64 t,
//     exact ties -> lower primitive id (R22); an fp32 filter with a forward
//     error bound rejects definite misses and recognises definite hits, whose
//     fp64 decision is deferred to the end of the walk;
//   * the voxel march (3D-DDA) computes each plane crossing directly in fp64
//     (no accumulated increments), chord lengths, exp(-sigma L), -ln(u)/sigma
//     in fp64 (R17-R20);
//   * range, Eq. 1/2 intensity and Eq. 7 amplitude in fp64 (R5, R14, R16).
#include <type_traits>
#include <math.h>

#include "internal.cuh"
#include "philox.cuh"

namespace helios {
namespace {

constexpr float kBoxSlack = 1e-6f;  // >> 5 * 2^-24 relative error of an fp32 slab value

// fp64 helpers with explicit round-to-nearest intrinsics: no FMA contraction,
// so every expression below evaluates exactly like the oracle's (same
// operation tree, IEEE double, -ffp-contract=off): decisions at shared edges
// and voxel faces are then bit-identical on both sides (P1 in DESIGN.md).
struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dif(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ D3 sub(D3 a, D3 b) { return {dif(a.x, b.x), dif(a.y, b.y), dif(a.z, b.z)}; }
__device__ __forceinline__ D3 scale(D3 a, double s) { return {mul(a.x, s), mul(a.y, s), mul(a.z, s)}; }
__device__ __forceinline__ D3 vadd(D3 a, D3 b) { return {add(a.x, b.x), add(a.y, b.y), add(a.z, b.z)}; }
__device__ __forceinline__ double dot(D3 a, D3 b) {
  return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z));
}
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {dif(mul(a.y, b.z), mul(a.z, b.y)), dif(mul(a.z, b.x), mul(a.x, b.z)),
          dif(mul(a.x, b.y), mul(a.y, b.x))};
}
__device__ __forceinline__ double norm(D3 a) { return __dsqrt_rn(dot(a, a)); }

#ifndef HELIOS_RCP_APPROX
#define HELIOS_RCP_APPROX 1
#endif
__device__ __forceinline__ float safe_inv(float d) {
  // a zero component would give (b - o) * inf = NaN on a box face through the
  // origin; 1e-30 keeps the slab finite and the test conservative
  const float x = fabsf(d) < 1e-30f ? copysignf(1e-30f, d) : d;
#if HELIOS_RCP_APPROX
  // rcp.approx: <= 1 ulp (2^-23 relative; |x| >= 1e-30 is never subnormal), so
  // a slab value carries <= 5 u of relative error, still << kBoxSlack
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
#else
  return __frcp_rn(x);  // correctly rounded: the value of 1.0f / x
#endif
}

// Slab test of one child box; returns the entry distance (or +inf on a miss).
// t = (b - o) * inv per slab has a purely RELATIVE error <= 5u (u = 2^-24:
// difference, approximate reciprocal (2u), product, and the fp32 rounding of
// the fp64 direction), whatever the direction (zero components are replaced by
// +-1e-30, so no NaN); the interval is widened by the relative slack
// kBoxSlack >> 4u: the fp32 test never culls a box the fp64 ray enters.
// (An fma(b, inv, -o*inv) form saves 6 instructions but carries an absolute
// error ~u |o * inv|, unbounded for axis-parallel rays -- not used.)
__device__ __forceinline__ float box_enter(float lox, float hix, float loy, float hiy, float loz,
                                           float hiz, float ox, float oy, float oz, float ix,
                                           float iy, float iz, float tbest) {
  const float tx0 = (lox - ox) * ix, tx1 = (hix - ox) * ix;
  const float ty0 = (loy - oy) * iy, ty1 = (hiy - oy) * iy;
  const float tz0 = (loz - oz) * iz, tz1 = (hiz - oz) * iz;
  const float tmin = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
  const float tmax = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tbest));
  constexpr float kWiden = (1.0f + kBoxSlack) / (1.0f - kBoxSlack);
  return (tmin <= tmax * kWiden) ? tmin : INFINITY;
}

// fp64 Moller-Trumbore (the oracle's definition and operation order, R21):
// t or -1.  The degeneracy cut |det| <= 1e-12 |e1||e2| is evaluated squared
// (no square roots); it differs from the oracle's form only for rays within
// ~1e-16 relative of the cut (parallel to the plane).
__device__ __forceinline__ double mt64(const D3& o, const D3& d, const TriRecord& tr) {
  const D3 v0 = d3(tr.a.x, tr.a.y, tr.a.z);
  const D3 e1 = sub(d3(tr.b.x, tr.b.y, tr.b.z), v0);
  const D3 e2 = sub(d3(tr.c.x, tr.c.y, tr.c.z), v0);
  const D3 p = cross(d, e2);
  const double det = dot(e1, p);
  if (mul(det, det) <= mul(mul(1e-24, dot(e1, e1)), dot(e2, e2))) return -1.0;
  const double inv = __drcp_rn(det);
  const D3 s = sub(o, v0);
  const double u = mul(dot(s, p), inv);
  if (u < 0.0 || u > 1.0) return -1.0;
  const D3 q = cross(s, e1);
  const double v = mul(dot(d, q), inv);
  if (v < 0.0 || add(u, v) > 1.0) return -1.0;
  const double t = mul(dot(e2, q), inv);
  return t > 0.0 ? t : -1.0;
}

// t of a hit the fp32 filter certified (mt32_classify == 2: |det|, u, v,
// 1 - u - v and t each beyond its forward-error bound, so the oracle's fp64
// test accepts it: its degeneracy cut |det| <= 1e-12 |e1||e2| lies far below
// the filter's det bound 32u |d|_1 |e1|_1 |e2|_1, and u, v keep their signs),
// by the oracle's own operations for t: det = e1.(d x e2), q = s x e1,
// t = (e2.q) / det -- bitwise mt64's t, without the tests it cannot fail.
__device__ __forceinline__ double mt64_t(const D3& o, const D3& d, const TriRecord& tr) {
  const D3 v0 = d3(tr.a.x, tr.a.y, tr.a.z);
  const D3 e1 = sub(d3(tr.b.x, tr.b.y, tr.b.z), v0);
  const D3 e2 = sub(d3(tr.c.x, tr.c.y, tr.c.z), v0);
  const double det = dot(e1, cross(d, e2));
  const double inv = __drcp_rn(det);
  const D3 q = cross(sub(o, v0), e1);
  return mul(dot(e2, q), inv);
}

// fp32 prefilter.  Returns true only when the triangle is DEFINITELY not a
// candidate (a miss of the fp64 test, or a hit farther than t_hi); otherwise
// the fp64 test above decides.  Forward-error argument: e1, e2, s are
// differences of fp32 inputs (relative error <= u = 2^-24 per component), the
// fp32 direction differs from the fp64 one by <= u relative per component, and
// each triple product (det, u*det, v*det, t*det) is a 5-operation sum of
// products, so |computed - exact| <= 8u * sum|terms| <= 8u * |a|_1 |b|_1 |c|_1.
// The margins below use 32u (4x slack) plus the rounding of the comparisons.
struct F3 {
  float x, y, z;
};
__device__ __forceinline__ F3 fsub(F3 a, F3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ float fdot(F3 a, F3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ F3 fcross(F3 a, F3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ float l1(F3 a) { return fabsf(a.x) + fabsf(a.y) + fabsf(a.z); }

// The same filter with a third outcome: 2 = a DEFINITE hit (u >= 0, v >= 0,
// u + v <= 1 and t > 0 each hold beyond the error bound, so the fp64 test
// accepts it) with t in [tlo, tup]; 1 = decide in fp64; 0 = not a candidate.
// A definite hit's fp64 evaluation can wait: its interval already bounds the
// ray's nearest hit from above (packet traversal, deferred decision).
__device__ __forceinline__ int mt32_classify(const F3& o, const F3& d, float dl1,
                                             const TriRecord& fr, float t_hi, float& tlo,
                                             float& tup) {
  // the bounds of mt32_definite_miss, factored as (kU |d|_1)(|e1|_1 |e2|_1)
  // etc., and tested as soon as each value exists (the coherent lanes of a
  // packet mostly leave together).  kU = HELIOS_FILTER_U x u on the 8u
  // first-order bound (default 32: 4x slack)
#ifndef HELIOS_FILTER_U
#define HELIOS_FILTER_U 32.0f
#endif
  constexpr float kU = HELIOS_FILTER_U * 5.9604645e-8f;
  // the filter record (lbvh.cu k_permute): v0, the fp32 edges e1 = v1 - v0,
  // e2 = v2 - v0 (correctly rounded differences), A = |e1|_1, B = |e2|_1, A B
  // -- the values this filter used to compute per test, bit for bit
  const F3 v0 = {fr.a.x, fr.a.y, fr.a.z};
  const F3 e1 = {fr.b.x, fr.b.y, fr.b.z};
  const F3 e2 = {fr.c.x, fr.c.y, fr.c.z};
  const F3 sv = fsub(o, v0);
  const float A = fr.b.w, B = fr.c.w, S = l1(sv);
  const float kd = kU * dl1, AB = fr.a.w;
  const F3 p = fcross(d, e2);
  const float det = fdot(e1, p);
  const float err_det = kd * AB;
  const float adet = fabsf(det);
  if (!(adet > err_det)) return 1;  // sign of det uncertain (or NaN): decide in fp64
  const float sg = det > 0.0f ? 1.0f : -1.0f;
  const float nu = fdot(sv, p) * sg;
  const float err_u = kd * S * B;
  if (nu < -err_u || nu - adet > err_u + err_det) return 0;  // u < 0, u > 1
  const F3 q = fcross(sv, e1);
  const float nv = fdot(d, q) * sg;
  const float err_v = kd * S * A;
  if (nv < -err_v) return 0;                                  // v < 0
  const float esum = (err_u + err_v + err_det) * 1.0001f;
  if ((nu + nv) - adet > esum) return 0;                      // u + v > 1
  const float nt = fdot(e2, q) * sg;
  const float err_t = kU * AB * S;
  if (nt < -err_t) return 0;                                  // t < 0
  // t = nt / adet > t_hi (cannot be the nearest hit)
  if (t_hi < 3.0e38f && nt - t_hi * adet > (err_t + t_hi * err_det) * 1.0001f + 1e-30f) return 0;
  if (nu >= err_u && nv >= err_v && nt > err_t && (nu + nv) + esum <= adet) {
    tlo = __fdividef(nt - err_t, adet + err_det) * (1.0f - 1e-6f);
    tup = __fdividef(nt + err_t, adet - err_det) * (1.0f + 1e-6f);
    return 2;
  }
  return 1;
}

// Per-lane nearest-hit state of the packet traversal: the exact (fp64
// decided) nearest so far, at most one deferred definite hit, and `bound`, an
// fp32 upper bound of the final nearest t (culls boxes, triangles, entries).
struct HitState {
  double t_best;
  uint32_t best_id, best_k;
  uint32_t def_k;  // deferred definite hit (triangle slot) or kNoTri
  float def_lo;    // its t interval's lower end
  float bound;
};
constexpr uint32_t kNoTri = 0xFFFFFFFFu;

__device__ __forceinline__ void take_hit(HitState& hs, double t, uint32_t id, uint32_t k) {
  if (t < hs.t_best || (t == hs.t_best && id < hs.best_id)) {
    hs.t_best = t;
    hs.best_id = id;
    hs.best_k = k;
  }
}

__device__ __forceinline__ TriRecord load_tri(const TriRecord* __restrict__ t, uint32_t k) {
  TriRecord r;
  r.a = __ldg(&t[k].a);
  r.b = __ldg(&t[k].b);
  r.c = __ldg(&t[k].c);
  return r;
}

#ifndef HELIOS_EXP_FILTER
#define HELIOS_EXP_FILTER 1
#endif
#ifndef HELIOS_DDA_RCP
#define HELIOS_DDA_RCP 1
#endif
// crossing of plane org + k vs, computed directly (no accumulated increments).
// HELIOS_DDA_RCP = 0: the oracle's exact operation ((org + k vs) - o) / d;
// 1 (default): times the per-ray reciprocal 1/d -- within 2 ulp of the
// quotient; the sub-ulp shifts of crossing times only move chord lengths by
// ~1e-16 relative (transmission decisions within the 1e-12 margin rule) and
// can turn an exact corner tie into a 1e-16-long segment, whose draw passes
// with probability 1 - 1e-16 (DESIGN.md s.7.1)
__device__ __forceinline__ double plane_t(double org, uint32_t k, double vs, double o, double d,
                                          double id) {
#if HELIOS_DDA_RCP
  (void)d;
  return __dmul_rn(__dsub_rn(__dadd_rn(org, __dmul_rn((double)k, vs)), o), id);
#else
  (void)id;
  return __ddiv_rn(__dsub_rn(__dadd_rn(org, __dmul_rn((double)k, vs)), o), d);
#endif
}

// a[i] for a runtime i in {0, 1, 2} by selects: the 3-element state arrays of
// the voxel march stay in registers (a runtime subscript would put them in
// local memory)
template <class T>
__device__ __forceinline__ T pick3(const T (&a)[3], int i) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}
template <class T>
__device__ __forceinline__ void put3(T (&a)[3], int i, T v) {
  a[0] = i == 0 ? v : a[0];
  a[1] = i == 1 ? v : a[1];
  a[2] = i == 2 ? v : a[2];
}

// Opaque / scaled voxel cube (Eq. 5; R31): minimum corner and side
// of voxel (ix, iy, iz), the oracle's operation order.
__device__ __forceinline__ double voxel_cube(const TraceArgs& a, const int idx[3], uint32_t id,
                                             float pad, double lo[3]) {
  const double org[3] = {a.gx0, a.gy0, a.gz0};
  if (a.voxel_mode != HELIOS_VOXEL_SCALED) {
#pragma unroll
    for (int k = 0; k < 3; ++k) lo[k] = __dadd_rn(org[k], __dmul_rn((double)idx[k], a.vs));
    return a.vs;
  }
  const double side = __dmul_rn(a.vs, pow(fmin(1.0, __ddiv_rn((double)pad, a.pad_max)),
                                          a.scale_alpha));
  double sh[3] = {0.0, 0.0, 0.0};
  if (a.scale_shift) {
    // stream tag 2: key (seed_lo, seed_hi ^ 2), counter (voxel id, 0, 0, 0)
    const uint4 x = philox4x32_10(make_uint4(id, 0u, 0u, 0u),
                                  make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32) ^ 2u));
    const uint32_t xs[3] = {x.x, x.y, x.z};
#pragma unroll
    for (int k = 0; k < 3; ++k)
      sh[k] = __dmul_rn(__dsub_rn(__dmul_rn((double)(xs[k] >> 8), 1.0 / 16777216.0), 0.5),
                        __dsub_rn(a.vs, side));
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double centre = __dadd_rn(org[k], __dmul_rn(__dadd_rn((double)idx[k], 0.5), a.vs));
    lo[k] = __dsub_rn(__dadd_rn(centre, sh[k]), __dmul_rn(0.5, side));
  }
  return side;
}

// fp64 slab test of a cube: entry t (> 0) and entry axis (largest near-plane
// time, lowest axis on ties) -- the oracle's ray_cube.
__device__ __forceinline__ bool ray_cube(const double o[3], const double d[3], const double lo[3],
                                         double side, double* t_enter, int* axis) {
  double tn = -INFINITY, tf = INFINITY;
  int ax = -1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double l = lo[k], h = __dadd_rn(lo[k], side);
    if (d[k] == 0.0) {
      if (o[k] < l || o[k] > h) return false;
      continue;
    }
    double t0 = __ddiv_rn(__dsub_rn(l, o[k]), d[k]), t1 = __ddiv_rn(__dsub_rn(h, o[k]), d[k]);
    if (t0 > t1) {
      const double tt = t0;
      t0 = t1;
      t1 = tt;
    }
    if (t0 > tn) {
      tn = t0;
      ax = k;
    }
    tf = fmin(tf, t1);
  }
  if (!(tn <= tf) || !(tn > 0.0) || ax < 0) return false;
  *t_enter = tn;
  *axis = ax;
  return true;
}

// Warp-cooperative masked packet traversal.  The 32 lanes of a warp hold
// consecutive (pulse, subray) rays -- the nearly parallel subrays of one or
// two pulses (beam divergence <= 0.5 mrad here).  The warp walks ONE
// path through the tree: at each node every lane whose bit is in the mask
// tests both child boxes against its own ray and t_best; a child is visited
// with the mask of the lanes that hit it (ballot), the far child is pushed
// with its own mask.  Control flow is warp-uniform, the node load is one
// broadcast per warp, and the stack of (node, mask) pairs is distributed over
// the lanes' registers (entry i lives in lane i % 32), so no local memory.
// Every lane visits a superset of the nodes its own per-ray traversal would
// visit, so the result is identical.
template <bool INSTR>
__device__ __forceinline__ void traverse_packet(const TraceArgs& a, unsigned m, int32_t ref,
                                                const D3& O, const D3& D, const F3& O32,
                                                const F3& D32, float dl1, float ix, float iy,
                                                float iz, HitState& hs,
                                                unsigned long long& c_nodes,
                                                unsigned long long& c_tris,
                                                unsigned long long& c_f64, unsigned* wc) {
  const unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int32_t stA_r = 0, stB_r = 0;
  unsigned stA_m = 0, stB_m = 0;
  int sp = 0;
  auto pop = [&]() -> bool {
    if (sp == 0) return false;
    --sp;
    ref = __shfl_sync(kFull, sp < 32 ? stA_r : stB_r, sp & 31);
    m = __shfl_sync(kFull, sp < 32 ? stA_m : stB_m, sp & 31);
    return true;
  };
  for (;;) {
    const bool mine = (m >> lane) & 1u;
    if (INSTR) ++wc[1];  // warp steps (nodes + leaves), counted once per warp
    if (ref_is_leaf(ref)) {
      if (INSTR) wc[2] += leaf_count(ref);  // triangles the warp iterates
      if (mine) {
        const uint32_t first = leaf_first(ref), cnt = leaf_count(ref);
        for (uint32_t k = first; k < first + cnt; ++k) {
          const TriRecord fr = load_tri(a.filt, k);
          if (INSTR) ++c_tris;
          float tlo, tup;
          const int cls = mt32_classify(O32, D32, dl1, fr, hs.bound, tlo, tup);
          if (cls == 0) continue;
          // a definite hit is deferred when it is the first, or surely nearer
          // than the deferred one (which then cannot be the nearest)
          if (cls == 2 && (hs.def_k == kNoTri || tup < hs.def_lo)) {
            hs.def_k = k;
            hs.def_lo = tlo;
            hs.bound = fminf(hs.bound, tup);
            continue;
          }
          if (INSTR) {
            ++c_f64;
            // warp-level: one count per group of lanes running this fp64 test together
            if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) ++wc[4];
            wc[5] += cls == 2;  // a second definite hit, not surely nearer
          }
          const TriRecord tr = load_tri(a.tris, k);  // the exact vertices and id
          const double t = mt64(O, D, tr);
          if (t > 0.0) {
            take_hit(hs, t, __float_as_uint(tr.a.w), k);
            hs.bound = fminf(hs.bound, __double2float_ru(t));
          }
        }
      }
      if (!pop()) break;
      continue;
    }
    const Node* nd = a.nodes + ref;
    const float4 xy0 = __ldg(&nd->xy0), xy1 = __ldg(&nd->xy1), z01 = __ldg(&nd->z01),
                 rf = __ldg(&nd->ref);
    // every lane tests (the warp issues the instructions either way); lanes
    // outside the mask are masked out of the result -- no divergent branch
    float t0 = INFINITY, t1 = INFINITY;
    if (mine) {
      if (INSTR) ++c_nodes;
      const float tb = hs.bound;
      t0 = box_enter(xy0.x, xy0.y, xy0.z, xy0.w, z01.x, z01.y, O32.x, O32.y, O32.z, ix, iy, iz,
                     tb);
      t1 = box_enter(xy1.x, xy1.y, xy1.z, xy1.w, z01.z, z01.w, O32.x, O32.y, O32.z, ix, iy, iz,
                     tb);
    }
    const int32_t r0 = __float_as_int(rf.x), r1 = __float_as_int(rf.y);
    const bool h0 = t0 < INFINITY, h1 = t1 < INFINITY;
    const unsigned m0 = __ballot_sync(kFull, h0), m1 = __ballot_sync(kFull, h1);
    if (m0 && m1) {
      const unsigned both = m0 & m1;
      const unsigned pref1 = __ballot_sync(kFull, h0 && h1 && t1 < t0);
      const bool near0 = both ? (2 * __popc(pref1) <= __popc(both)) : (__popc(m0) >= __popc(m1));
      const int32_t far_r = near0 ? r1 : r0;
      const unsigned far_m = near0 ? m1 : m0;
      if (lane == (sp & 31)) {
        if (sp < 32) {
          stA_r = far_r;
          stA_m = far_m;
        } else {
          stB_r = far_r;
          stB_m = far_m;
        }
      }
      ++sp;
      HELIOS_DASSERT(sp <= kStackSize);  // the build checked depth <= kStackSize
      ref = near0 ? r0 : r1;
      m = near0 ? m0 : m1;
    } else if (m0) {
      ref = r0;
      m = m0;
    } else if (m1) {
      ref = r1;
      m = m1;
    } else {
      if (!pop()) break;
    }
  }
}

// Pulse frame (R4, R24): d = the direction normalised in fp64 (false
// and a placeholder frame for a zero / non-finite direction: the pulse reports
// no hit); a = x if |d_z| > 0.9 else z; u = normalize(a x d); v = d x u.
__device__ __forceinline__ bool pulse_frame(const float* dir, D3& Dp, D3& U, D3& V) {
  Dp = d3(__ldg(dir), __ldg(dir + 1), __ldg(dir + 2));
  const double dn = norm(Dp);
  bool ok = true;
  if (!(dn > 0.0) || !isfinite(dn)) {
    ok = false;
    Dp = d3(0.0, 0.0, 1.0);  // placeholder
  } else {
    Dp = scale(Dp, __drcp_rn(dn));
  }
  const D3 ax = fabs(Dp.z) > 0.9 ? d3(1.0, 0.0, 0.0) : d3(0.0, 0.0, 1.0);
  U = cross(ax, Dp);
  U = scale(U, __drcp_rn(norm(U)));
  V = cross(Dp, U);
  return ok;
}

// ---- K6a: beam pre-pass.  The subrays of a pulse share its origin and lie in
// the cone of half-angle max_i theta_i about its axis (R2).  One
// thread per pulse walks the top of the tree with that cone and lists the
// subtrees K6 must enter, near-first: a node is listed once it is small next
// to the cone's cross-section (extent <= beam_k * radius at its entry
// distance; below that the per-subray tests of K6 cull better than the cone)
// or when it is a leaf.  K6 then starts its packet walks at the listed nodes
// instead of at the root, so the top levels are tested once per pulse
// instead of once per warp of subrays.
//
// Conservative by construction: the listed subtrees cover every node whose
// box an fp64 subray enters.  The cone is replaced by the box of directions
// (per axis, the exact component range over the cone, widened by 1e-9 and
// rounded outward to fp32): for a box [bl, bh], t * [lo, hi] must meet
// [bl - o, bh - o] on every axis for some t >= 0 -- the interval form of the
// slab test.  In fp32: each bound (b - o) * (1 / lo or hi) carries <= 3u of
// purely relative error (u = 2^-24; difference, correctly rounded reciprocal,
// product; signs exact), so widening by the relative slack kBoxSlack keeps
// the test conservative (the same argument as K6's box test).
struct Cone {
  float o[3];
  // per axis, with P = (bh - o) / lo and Q = (bl - o) / hi (lo, hi: the
  // direction interval): mode lo > 0 -> t in [Q, P]; hi < 0 (the inequalities
  // flip) -> t in [P, Q]; lo < 0 < hi -> t >= P, Q.  Branch-free: a lower-bound
  // term that does not apply gets multiplier 0 (-> 0, harmless under max with
  // t >= 0); an upper-bound term that does not apply is fma(e, 0, +inf).
  float lp[3], lq[3];  // lower-bound multipliers of (bh - o) and (bl - o)
  float up[3], uq[3];  // upper-bound multipliers
  float cp[3], cq[3];  // upper-bound addends: 0 or +inf
};

// entry distance (a lower bound of every subray's entry parameter) or +inf
__device__ __forceinline__ float cone_box(const Cone& c, float lx, float hx, float ly, float hy,
                                          float lz, float hz) {
  const float bl[3] = {lx, ly, lz}, bh[3] = {hx, hy, hz};
  float tlo = 0.0f, thi = INFINITY;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float ep = bh[k] - c.o[k], eq = bl[k] - c.o[k];
    tlo = fmaxf(tlo, fmaxf(ep * c.lp[k], eq * c.lq[k]));
    thi = fminf(thi, fminf(fmaf(ep, c.up[k], c.cp[k]), fmaf(eq, c.uq[k], c.cq[k])));
  }
  constexpr float kWiden = (1.0f + kBoxSlack) / (1.0f - kBoxSlack);
  return tlo <= thi * kWiden ? tlo * (1.0f - kBoxSlack) : INFINITY;
}

#ifndef HELIOS_BEAM_T
#define HELIOS_BEAM_T 128  // K6a threads per block
#endif
#ifndef HELIOS_BEAM_PREFETCH
#define HELIOS_BEAM_PREFETCH 1  // far children prefetched into L1 (C3 K6a -4.5 %, C5 +2 %)
#endif
template <bool INSTR>
__global__ void __launch_bounds__(HELIOS_BEAM_T) k_beam(const TraceArgs a) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.n_pulses) return;
  int2* row = a.entries + p * kEntryStride;
  // the pulse frame, once per pulse for all its subrays in K6
  D3 Dp, U, V;
  const bool ok = pulse_frame(a.direction + 3 * p, Dp, U, V);
  double2* f = reinterpret_cast<double2*>(a.frames) + p * 5;
  f[0] = make_double2(Dp.x, Dp.y);
  f[1] = make_double2(Dp.z, U.x);
  f[2] = make_double2(U.y, U.z);
  f[3] = make_double2(V.x, V.y);
  f[4] = make_double2(V.z, ok ? 1.0 : 0.0);
  if (!ok) {  // K6 reports the pulse as hitless
    row[0] = make_int2(0, 0);
    return;
  }
  Cone c;
  const double dd[3] = {Dp.x, Dp.y, Dp.z};
  const double sa = a.cone_sin;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c.o[k] = __ldg(a.origin + 3 * p + k);
    // over the cone, component k lies in d_k cos(a) -+ sqrt(1 - d_k^2) sin(a);
    // 1 - cos(a) <= sin^2(a)
    const double h = sqrt(fmax(0.0, 1.0 - dd[k] * dd[k])) * sa + fabs(dd[k]) * sa * sa + 1e-9;
    float lo = __double2float_rd(dd[k] - h), hi = __double2float_ru(dd[k] + h);
    int mode;
    if (lo >= 1e-30f) {
      mode = 0;
    } else if (hi <= -1e-30f) {
      mode = 1;
    } else {  // contains 0 (or nearly): widen to |lo|, |hi| >= 1e-30 (finite reciprocals)
      mode = 2;
      lo = fminf(lo, -1e-30f);
      hi = fmaxf(hi, 1e-30f);
    }
    const float rl = __frcp_rn(lo), rh = __frcp_rn(hi);
    c.lp[k] = mode == 0 ? 0.0f : rl;
    c.lq[k] = mode == 1 ? 0.0f : rh;
    c.up[k] = mode == 0 ? rl : 0.0f;
    c.cp[k] = mode == 0 ? 0.0f : INFINITY;
    c.uq[k] = mode == 1 ? rh : 0.0f;
    c.cq[k] = mode == 1 ? 0.0f : INFINITY;
  }
  const float kr = (float)(a.beam_k * sa);  // hand-over: extent <= beam_k * cone radius
  int visits = 0;
  // work stack of (ref, entry distance); bit i of `emit` marks entry i as
  // final (listed when popped).  Invariant: count + sp <= kEntryMax, so the
  // list never overflows: a node is expanded only while both children still
  // fit, else it is listed whole (coarser, still exact).  Listed distances are
  // shrunk by kBoxSlack: K6 drops a lane from an entry only when its nearest
  // hit is strictly nearer than any point of the box.
  int32_t stk[kEntryMax];
  float stt[kEntryMax];
  uint32_t emit = 0;
  int sp = 0, cnt = 0;
  constexpr int cap = kEntryMax;
  // the node to handle next stays in registers (the near child of the node
  // just expanded: it would be pushed and popped at once); only far children
  // go through the stack in local memory.  Same order, same lists.
  int32_t ref = a.root;
  float tref = 0.0f;
  bool fin = false, have = true;
  for (;;) {
    if (!have) {
      if (sp == 0) break;
      --sp;
      ref = stk[sp];
      tref = stt[sp];
      fin = (emit >> sp) & 1u;
    }
    have = false;
    // listed: final entries, leaves, and nodes whose children would not fit
    if (fin || ref_is_leaf(ref) || cnt + sp + 2 > cap) {
      HELIOS_DASSERT(cnt < kEntryMax);
      row[1 + cnt++] = make_int2(ref, __float_as_int(tref));
      continue;
    }
    const Node* nd = a.nodes + ref;
    const float4 xy0 = __ldg(&nd->xy0), xy1 = __ldg(&nd->xy1), z01 = __ldg(&nd->z01),
                 rf = __ldg(&nd->ref);
    ++visits;
    const float t0 = cone_box(c, xy0.x, xy0.y, xy0.z, xy0.w, z01.x, z01.y);
    const float t1 = cone_box(c, xy1.x, xy1.y, xy1.z, xy1.w, z01.z, z01.w);
    const bool h0 = t0 < INFINITY, h1 = t1 < INFINITY;
    const int32_t r0 = __float_as_int(rf.x), r1 = __float_as_int(rf.y);
    // listed as a whole once the node is small next to the cone's cross-section
    const float e0 = fmaxf(fmaxf(xy0.y - xy0.x, xy0.w - xy0.z), z01.y - z01.x);
    const float e1 = fmaxf(fmaxf(xy1.y - xy1.x, xy1.w - xy1.z), z01.w - z01.z);
    const bool f0 = e0 <= kr * t0, f1 = e1 <= kr * t1;
    const bool near0 = !h1 || (h0 && t0 <= t1);
    // far child (if both are hit) onto the stack, near child next
    const bool both = h0 && h1;
    if (both) {
      stk[sp] = near0 ? r1 : r0;
      stt[sp] = near0 ? t1 : t0;
      const bool ff = near0 ? f1 : f0;
      emit = ff ? emit | (1u << sp) : emit & ~(1u << sp);
#if HELIOS_BEAM_PREFETCH
      // the far child is expanded later: bring its node into L1 meanwhile
      if (!ff && !ref_is_leaf(stk[sp]))
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a.nodes + stk[sp]));
#endif
      ++sp;
    }
    if (h0 || h1) {
      ref = near0 ? r0 : r1;
      tref = near0 ? t0 : t1;
      fin = near0 ? f0 : f1;
      have = true;
    }
  }
  row[0] = make_int2(cnt, 0);
  if (INSTR) {
    const unsigned mask = __activemask();
    const unsigned w = __reduce_add_sync(mask, (unsigned)visits);
    if ((threadIdx.x & 31) == __ffs(mask) - 1 && w) atomicAdd(a.counters + 7, (unsigned long long)w);
  }
}

// A5 -> A6 hand-over of one subray's event (range R, amplitude A_s, prim; a
// miss has prim UINT32_MAX): the 8-B waveform record {k_s, A_s} K7 bins
// (k_s = floor(2 R / (c Delta)), R8/R9, computed here in fp64), the prim id
// K7 reads only to attribute a return (R13), and the optional 16-B export.
__device__ __forceinline__ void store_event(const TraceArgs& a, uint64_t slot, double R,
                                            float amp, uint32_t pid) {
  const bool hit = pid != 0xFFFFFFFFu;
  WaveRec w;
  w.k = hit ? (int32_t)bin_of(R, a.delta_ns, a.inv_bin) : -1;
  w.amp = hit ? amp : 0.0f;
  *reinterpret_cast<int2*>(a.wrec + slot) = make_int2(w.k, __float_as_int(w.amp));
  a.prim[slot] = pid;
  if (a.out) {
    helios_subray_hit h;
    h.range_m = hit ? R : __longlong_as_double(0x7FF8000000000000ll);  // NaN on a miss
    h.amplitude = w.amp;
    h.prim_id = pid;
    a.out[slot] = h;
  }
}

#ifndef HELIOS_TRACE_T
#define HELIOS_TRACE_T 128  // K6 threads per block
#endif
#ifndef HELIOS_TRACE_MIN_BLOCKS
#define HELIOS_TRACE_MIN_BLOCKS 9  // 56 registers: measured best (profiles/r02_k6_regs_ab.txt; r01: 64 > 80)
#endif
// GRID: 0 no voxel grid, 1 transmissive voxels, 2 opaque / scaled cubes --
// the A4 march is compiled in only where needed, so each scene kind keeps
// the traversal's register budget
// ENT: whether K6a's entry lists and pulse frames exist (every scene with
// an inner tree node unless the pre-pass is switched off) is known when the
// kernel is launched, so each kernel holds one copy of the inlined traversal:
// ENT walks the lists with the stored frames, !ENT walks from the root with
// the frame computed here.  Triangle scenes: 2024 -> 1376 instructions,
// spills 168 -> 100 B, K6 -1.2 % (C5), -2.4 % (C2, C3), -2.9 % (C6); the
// voxel kernel without lists (C4): spills 264 -> 188 B, K6 -1.2 %.  A further
// variant for warps that hold one pulse only (C5's 96 lanes: no second-pulse
// state) spilled less still but ran 3.5 % slower on C5
// (profiles/r02s5_ent_ab.txt).
template <bool INSTR, int GRID, bool ENT>
__global__ void __launch_bounds__(HELIOS_TRACE_T, HELIOS_TRACE_MIN_BLOCKS * 128 / HELIOS_TRACE_T) k_trace(const TraceArgs a) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // a pulse occupies a.lanes (>= N) consecutive threads: N, or N padded to
  // whole warps when that wastes few lanes (then no warp holds two pulses)
  const uint32_t NL = a.lanes;
  const uint64_t total = a.n_pulses * (uint64_t)NL;
  // one launch covers < 2^32 lanes (launch_trace checks): 32-bit division
  const uint32_t gq = (uint32_t)(gid < total ? gid : 0);
  const uint64_t pq0 = gq / NL;
  const bool in_range = gid < total && gq - (uint32_t)pq0 * NL < a.N;
  const uint32_t g32 = in_range ? gq : 0;  // padding / out-of-range lanes ride along
  const uint64_t p = g32 / NL;
  // lane position j of the pulse -> subray s (the table is in K6's lane order,
  // each entry carries its index; the record goes to slot s)
  const uint32_t j = g32 - (uint32_t)p * NL;
  HELIOS_DASSERT(j < NL);
  const SubrayConst sc = a.sub[j];
  HELIOS_DASSERT(!in_range || sc.index < a.N);
  const uint32_t s = sc.index;
  const uint64_t slot = p * a.N + s;  // [pulse][subray] (R4 order) in every output
  unsigned long long c_nodes = 0, c_tris = 0, c_vox = 0, c_voxret = 0, c_f64 = 0;
  // warp-level counts (instrumented variant): entries examined, packet steps,
  // leaf triangles iterated, entries walked -- once per warp, not per lane
  unsigned wc[6] = {0, 0, 0, 0, 0, 0};


  // ---- A2: subray fan-out (R2, R4), fp64
  // the pulse's entry row (K6a) is read only after the fan-out and a vote:
  // start bringing it into L1 now (no register, no scoreboard; C3 K6 -1.1 %)
  if (a.entries != nullptr) {
    const char* er = reinterpret_cast<const char*>(a.entries + p * kEntryStride);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(er));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(er + 128));
  }
  const float ox = __ldg(a.origin + 3 * p), oy = __ldg(a.origin + 3 * p + 1),
              oz = __ldg(a.origin + 3 * p + 2);
  D3 Dp, U, V;
  bool valid = in_range;
  if (ENT) {  // the pulse frame K6a computed (bitwise the same values)
    const double2* f = reinterpret_cast<const double2*>(a.frames) + p * 5;
    const double2 f0 = __ldg(f), f1 = __ldg(f + 1), f2 = __ldg(f + 2), f3 = __ldg(f + 3),
                  f4 = __ldg(f + 4);
    Dp = d3(f0.x, f0.y, f1.x);
    U = d3(f1.y, f2.x, f2.y);
    V = d3(f3.x, f3.y, f4.x);
    if (!(f4.y > 0.0)) valid = false;
  } else {
    valid = pulse_frame(a.direction + 3 * p, Dp, U, V) && in_range;
  }
  if (in_range && !valid && s == 0) atomicOr(a.err_flag, 1u);
  // d_s = cos(theta) d + sin(theta) (cos(phi) u + sin(phi) v)
  const D3 ring = vadd(scale(U, sc.cos_p), scale(V, sc.sin_p));
  const D3 D = vadd(scale(Dp, sc.cos_t), scale(ring, sc.sin_t));
  const D3 O = d3(ox, oy, oz);

  // ---- A3: nearest triangle (LBVH; fp32 boxes, fp64 decisions)
  double t_best = INFINITY;
  uint32_t best_id = 0xFFFFFFFFu, best_k = 0;
  if (a.n_tris > 0) {
    const float ix = safe_inv((float)D.x), iy = safe_inv((float)D.y), iz = safe_inv((float)D.z);
    const F3 O32 = {ox, oy, oz};
    const F3 D32 = {(float)D.x, (float)D.y, (float)D.z};
    const float dl1 = l1(D32);
    {
      const unsigned m = __ballot_sync(0xffffffffu, valid);
      if (m) {
        {
          // beam entry lists (K6a): the warp walks, pulse by pulse, the subtrees
          // the pulse's cone reaches, each with the lanes of that pulse; without
          // lists, one walk from the root with every lane.  A warp can hold the
          // subrays of two or more pulses.  Walking the leader pulse's entries,
          // the lanes of the next pulse join any entry its own list shares (lane
          // j holds that pulse's entry j; a vote finds it), and that entry is
          // skipped when the next pulse leads.
          HitState hs;
          hs.t_best = INFINITY;
          hs.best_id = 0xFFFFFFFFu;
          hs.best_k = 0;
          hs.def_k = kNoTri;
          hs.def_lo = INFINITY;
          hs.bound = INFINITY;
          const int lane = threadIdx.x & 31;
          unsigned rem = m, skip = 0;
          while (rem) {
            if (!ENT) {
              traverse_packet<INSTR>(a, rem, a.root, O, D, O32, D32, dl1, ix, iy, iz, hs,
                                     c_nodes, c_tris, c_f64, wc);
              break;
            }
            const uint32_t pq = __shfl_sync(0xffffffffu, (uint32_t)p, __ffs(rem) - 1);
            const bool in_q = valid && (uint32_t)p == pq;
            rem &= ~__ballot_sync(0xffffffffu, in_q);
            bool in_r = false;
            int2 er = make_int2(0, 0);
            int cntr = 0;
            if (rem) {  // the next pulse of the warp
              const uint32_t pr = __shfl_sync(0xffffffffu, (uint32_t)p, __ffs(rem) - 1);
              in_r = valid && (uint32_t)p == pr;
              const int2* rowr = a.entries + (uint64_t)pr * kEntryStride;
              cntr = __ldg(&rowr->x);
              if (lane < cntr) er = __ldg(rowr + 1 + lane);
            }
            unsigned taken = 0;  // entries of the next pulse walked here
            const int2* row = a.entries + (uint64_t)pq * kEntryStride;
            const int cnt = __ldg(&row->x);
            for (int i = 1; i <= cnt; ++i) {
              if ((skip >> (i - 1)) & 1u) continue;
              const int2 en = __ldg(row + i);
              // lanes whose nearest hit is already nearer than the box drop out
              bool go = in_q && !(hs.bound < __int_as_float(en.y));
              if (cntr) {
                const unsigned hit = __ballot_sync(0xffffffffu, lane < cntr && er.x == en.x) & ~taken;
                if (hit) {
                  const int j = __ffs(hit) - 1;
                  taken |= 1u << j;
                  const float tr = __int_as_float(__shfl_sync(0xffffffffu, er.y, j));
                  go = go || (in_r && !(hs.bound < tr));
                }
              }
              const unsigned me = __ballot_sync(0xffffffffu, go);
              if (INSTR) ++wc[0];  // entries the warp examines
              if (INSTR && me) ++wc[3];  // entries it walks
              if (me)
                traverse_packet<INSTR>(a, me, en.x, O, D, O32, D32, dl1, ix, iy, iz, hs,
                                       c_nodes, c_tris, c_f64, wc);
            }
            skip = taken;
          }
          // the deferred definite hit is decided last (in step across the warp)
          if (hs.def_k != kNoTri) {
            const TriRecord tr = load_tri(a.tris, hs.def_k);
            if (INSTR) ++c_f64;
            const double t = mt64_t(O, D, tr);
            if (t > 0.0) take_hit(hs, t, __float_as_uint(tr.a.w), hs.def_k);
          }
          t_best = hs.t_best;
          best_id = hs.best_id;
          best_k = hs.best_k;
        }
      }
    }
  }
  if (!valid) {
    if (in_range) store_event(a, slot, 0.0, 0.0f, 0xFFFFFFFFu);
    return;
  }

  // ---- A4: transmissive voxels before the triangle hit
  bool vox_hit = false;
  double t_vox = 0.0, sigma_vox = 0.0;
  uint32_t vox_id = 0;
  if (GRID != 0 && a.pad != nullptr) {
    const double org[3] = {a.gx0, a.gy0, a.gz0};
    const uint32_t nn[3] = {a.nx, a.ny, a.nz};
    const double o3[3] = {O.x, O.y, O.z}, d3v[3] = {D.x, D.y, D.z};
    double t_in = 0.0, t_out = (best_id != 0xFFFFFFFFu) ? t_best : INFINITY;
    bool inside = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double lo = org[ax], hi = add(org[ax], mul((double)nn[ax], a.vs));
      if (d3v[ax] == 0.0) {
        if (o3[ax] < lo || o3[ax] > hi) inside = false;
        continue;
      }
      double ta = __ddiv_rn(dif(lo, o3[ax]), d3v[ax]), tb = __ddiv_rn(dif(hi, o3[ax]), d3v[ax]);
      if (ta > tb) {
        const double tmp = ta;
        ta = tb;
        tb = tmp;
      }
      t_in = fmax(t_in, ta);
      t_out = fmin(t_out, tb);
    }
    if (inside && t_in < t_out) {
      // G(|d_z|) (R15)
      double G = 0.5;
      if (GRID == 1 && a.g_lut != nullptr) {
        const double x = fabs(D.z) * (double)(a.n_lut - 1);
        int64_t k = (int64_t)floor(x);
        k = k < 0 ? 0 : (k > (int64_t)a.n_lut - 2 ? (int64_t)a.n_lut - 2 : k);
        const double f = x - (double)k;
        G = (double)__ldg(a.g_lut + k) * (1.0 - f) + (double)__ldg(a.g_lut + k + 1) * f;
      }
      int idx[3];
      double tn[3];
      int stp[3];
      const double inv3[3] = {__drcp_rn(d3v[0]), __drcp_rn(d3v[1]), __drcp_rn(d3v[2])};
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const double c = (o3[ax] + t_in * d3v[ax] - org[ax]) / a.vs;
        int k = (int)floor(c);
        k = k < 0 ? 0 : (k >= (int)nn[ax] ? (int)nn[ax] - 1 : k);
        idx[ax] = k;
        stp[ax] = d3v[ax] > 0.0 ? 1 : (d3v[ax] < 0.0 ? -1 : 0);
        tn[ax] = stp[ax] > 0   ? plane_t(org[ax], (uint32_t)(k + 1), a.vs, o3[ax], d3v[ax],
                                          inv3[ax])
                 : stp[ax] < 0 ? plane_t(org[ax], (uint32_t)k, a.vs, o3[ax], d3v[ax], inv3[ax])
                               : INFINITY;
      }
      double t_cur = t_in;
      for (;;) {
        // empty 4^3 brick: jump to its exit crossing.  No decision happens in
        // it (PAD = 0 everywhere), and the state after the jump is the one the
        // cell-by-cell march would reach: every plane crossed before the exit
        // (the tie order x < y < z included) is counted per axis.
        if (a.bricks != nullptr) {
          const int bx = idx[0] >> kBrickShift, by = idx[1] >> kBrickShift,
                    bz = idx[2] >> kBrickShift;
          if (!__ldg(a.bricks + bx + a.nbx * (by + a.nby * bz))) {
            const int bi[3] = {bx, by, bz};
            double tb[3];
            int kb[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              kb[q] = stp[q] > 0 ? min((bi[q] + 1) << kBrickShift, (int)nn[q]) : bi[q] << kBrickShift;
              tb[q] = stp[q] != 0 ? plane_t(org[q], (uint32_t)kb[q], a.vs, o3[q], d3v[q], inv3[q])
                                  : INFINITY;
            }
            const int e = (tb[0] <= tb[1] && tb[0] <= tb[2]) ? 0 : (tb[1] <= tb[2] ? 1 : 2);
            const double t_bx = pick3(tb, e);
            if (INSTR) ++c_vox;
            if (!(t_bx < t_out)) break;  // the ray ends inside the empty brick
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              if (q == e || stp[q] == 0) continue;
              while (tn[q] < t_bx || (tn[q] == t_bx && q < e)) {
                idx[q] += stp[q];
                tn[q] = plane_t(org[q], (uint32_t)(stp[q] > 0 ? idx[q] + 1 : idx[q]), a.vs, o3[q],
                                d3v[q], inv3[q]);
              }
            }
            const int ste = pick3(stp, e), kbe = pick3(kb, e);
            const int ie = ste > 0 ? kbe : kbe - 1;
            if (ie < 0 || ie >= (int)pick3(nn, e)) break;
            put3(idx, e, ie);
            put3(tn, e,
                 plane_t(pick3(org, e), (uint32_t)(ste > 0 ? ie + 1 : ie), a.vs, pick3(o3, e),
                         pick3(d3v, e), pick3(inv3, e)));
            t_cur = t_bx;
            continue;
          }
        }
        const int ax = (tn[0] <= tn[1] && tn[0] <= tn[2]) ? 0 : (tn[1] <= tn[2] ? 1 : 2);
        const double t_exit = pick3(tn, ax);
        const double t_end = fmin(t_exit, t_out);
        const double L = t_end - t_cur;
        if (INSTR) ++c_vox;
        if (L > 0.0) {
          const uint32_t id = (uint32_t)idx[0] + a.nx * ((uint32_t)idx[1] + a.ny * (uint32_t)idx[2]);
          const float pad = __ldg(a.pad + id);
          if (GRID == 2 && pad > 0.0f) {
            // opaque / scaled cube (R31): the first one entered ahead of the triangle
            double lo[3], te;
            int eax;
            const double side = voxel_cube(a, idx, id, pad, lo);
            const double t_lim = (best_id != 0xFFFFFFFFu) ? t_best : INFINITY;
            if (ray_cube(o3, d3v, lo, side, &te, &eax) && te < t_lim) {
              vox_hit = true;
              t_vox = te;
              sigma_vox = __dmul_rn(a.voxel_refl, fabs(d3v[eax]));  // Lambertian face
              vox_id = id;
              if (INSTR) ++c_voxret;
              break;
            }
          } else if (GRID == 1 && pad > 0.0f) {
            const double sigma = (double)pad * G;  // Eq. 4 via the G LUT
            const double u = transmission_u(a.seed, a.pulse_base + p, s, id);
            // u < exp(-sigma L) decided by an fp32 estimate whenever u is
            // farther from it than its error bound, else by the fp64 exp:
            // the decision is the fp64 one either way.  For x = sigma L < 16.6
            // the estimate __expf(-(float)x) is within (2 + 1.17 x) ulp (<= 21.5
            // ulp = 1.3e-6 relative) of e^-(float)x, and rounding x to fp32
            // moves e^-x by <= x 2^-24 (<= 1e-6) relative: < 2.3e-6 in all,
            // below the 1e-5 margin.  For x >= 16.6, e^-x < 6.2e-8 and the
            // fp64 exp decides (u is a multiple of 2^-24 = 6e-8, so only u = 0
            // can pass there; the filter's bound is not needed).
            const double x = sigma * L;
            bool pass;
            if (HELIOS_EXP_FILTER && x < 16.6) {
              const double e32 = (double)__expf(-(float)x);
              pass = fabs(u - e32) > 1e-5 * e32 ? u < e32 : u < exp(-x);
            } else {
              pass = u < exp(-x);
            }
            if (!pass) {  // s = -ln(u)/sigma <= L: echo (R17)
              vox_hit = true;
              t_vox = t_cur + (-log(u)) / sigma;  // Eq. 6
              sigma_vox = sigma;
              vox_id = id;
              if (INSTR) ++c_voxret;
              break;
            }
          }
        }
        if (t_exit >= t_out) break;
        const int sta = pick3(stp, ax), ia = pick3(idx, ax) + sta;
        if (ia < 0 || ia >= (int)pick3(nn, ax)) break;
        put3(idx, ax, ia);
        put3(tn, ax,
             plane_t(pick3(org, ax), (uint32_t)(sta > 0 ? ia + 1 : ia), a.vs, pick3(o3, ax),
                     pick3(d3v, ax), pick3(inv3, ax)));
        t_cur = t_exit;
      }
    }
  }

  // ---- A5: range + radiometry (Eq. 1, 2, 7; R5, R14, R16)
  double R = 0.0, sig_eff = 0.0;
  uint32_t pid = 0xFFFFFFFFu;
  if (vox_hit) {
    R = t_vox;
    sig_eff = sigma_vox;
    pid = a.n_tris + vox_id;
  } else if (best_id != 0xFFFFFFFFu) {
    const TriRecord tr = load_tri(a.tris, best_k);
    const D3 v0 = d3(tr.a.x, tr.a.y, tr.a.z);
    const D3 n = cross(sub(d3(tr.b.x, tr.b.y, tr.b.z), v0), sub(d3(tr.c.x, tr.c.y, tr.c.z), v0));
    // |n.d| / (|n| |d|): only the amplitude depends on it (tolerance 1e-4
    // relative), so |d| = 1 (+-1e-16) is dropped and 1/|n| is the fp64 rsqrt
    // (<= 2 ulp) instead of a square root and a division
    const double cos_inc = fabs(dot(n, D)) * rsqrt(dot(n, n));
    R = t_best;
    sig_eff = (double)tr.b.w * cos_inc;
    pid = best_id;
  }
  float amp = 0.0f;
  if (pid != 0xFFFFFFFFu) {
    double I;
    if (a.eq2) {
      const double r = R * sc.sin_t;
      const double om = a.lambda_m * R / (kPi * a.w0 * a.w0);
      const double om0 = a.lambda_m * a.R0 / (kPi * a.w0 * a.w0);
      const double w = a.w0 * sqrt(om0 * om0 + om * om);
      I = (r == 0.0) ? a.I0 : a.I0 * exp(-2.0 * r * r / (w * w));
    } else {
      I = a.I0 * sc.w_far;
    }
    const double r2 = R * R;
    amp = (float)(a.K * sig_eff * I * __drcp_rn(r2 * r2));
  }
  store_event(a, slot, R, amp, pid);

  if (INSTR) {
    // warp-aggregated (one atomic per warp and counter; per-thread counts < 2^32)
    const unsigned mask = __activemask();
    const bool leader = (threadIdx.x & 31) == __ffs(mask) - 1;
    const unsigned long long v[5] = {c_nodes, c_tris, c_vox, c_voxret, c_f64};
    const int cslot[5] = {0, 1, 2, 3, 6};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const unsigned w = __reduce_add_sync(mask, (unsigned)v[i]);
      if (leader && w) atomicAdd(a.counters + cslot[i], (unsigned long long)w);
    }
    // warp-uniform counts: the leader's copy (every active lane holds the same)
    if (leader)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (wc[i]) atomicAdd(a.counters + 8 + i, (unsigned long long)wc[i]);
    // per lane: in-loop fp64 tests run by a lane-group leader, second definite hits
    const unsigned w4 = __reduce_add_sync(mask, wc[4]), w5 = __reduce_add_sync(mask, wc[5]);
    if (leader) {
      if (w4) atomicAdd(a.counters + 12, (unsigned long long)w4);
      if (w5) atomicAdd(a.counters + 13, (unsigned long long)w5);
    }
  }
}

}  // namespace

cudaError_t launch_beam(const TraceArgs& a, bool instrumented, cudaStream_t s) {
  if (a.n_pulses == 0) return cudaSuccess;
  if (a.entries == nullptr || a.frames == nullptr || ref_is_leaf(a.root))
    return cudaErrorInvalidValue;
  const unsigned T = HELIOS_BEAM_T;
  const uint64_t blocks = (a.n_pulses + T - 1) / T;
  if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  if (instrumented)
    k_beam<true><<<(unsigned)blocks, T, 0, s>>>(a);
  else
    k_beam<false><<<(unsigned)blocks, T, 0, s>>>(a);
  return cudaGetLastError();
}

// K6 / K6a use no shared memory and live on L1 hits (nodes, triangle
// records: 93 %): they ask for the smallest carveout (the largest L1) even
// where K7 blocks (44 KB of shared memory each) overlap them -- pipelined C5
// +1.4 %, C3 +1 %, exclusive times unchanged (profiles/r02s4/carveout_ab.txt;
// -1 leaves the driver's choice)
#ifndef HELIOS_K6_CARVEOUT
#define HELIOS_K6_CARVEOUT 0
#endif
cudaError_t launch_trace(const TraceArgs& a, bool instrumented, cudaStream_t s) {
#if HELIOS_K6_CARVEOUT >= 0
  static bool carve_set = [] {
    for (const void* f : {(const void*)k_trace<false, 0, false>, (const void*)k_trace<false, 0, true>,
                          (const void*)k_trace<false, 1, false>, (const void*)k_trace<false, 1, true>,
                          (const void*)k_trace<false, 2, false>, (const void*)k_trace<false, 2, true>,
                          (const void*)k_beam<false>})
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, HELIOS_K6_CARVEOUT);
    cudaGetLastError();
    return true;
  }();
  (void)carve_set;
#endif
  if (a.lanes < a.N) return cudaErrorInvalidValue;
  const uint64_t total = a.n_pulses * (uint64_t)a.lanes;
  if (total == 0) return cudaSuccess;
  const unsigned T = HELIOS_TRACE_T;
  const uint64_t blocks = (total + T - 1) / T;
  if (blocks > 0x7FFFFFFFull || total >= (1ull << 32)) return cudaErrorInvalidValue;
  const unsigned g = (unsigned)blocks;
  const int grid = a.pad == nullptr ? 0 : (a.voxel_mode == HELIOS_VOXEL_TRANSMISSIVE ? 1 : 2);
  const bool ent = a.entries != nullptr && a.frames != nullptr;
  auto go = [&](auto instr, auto gr) {
    if (ent) k_trace<decltype(instr)::value, decltype(gr)::value, true><<<g, T, 0, s>>>(a);
    else k_trace<decltype(instr)::value, decltype(gr)::value, false><<<g, T, 0, s>>>(a);
  };
  auto by_grid = [&](auto instr) {
    if (grid == 1) go(instr, std::integral_constant<int, 1>{});
    else if (grid == 2) go(instr, std::integral_constant<int, 2>{});
    else go(instr, std::integral_constant<int, 0>{});
  };
  if (instrumented) by_grid(std::true_type{});
  else by_grid(std::false_type{});
  return cudaGetLastError();
}

}  // namespace helios
