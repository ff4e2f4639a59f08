// waveform.cu -- K7: full-waveform binning + local-maximum peaks -> returns.
//
// One warp per pulse (grid-stride).  The pulse's 8-B subray records
// {k_s, A_s} (written by K6, which computes k_s from the fp64 range) are read
// once; the prim ids only when a return is attributed.  P:215: "the recorded
// power for each bin is taken as the sum of the subray's waveforms, shifted
// according to the different ranges of the subrays":
//
//   k_s  = floor(2 R_s / c / Delta)                  (R8, R9; in K6, the oracle's fp64 operations)
//   k0   = min_s k_s                                  (window anchor, R9)
//   W[k] = sum_s A_s p[k - (k_s - k0)],  p[j] = f((j + 1/2) Delta / tau),
//          f(x) = x^2 e^-x  (Eq. 3),  j < L_p = ceil(20 tau / Delta)
//   peak at k in [1, n_bins-2]: W[k] > W[k-1], W[k] > W[k+1], W[k] >= thr max W
//   (P:215 local-maximum filter; R11), earliest max_returns kept,
//   range (c/2)(k0 + k - j* + 1/2) Delta (R12), prim = argmax_s contribution (R13).
//
// Evaluation (deterministic, fp64, no atomics): the subrays of a pulse fall
// into few distinct bin offsets o_s = k_s - k0 (coherent footprint), so the
// amplitudes are first summed per offset group (each group in subray order),
// then each lane computes its bins W[k] = sum_o A_o p[k - o] directly.  Pulses
// whose offsets spread over >= kAggCap bins form match_any groups per 32-subray
// chunk and add each group's shifted kernel into W, group after group.
// The waveform window lives in a small per-warp shared-memory buffer; a pulse
// whose support exceeds it (rare: a footprint spanning > kWCap - L_p bins) is
// deferred to a second pass that keeps its row in a per-warp global scratch
// row.  Rows are stored as fp32 with 16-byte vector stores (zeros outside the
// support).
#include <math.h>

#include <algorithm>

#include "internal.cuh"
#include "philox.cuh"

namespace helios {
namespace {

#ifndef HELIOS_WAVE_WARPS
#define HELIOS_WAVE_WARPS 8
#endif
constexpr int kMaxWarps = HELIOS_WAVE_WARPS;
#ifndef HELIOS_WAVE_WCAP
#define HELIOS_WAVE_WCAP 512
#endif
#ifndef HELIOS_WAVE_MIN_BLOCKS
#define HELIOS_WAVE_MIN_BLOCKS 4
#endif
constexpr int kWCap = HELIOS_WAVE_WCAP;  // fp64 bins per warp in shared memory
constexpr int kAggCap = 64;   // offset groups handled by the grouped path
// ceil(2^32 / d): floor(x / d) = umulhi(x, c_inv[d]) for x <= 3168, 2 <= d <= 32
__constant__ uint32_t c_inv[33] = {
    0u, 0u, 2147483648u, 1431655766u, 1073741824u, 858993460u, 715827883u, 613566757u,
    536870912u, 477218589u, 429496730u, 390451573u, 357913942u, 330382100u, 306783379u,
    286331154u, 268435456u, 252645136u, 238609295u, 226050911u, 214748365u, 204522253u,
    195225787u, 186737709u, 178956971u, 171798692u, 165191050u, 159072863u, 153391690u,
    148102321u, 143165577u, 138547333u, 134217728u};
constexpr size_t kSmemCap = 200 * 1024;

// Echo width ("Optionally, a Gaussian may be fitted to the resulting
// waveform, to get a measure of echo width (i.e. standard deviation of the
// Gaussian)"; non-linear least squares).  Reading R28 (DESIGN.md s.3):
// the echo's bins -- W strictly decreasing away from the peak k, at most
// w = ceil(3 pulse_length / Delta) on each side; x = (i - k) Delta, y = W[i];
// g(x) = A exp(-(x-m)^2 / 2s^2); Levenberg-Marquardt from (W[k], 0, s0),
// lambda 1e-3, (J^T J + lambda diag J^T J) d = J^T r by Cramer's rule, accept iff
// the sum of squares drops (lambda /= 10) else lambda *= 10; converged when an
// accepted step has max |d_i| / (|p_i| + 1e-12) < 1e-10 or lambda > 1e16;
// 100 iterations without convergence, A <= 0, |m| > w Delta or |s| > w Delta
// (not identifiable from the window) -> NaN.
//
// Split in two: K7 finds each return's echo window (warp ballots over the
// fp64 waveform in shared memory) and appends a job {slot, window} to a
// per-launch list; k_fit then runs one LM per THREAD, summing the window
// sequentially in bin order (no warp reductions on the critical path; 1/s
// once per pass instead of a division per bin -- same optimum, rounding-level
// differences from the oracle's (x - m) / s).

// window [k + lo, k + hi] of the echo at k (all lanes; result warp-uniform)
__device__ __forceinline__ void echo_window(const double* __restrict__ W, uint32_t S, uint32_t nb,
                                            int k, int half, int& lo, int& hi) {
  const int lane = threadIdx.x & 31;
  auto wv = [&](int i) { return (uint32_t)i < S ? W[i] : 0.0; };  // bins >= S are zero
  lo = k;
  hi = k;
  for (int base = 0;; base += 32) {
    const int i = k - 1 - base - lane;
    const unsigned stop = __ballot_sync(0xffffffffu, !(i >= max(0, k - half) && wv(i) < wv(i + 1)));
    if (stop) {
      lo = k - base - (__ffs(stop) - 1);
      break;
    }
  }
  for (int base = 0;; base += 32) {
    const int i = k + 1 + base + lane;
    const unsigned stop = __ballot_sync(0xffffffffu,
                                        !(i <= min((int)nb - 1, k + half) && wv(i) < wv(i - 1)));
    if (stop) {
      hi = k + base + (__ffs(stop) - 1);
      break;
    }
  }
}

// The sum of squared residuals at (A, m, s) and, in the same pass over the
// window (one exp per bin), J^T J and J^T r there -- the values the oracle
// computes at an accepted point; a rejected candidate's are simply dropped
// (so every iteration costs one exp pass, not two after an accepted step).
struct FitEval {
  double sse, h00, h01, h02, h11, h12, h22, g0, g1, g2;
};
__device__ __forceinline__ FitEval fit_eval(const double* __restrict__ y, int n, int lo,
                                            double delta, double A, double m, double s) {
  FitEval f{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double is = 1.0 / s, Ais = A * is;  // one division per pass, not per bin
#pragma unroll 2
  for (int i = 0; i < n; ++i) {
    const double z = ((double)(lo + i) * delta - m) * is;
    const double e = exp(-0.5 * z * z);
    const double j0 = e, j1 = Ais * e * z, j2 = j1 * z;
    const double r = y[i] - A * e;
    f.sse += r * r;
    f.g0 += j0 * r; f.g1 += j1 * r; f.g2 += j2 * r;
    f.h00 += j0 * j0; f.h01 += j0 * j1; f.h02 += j0 * j2;
    f.h11 += j1 * j1; f.h12 += j1 * j2; f.h22 += j2 * j2;
  }
  return f;
}

// One LM fit per thread over the job list of one K7 launch.
__global__ void __launch_bounds__(64) k_fit(const FitJob* __restrict__ jobs,
                                             const double* __restrict__ ys, uint32_t stride,
                                             const unsigned* __restrict__ count, int half,
                                             double delta, double s0,
                                             helios_return* __restrict__ ret) {
  const unsigned nj = *count;
  for (unsigned j = blockIdx.x * blockDim.x + threadIdx.x; j < nj; j += gridDim.x * blockDim.x) {
    const FitJob job = jobs[j];
    const double* y = ys + (size_t)j * stride;
    const int n = job.n;
    const int lo = job.lo;  // first window bin relative to the peak: x_i = (lo + i) Delta
    double A = job.peak, m = 0.0, s = s0, lambda = 1e-3;
    FitEval c = fit_eval(y, n, lo, delta, A, m, s);  // at the current point
    bool converged = false;
    for (int it = 0; it < 100; ++it) {
      const double m00 = c.h00 + lambda * c.h00, m11 = c.h11 + lambda * c.h11,
                   m22 = c.h22 + lambda * c.h22;
      const double m01 = c.h01, m02 = c.h02, m12 = c.h12;  // symmetric
      const double g0 = c.g0, g1 = c.g1, g2 = c.g2;
      const double c00 = m11 * m22 - m12 * m12, c01 = m01 * m22 - m12 * m02,
                   c02 = m01 * m12 - m11 * m02;
      const double det = m00 * c00 - m01 * c01 + m02 * c02;
      if (!(fabs(det) > 0.0) || !isfinite(det)) break;
      // Cramer's rule: column c of M replaced by g
      const double d0 = (g0 * c00 - m01 * (g1 * m22 - m12 * g2) + m02 * (g1 * m12 - m11 * g2)) / det;
      const double d1 = (m00 * (g1 * m22 - m12 * g2) - g0 * c01 + m02 * (m01 * g2 - g1 * m02)) / det;
      const double d2 = (m00 * (m11 * g2 - g1 * m12) - m01 * (m01 * g2 - g1 * m02) + g0 * c02) / det;
      const double nA = A + d0, nm = m + d1, ns = s + d2;
      const FitEval nx = fit_eval(y, n, lo, delta, nA, nm, ns);
      if (isfinite(nx.sse) && nx.sse < c.sse) {
        const double rel = fmax(fmax(fabs(d0) / (fabs(A) + 1e-12), fabs(d1) / (fabs(m) + 1e-12)),
                                fabs(d2) / (fabs(s) + 1e-12));
        A = nA;
        m = nm;
        s = ns;
        c = nx;
        lambda /= 10.0;
        if (rel < 1e-10) {
          converged = true;
          break;
        }
      } else {
        lambda *= 10.0;
        if (lambda > 1e16) {
          converged = true;
          break;
        }
      }
    }
    // identifiable only with centre and width inside the window (R28)
    const double span = (double)half * delta;
    const bool ok = converged && isfinite(s) && A > 0.0 && fabs(m) <= span && fabs(s) <= span;
    ret[job.slot].echo_width_ns = ok ? (float)fabs(s) : __int_as_float(0x7fc00000);
  }
}

// Support length of each pulse's waveform (compact output): one warp per
// pulse, the same k0 / offset rules as K7 (R9).
__global__ void k_support(const WaveRec* __restrict__ rec, uint32_t N, uint64_t n, uint32_t nb,
                          uint32_t taps, uint64_t* __restrict__ len) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t p = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += warps) {
    const int2* r = reinterpret_cast<const int2*>(rec + p * N);
    int kmin = INT_MAX;
    for (uint32_t s = lane; s < N; s += 32) {
      const int k = r[s].x;
      if (k >= 0) kmin = min(kmin, k);
    }
    const int k0 = __reduce_min_sync(0xffffffffu, kmin);
    uint64_t L = 0;
    if (k0 != INT_MAX) {
      int kmax = 0;
      for (uint32_t s = lane; s < N; s += 32) {
        const int k = r[s].x;
        if (k >= 0 && k - k0 < (int)nb) kmax = max(kmax, k - k0);
      }
      kmax = __reduce_max_sync(0xffffffffu, kmax);
      L = (uint64_t)min(nb, (uint32_t)kmax + taps);
    }
    if (lane == 0) len[p] = L;
  }
}

// Ranging error (R29): every used return slot's range += sigma z,
// z from Philox stream tag 1 at (pulse, return number).  A separate pass so
// K7 keeps its register budget (fp64 log / cos / sqrt).
__global__ void k_range_noise(helios_return* __restrict__ ret, const uint8_t* __restrict__ nr,
                              uint64_t n, uint32_t R, double sd, uint64_t seed,
                              uint64_t pulse_base) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * R;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = i / R;
    const uint32_t j = (uint32_t)(i - p * R);
    if (j < nr[p]) ret[i].range_m += sd * range_noise(seed, pulse_base + p, j + 1u);
  }
}

struct Layout {
  size_t ker_d, kr_d, per_warp_d, w_off, agg_off, rec_off;
};
// wcap: bins of the per-warp W window in shared memory (main pass kWCap; the
// wide pass n_bins rounded to even, or 0 when its rows live in global memory)
__host__ __device__ inline Layout layout_for(uint32_t N, uint32_t taps, uint32_t wcap) {
  Layout L;
  L.ker_d = (taps + 1) & ~1u;
  L.kr_d = (taps + 4) & ~1u;                   // one reversed, zero-padded copy (x2)
  L.w_off = 0;
  L.agg_off = wcap;
  L.rec_off = wcap + kAggCap + 2;              // int2[N] {offset o_s, bits of A_s}
  L.per_warp_d = (L.rec_off + N + 1) & ~(size_t)1;  // even: 16-B aligned per warp
  return L;
}

// maximum of non-negative doubles over the warp: their bit patterns order
// like the values, so two 32-bit warp reductions (high words, then the low
// words of the lanes holding the highest high word) give it exactly
__device__ __forceinline__ double warp_max_nonneg(double v) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned hmax = __reduce_max_sync(0xffffffffu, hi);
  const unsigned lmax = __reduce_max_sync(0xffffffffu, hi == hmax ? lo : 0u);
  return __hiloint2double((int)hmax, (int)lmax);
}

// offset of a record relative to the window anchor k0: -1 no event, -2
// beyond maxFullwaveRange (discarded), else o_s = k_s - k0 < n_bins
__device__ __forceinline__ int rec_offset(int k, unsigned k0u, uint32_t nb) {
  const unsigned o = (unsigned)k - k0u;
  return k < 0 ? -1 : (o < nb ? (int)o : -2);
}

// K7: one warp per pulse, persistent grid-stride loop.  Reads the pulse's
// 8-B records (k_s, A_s) once, k0 = min k_s (one warp reduction), the
// per-offset amplitude sums A_o (deterministic order), the support
// W[k] = sum_o A_o p[k - o] (k < S = maxoff + L_p) in fp64, maximum, local
// maxima and returns, then the output row.
//
// Two passes share this body.  The main pass (MODE 0) keeps W in the warp's
// shared-memory window of kWCap bins; a pulse whose support exceeds it (C5:
// 0.8 % of pulses, roof edges over the ground) is appended to a list and left
// untouched.  The wide pass (launched right after on the same stream) runs
// those pulses with a whole n_bins row per warp in shared memory (MODE 1,
// fewer warps per block), or, when even one such row does not fit, in a
// per-warp global scratch row (MODE 2).  Keeping the modes apart lets the
// compiler address W as shared memory (LDS/STS, not generic loads).  R = ceil(N / 32) <= 3: records of
// the next pulse prefetched into registers (R = 0: read in the loop, any N).  FIT: the echo-width jobs (R28) are
// compiled in only where asked for (a smaller loop body for the usual case).
template <int MODE, bool FIT, int R>
__global__ void __launch_bounds__(kMaxWarps * 32, HELIOS_WAVE_MIN_BLOCKS)
    k_waveform(const WaveArgs a, double* __restrict__ gscratch) {
  constexpr bool WIDE = MODE != 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t N = a.N, nb = a.n_bins, taps = a.taps;
  const uint32_t count = WIDE ? *a.wide_count : (uint32_t)a.n_pulses;
  if (WIDE && count == 0) return;  // the usual case: nothing deferred
  const Layout L = layout_for(N, taps, MODE == 0 ? kWCap : MODE == 1 ? (nb + 1) & ~1u : 0u);
  double* ker = reinterpret_cast<double*>(smem_raw);
  double* krev = ker + L.ker_d;  // two copies of kr[m] = ker[taps - 1 - m], zero-padded
  double* base = krev + 2 * L.kr_d + (size_t)warp * L.per_warp_d;
  double* agg = base + L.agg_off;
  int2* sr = reinterpret_cast<int2*>(base + L.rec_off);  // {o_s, bits of A_s}
  const unsigned kFull = 0xffffffffu;

  for (uint32_t j = threadIdx.x; j < taps; j += blockDim.x) ker[j] = a.kernel[j];
  for (uint32_t j = threadIdx.x; j < 2 * L.kr_d; j += blockDim.x) {
    const uint32_t q = j >= L.kr_d, i = j - q * (uint32_t)L.kr_d;  // copy q holds kr[m] at 2 - q + m
    const int m = (int)i - 2 + (int)q;
    krev[j] = (m >= 0 && m < (int)taps) ? a.kernel[taps - 1 - m] : 0.0;
  }
  __syncthreads();

  const uint32_t gw = blockIdx.x * (uint32_t)nw + (uint32_t)warp;
  const uint32_t stride = gridDim.x * (uint32_t)nw;
  double* W = MODE == 2 ? gscratch + (size_t)gw * nb : base + L.w_off;

  // software pipelining (N <= 96: R = ceil(N / 32) records per lane): the
  // records of the warp's next pulse are loaded into registers while this
  // pulse is binned, so their DRAM latency is hidden (measured faster on C5
  // than a cp.async double buffer in shared memory, profiles/r02_k7_rework_ab.txt)
  constexpr int RR = R > 0 ? R : 1;
  int2 nx[RR];
  auto fetch = [&](uint32_t q) {
    const int2* rq = reinterpret_cast<const int2*>(a.rec) + (size_t)q * N;
#pragma unroll
    for (int i = 0; i < RR; ++i)
      nx[i] = (uint32_t)(lane + 32 * i) < N ? __ldcs(rq + lane + 32 * i) : make_int2(-1, 0);
  };
  if (R > 0 && gw < count) fetch(gw);

  for (uint32_t it = gw; it < count; it += stride) {  // @region prologue
    const uint32_t p = WIDE ? a.wide_list[it] : it;
    // the pulse's time is needed only by its returns: load it early
    const double tsec = (a.time_s && lane == 0) ? a.time_s[p] : 0.0;
    // records: k0 = min k_s over the events (a miss, k_s = -1, is the
    // largest unsigned value), then o_s = k_s - k0 into shared memory
    unsigned kmin = 0xFFFFFFFFu;  // @region records
    int2 c[RR];
    if constexpr (R > 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) c[i] = nx[i];
      if (it + stride < count) fetch(it + stride);
#pragma unroll
      for (int i = 0; i < R; ++i) kmin = min(kmin, (unsigned)c[i].x);
    } else {
      const int2* rq = reinterpret_cast<const int2*>(a.rec) + (size_t)p * N;
      for (uint32_t s = lane; s < N; s += 32) {
        const int2 r = __ldcs(rq + s);
        sr[s] = r;
        kmin = min(kmin, (unsigned)r.x);
      }
    }
    const unsigned k0u = __reduce_min_sync(kFull, kmin);
    const bool any = k0u != 0xFFFFFFFFu;
    int maxoff = 0;
    if constexpr (R > 0) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int o = rec_offset(c[i].x, k0u, nb);
        maxoff = max(maxoff, o);
        if ((uint32_t)(lane + 32 * i) < N) sr[lane + 32 * i] = make_int2(o, c[i].y);
      }
    } else {
      for (uint32_t s = lane; s < N; s += 32) {
        const int o = rec_offset(sr[s].x, k0u, nb);
        maxoff = max(maxoff, o);
        sr[s].x = o;
      }
    }
    maxoff = __reduce_max_sync(kFull, maxoff);
    const uint32_t S = any ? min(nb, (uint32_t)maxoff + taps) : 0u;
    __syncwarp();
    if (!WIDE && S > (uint32_t)kWCap) {
      // the wide pass bins this pulse (and writes all its outputs)
      if (lane == 0) a.wide_list[atomicAdd(a.wide_count, 1u)] = p;
      continue;
    }
    helios_return* slots = a.returns + (size_t)p * a.max_returns;
    float* row = a.waveform ? a.waveform + (size_t)p * nb : nullptr;
    // returns 0..31 are assembled in the registers of lane r and stored once
    // their count is known (one 32-B record per lane)
    const bool reg_ret = a.max_returns <= 32;
    double rr_range = 0.0;
    float rr_int = 0.0f;
    uint32_t rr_prim = 0;
    uint32_t nret = 0;
    if (any) {
      HELIOS_DASSERT(maxoff >= 0 && maxoff < (int)nb && S >= 1 && S <= nb);
      double Mlane = 0.0;  // this lane's maximum of W (grouped path: while computing W)
      bool have_max = false;
      if (maxoff < kAggCap) {
        have_max = true;
        // amplitude per offset group, in a fixed order (deterministic)  @region group_sums
        const int G = maxoff + 1;
        if (G <= 16) {
          // lane (o, c) = (lane mod G, lane / G) sums group o over subray
          // chunk c of C = floor(32 / G) (lanes >= C G idle; divisions as
          // exact reciprocal multiplies), then a fixed binary tree over the chunks
          const uint32_t C = 32u / (uint32_t)G;  // warp-uniform
          const uint32_t c = G == 1 ? (uint32_t)lane : __umulhi((uint32_t)lane, c_inv[G]);
          const int o = lane - (int)c * G;
          double acc = 0.0, acc2 = 0.0;  // two chains (subrays of even / odd rank)
          if (c < C) {
            const uint32_t s0 = __umulhi(N * c, c_inv[C]), s1 = __umulhi(N * (c + 1), c_inv[C]);
            uint32_t s = s0;
            for (; s + 1 < s1; s += 2) {
              const int2 r = sr[s], r2 = sr[s + 1];
              if (r.x == o) acc += (double)__int_as_float(r.y);
              if (r2.x == o) acc2 += (double)__int_as_float(r2.y);
            }
            if (s < s1) {
              const int2 r = sr[s];
              if (r.x == o) acc += (double)__int_as_float(r.y);
            }
            acc += acc2;
          }
          for (uint32_t st = 1; st < C; st <<= 1) {
            const double other = __shfl_down_sync(kFull, acc, st * (uint32_t)G);
            if ((c & (2 * st - 1)) == 0 && c + st < C) acc += other;
          }
          if (lane < G) agg[lane] = acc;
        } else {
          // 17..64 offsets: within each 32-subray chunk the lanes of equal
          // offset (match_any); the lowest sums its members in subray order
          // and adds the partial to its group's sum, chunk after chunk
          for (int o = lane; o < G; o += 32) agg[o] = 0.0;
          __syncwarp();
          for (uint32_t c0 = 0; c0 < N; c0 += 32) {
            const uint32_t s = c0 + lane;
            const int2 r = s < N ? sr[s] : make_int2(-1, 0);
            const unsigned peers = __match_any_sync(kFull, r.x);
            if (r.x >= 0 && (peers & ((1u << lane) - 1u)) == 0u) {
              double acc = (double)__int_as_float(r.y);
              for (unsigned b = peers & (peers - 1u); b; b &= b - 1u)
                acc += (double)__int_as_float(sr[c0 + __ffs(b) - 1].y);
              agg[r.x] += acc;
            }
            __syncwarp();
          }
        }
        __syncwarp();
        // W[k] = sum_o A_o p[k - o], two fp64 chains per bin (even / odd  @region W_grouped
        // offsets), the lane's running maximum on the way
        {
          // pairs of terms by 16-B loads: agg[o], agg[o + 1] and the reversed
          // kernel kr[m], kr[m + 1] (ker[k - o] = kr[taps - 1 - k + o]); the
          // copy of kr (shifted by one) that aligns the pair with agg's is
          // taken per bin; an odd first or last term meets a zero pad
          if (lane < 2) agg[G + lane] = 0.0;
          __syncwarp();
          for (uint32_t k = lane; k < S; k += 32) {
            const int olo = max(0, (int)k - (int)taps + 1), ohi = min(maxoff, (int)k);
            const int o0 = olo & ~1;                  // even start (agg[-1] never read)
            const int m0 = (int)taps - 1 - (int)k + o0;  // kr index of the first term (>= -1)
            // copy q = m0 mod 2 holds kr[m] at index 2 - q + m: the pairs
            // {m0 + 2t, m0 + 2t + 1} start at even indices (16-B aligned)
            const int q = m0 & 1;
            const double2* kp = reinterpret_cast<const double2*>(krev + q * L.kr_d + 2 - q + m0);
            const double2* ap = reinterpret_cast<const double2*>(agg + o0);
            double w = 0.0, w2 = 0.0;
            for (int t = 0; o0 + 2 * t <= ohi; ++t) {
              const double2 av = ap[t], kv = kp[t];
              w = fma(av.x, kv.x, w);
              w2 = fma(av.y, kv.y, w2);
            }
            w += w2;
            W[k] = w;
            Mlane = fmax(Mlane, w);
          }
        }
      } else {
        // wide footprint (offsets spread over >= kAggCap bins, e.g. a crown and  @region wide
        // the ground below it).  Groups: within each 32-subray chunk the lanes
        // with equal offsets (match_any); the lowest lane sums its members in
        // subray order; the chunk's groups are then added into W one after the
        // other in lane order (broadcast by shuffles), chunk after chunk:
        // deterministic, any number of groups.
        for (uint32_t k = lane; k < S; k += 32) W[k] = 0.0;
        // the lane's kernel taps j = lane, lane + 32 in registers (L_p <= 64)
        const bool short_ker = taps <= 64;
        const double kr0 = (uint32_t)lane < taps ? ker[lane] : 0.0;
        const double kr1 = (uint32_t)lane + 32 < taps ? ker[lane + 32] : 0.0;
        __syncwarp();
        for (uint32_t c0 = 0; c0 < N; c0 += 32) {
          const uint32_t s = c0 + lane;
          const int o = s < N ? sr[s].x : -1;
          const unsigned peers = __match_any_sync(kFull, o);
          const bool lead = o >= 0 && (peers & ((1u << lane) - 1u)) == 0u;
          double acc = 0.0;
          if (lead)
            for (unsigned b = peers; b; b &= b - 1u)
              acc += (double)__int_as_float(sr[c0 + __ffs(b) - 1].y);
          for (unsigned leads = __ballot_sync(kFull, lead); leads; leads &= leads - 1u) {
            const int src = __ffs(leads) - 1;
            const double A = __shfl_sync(kFull, acc, src);
            const uint32_t og = (uint32_t)__shfl_sync(kFull, o, src);
            if (short_ker) {
              const uint32_t k = og + lane;
              if ((uint32_t)lane < taps && k < S) W[k] = fma(A, kr0, W[k]);
              if ((uint32_t)lane + 32 < taps && k + 32 < S) W[k + 32] = fma(A, kr1, W[k + 32]);
            } else {
              for (uint32_t j = lane; j < taps; j += 32) {
                const uint32_t k = og + j;
                if (k < S) W[k] = fma(A, ker[j], W[k]);
              }
            }
            __syncwarp();
          }
        }
      }
      __syncwarp();
      // maximum (all W >= 0)  @region max
      if (!have_max)
        for (uint32_t k = lane; k < S; k += 32) Mlane = fmax(Mlane, W[k]);
      const double M = warp_max_nonneg(Mlane);
      const double thr = (double)a.thr * M;
      const int k0 = (int)k0u;
      // local maxima in time order (ballot over 32 consecutive bins)  @region peaks_attr
      for (uint32_t b0 = 0; b0 < S && nret < a.max_returns; b0 += 32) {
        const uint32_t k = b0 + lane;
        bool pk = false;
        // a block with no bin at or above the threshold holds no peak: one
        // load and one vote instead of three loads and the comparisons
        const bool inb = k >= 1 && k + 1 < nb && k < S;
        const double w = inb ? W[k] : 0.0;
        if (!__any_sync(kFull, inb && w >= thr)) continue;
        if (inb) {
          const double wl = W[k - 1], wr = (k + 1 < S) ? W[k + 1] : 0.0;
          pk = w > wl && w > wr && w >= thr;
        }
        unsigned m = __ballot_sync(kFull, pk);
        while (m && nret < a.max_returns) {
          const uint32_t kk = b0 + (__ffs(m) - 1);
          HELIOS_DASSERT(kk >= 1 && kk + 1 < nb && kk < S);
          m &= m - 1;
          // attribution (R13): largest contribution A_s p[kk - o_s], ties ->
          // lowest s: exact max over the warp, then the lowest s holding it
          double bc = 0.0;
          uint32_t bs = 0xFFFFFFFFu;
          for (uint32_t s = lane; s < N; s += 32) {
            const int2 r = sr[s];
            const int o = r.x;
            const int j = (int)kk - o;
            if (o < 0 || j < 0 || j >= (int)taps) continue;
            const double cc = (double)__int_as_float(r.y) * ker[j];
            if (bs == 0xFFFFFFFFu || cc > bc) {
              bc = cc;
              bs = s;
            }
          }
          const double cmax = warp_max_nonneg(bs == 0xFFFFFFFFu ? 0.0 : bc);
          bs = __reduce_min_sync(kFull, (bs != 0xFFFFFFFFu && bc == cmax) ? bs : 0xFFFFFFFFu);
          HELIOS_DASSERT(bs < N);  // a peak bin always has a contributor
          if (FIT) {
            // echo-width job (R28): the echo's window, fitted later by k_fit
            int lo, hi;
            echo_window(W, S, nb, (int)kk, a.fit_half, lo, hi);
            unsigned job = 0;
            if (lane == 0) job = atomicAdd(a.fit_count, 1u);
            job = __shfl_sync(kFull, job, 0);
            double* y = a.fit_y + (size_t)job * a.fit_stride;
            for (int i = lane; i <= hi - lo; i += 32)
              y[i] = (uint32_t)(lo + i) < S ? W[lo + i] : 0.0;
            if (lane == 0) {
              FitJob fj;
              fj.slot = (uint32_t)((size_t)p * a.max_returns + nret);
              fj.lo = (int16_t)(lo - (int)kk);
              fj.n = (uint16_t)(hi - lo + 1);
              fj.peak = W[kk];
              a.fit_jobs[job] = fj;
            }
          }
          const double range = 0.5 * kC *
              ((double)((long long)k0 + (long long)kk - (long long)a.jstar) + 0.5) * a.delta_ns * 1e-9;
          if (reg_ret) {
            if (lane == nret) {
              rr_range = range;
              rr_int = (float)W[kk];
              rr_prim = a.prim[(size_t)p * N + bs];
            }
          } else if (lane == 0) {
            helios_return r;
            r.range_m = range;
            r.gps_time_s = tsec;
            r.intensity = (float)W[kk];
            r.prim_id = a.prim[(size_t)p * N + bs];
            r.return_number = (uint8_t)(nret + 1);
            r.n_returns = 0;  // patched below once the count is known
            r.pad[0] = r.pad[1] = 0;
            r.echo_width_ns = __int_as_float(0x7fc00000);  // NaN until k_fit (R28)
            slots[nret] = r;
          }
          ++nret;
        }
      }
    }
    __syncwarp();
    // return slots: the used ones with their count, the unused ones zeroed  @region returns
    if (reg_ret) {
      const double t_ret = __shfl_sync(kFull, tsec, 0);
      if ((uint32_t)lane < a.max_returns) {
        uint4 w0 = make_uint4(0u, 0u, 0u, 0u), w1 = w0;
        if ((uint32_t)lane < nret) {
          // {range_m, gps_time_s} {intensity, prim_id, (number, count, 0, 0), echo width NaN}
          w0 = make_uint4((uint32_t)__double2loint(rr_range), (uint32_t)__double2hiint(rr_range),
                          (uint32_t)__double2loint(t_ret), (uint32_t)__double2hiint(t_ret));
          w1 = make_uint4(__float_as_uint(rr_int), rr_prim, (lane + 1u) | (nret << 8), 0x7fc00000u);
        }
        uint4* q = reinterpret_cast<uint4*>(slots + lane);
        q[0] = w0;
        q[1] = w1;
      }
    } else {
      for (uint32_t r = lane; r < a.max_returns; r += 32) {
        if (r < nret) {
          slots[r].n_returns = (uint8_t)nret;
        } else {
          double2* q = reinterpret_cast<double2*>(slots + r);
          q[0] = make_double2(0.0, 0.0);
          q[1] = make_double2(0.0, 0.0);
        }
      }
    }
    if (lane == 0) {
      a.first_bin[p] = any ? (int64_t)k0u : -1;
      a.n_returns[p] = (uint8_t)nret;
    }
    if (a.counters) {  // @region counters_compact
      unsigned h = 0;
      for (uint32_t s = lane; s < N; s += 32) h += (sr[s].x != -1);
      h = __reduce_add_sync(kFull, h);
      if (lane == 0) {
        atomicAdd(a.counters + 0, (unsigned long long)h);
        atomicAdd(a.counters + 1, (unsigned long long)nret);
      }
    }
    if (a.offs) {
      // compact row: W[0 .. len) at its packed offset (lossless; bins >= len are 0)
      const uint64_t o0 = a.offs[p], len = a.offs[p + 1] - o0;
      if (lane == 0 && len != (uint64_t)S) atomicOr(a.err_flag, 4u);
      if (a.compact && o0 + len <= a.capacity) {
        float* dst = a.compact + (a.compact_staged ? o0 - a.offs[0] : o0);
        for (uint32_t k = lane; k < (uint32_t)len; k += 32) dst[k] = k < S ? (float)W[k] : 0.0f;
      }
    }
    if (row) {
      // dense fp32 row: scalar head/tail, 16-byte streaming stores for the  @region row
      // aligned body (the support converted from W, then zeros)
      const uint32_t mis = (uint32_t)(((uintptr_t)row >> 2) & 3u);
      const uint32_t head = min(nb, (4u - mis) & 3u);
      if ((uint32_t)lane < head) row[lane] = (uint32_t)lane < S ? (float)W[lane] : 0.0f;
      const uint32_t nvec = (nb - head) >> 2;
      float4* body = reinterpret_cast<float4*>(row + head);
      const uint32_t qs = S > head ? min(nvec, (S - head + 3u) >> 2) : 0u;
      for (uint32_t q = lane; q < qs; q += 32) {
        const uint32_t k = head + 4 * q;
        float4 v;
        v.x = (float)W[k];
        v.y = k + 1 < S ? (float)W[k + 1] : 0.0f;
        v.z = k + 2 < S ? (float)W[k + 2] : 0.0f;
        v.w = k + 3 < S ? (float)W[k + 3] : 0.0f;
        __stcs(body + q, v);
      }
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      uint32_t q = qs + lane;
      for (; q + 96 < nvec; q += 128) {
        __stcs(body + q, z4);
        __stcs(body + q + 32, z4);
        __stcs(body + q + 64, z4);
        __stcs(body + q + 96, z4);
      }
      for (; q < nvec; q += 32) __stcs(body + q, z4);
      const uint32_t t0 = head + 4 * nvec;
      if (t0 + lane < nb) row[t0 + lane] = t0 + lane < S ? (float)W[t0 + lane] : 0.0f;
    }
    __syncwarp();
  }
}

size_t smem_for(uint32_t N, uint32_t taps, int warps, uint32_t wcap = kWCap) {
  const Layout L = layout_for(N, taps, wcap);
  return 8 * (L.ker_d + 2 * L.kr_d + (size_t)warps * L.per_warp_d);
}

}  // namespace

WavePlan plan_waveform(uint32_t n_bins, uint32_t N, uint32_t taps) {
  WavePlan pl{};
  int warps = 0;
  for (int w = kMaxWarps; w >= 1; --w)
    if (smem_for(N, taps, w) <= kSmemCap) {
      warps = w;
      break;
    }
  if (warps == 0) return pl;
  pl.warps = warps;
  pl.smem = smem_for(N, taps, warps);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* kernels[] = {
      (const void*)k_waveform<0, false, 0>, (const void*)k_waveform<0, false, 1>,
      (const void*)k_waveform<0, false, 2>, (const void*)k_waveform<0, false, 3>,
      (const void*)k_waveform<0, true, 0>,  (const void*)k_waveform<0, true, 1>,
      (const void*)k_waveform<0, true, 2>,  (const void*)k_waveform<0, true, 3>};
  for (const void* k : kernels)
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem) !=
        cudaSuccess) {
      cudaGetLastError();
      pl.warps = 0;
      return pl;
    }
  const int R = N <= 96 ? (int)((N + 31) / 32) : 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernels[R], warps * 32, pl.smem) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    pl.warps = 0;
    return pl;
  }
  pl.grid = (uint32_t)(sms * per_sm);
  // the wide pass (pulses whose support exceeds kWCap bins): a whole n_bins
  // row per warp in shared memory with as many warps per block as fit (C5:
  // 8 warps x 10.7 KB), one block per SM; else (very long windows) each warp's
  // row in a global scratch row, fewer blocks so that scratch stays within
  // kScratchCap (the pass stays correct, only its parallelism shrinks)
  const uint32_t wrow = (n_bins + 1) & ~1u;
  pl.wide_warps = 0;
  for (int w = kMaxWarps; w >= 1; --w)
    if (smem_for(N, taps, w, wrow) <= kSmemCap) {
      pl.wide_warps = w;
      break;
    }
  const void* wide[] = {(const void*)k_waveform<1, false, 0>, (const void*)k_waveform<1, true, 0>,
                        (const void*)k_waveform<2, false, 0>, (const void*)k_waveform<2, true, 0>};
  pl.wide_grid = (uint32_t)sms;
  if (pl.wide_warps > 0) {
    pl.wide_smem = smem_for(N, taps, pl.wide_warps, wrow);
    pl.scratch_bytes = 0;
  } else {
    pl.wide_warps = warps;
    pl.wide_smem = smem_for(N, taps, warps, 0);
    constexpr size_t kScratchCap = 512ull << 20;
    const size_t per_block = sizeof(double) * (size_t)warps * n_bins;
    if ((size_t)pl.wide_grid * per_block > kScratchCap)
      pl.wide_grid = (uint32_t)std::max<size_t>(1, kScratchCap / per_block);
    pl.scratch_bytes = per_block * pl.wide_grid;
  }
  for (const void* k : wide)
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.wide_smem) !=
        cudaSuccess) {
      cudaGetLastError();
      pl.warps = 0;
      return pl;
    }
  // shared-memory rows: as many blocks as fit per SM (the pass is as long as
  // its slowest warp's share of the deferred pulses)
  int per_sm_w = 1;
  if (pl.scratch_bytes == 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, wide[0], pl.wide_warps * 32,
                                                    pl.wide_smem) == cudaSuccess &&
      per_sm_w > 1)
    pl.wide_grid = (uint32_t)(sms * per_sm_w);
  cudaGetLastError();
  return pl;
}

bool waveform_fits(uint32_t n_bins, uint32_t N, uint32_t taps) {
  (void)n_bins;
  return smem_for(N, taps, 1) <= kSmemCap;
}

cudaError_t launch_support(const WaveRec* rec, uint32_t N, uint64_t n_pulses, uint32_t n_bins,
                           uint32_t taps, uint64_t* len, cudaStream_t s) {
  if (n_pulses == 0) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((n_pulses + 7) / 8, 148ull * 16);
  k_support<<<(unsigned)blocks, 256, 0, s>>>(rec, N, n_pulses, n_bins, taps, len);
  return cudaGetLastError();
}

cudaError_t launch_range_noise(const WaveArgs& a, cudaStream_t s) {
  if (a.n_pulses == 0 || !(a.noise_sd > 0.0)) return cudaSuccess;
  const uint64_t total = a.n_pulses * a.max_returns;
  const uint64_t blocks = std::min<uint64_t>((total + 255) / 256, 148ull * 8);
  k_range_noise<<<(unsigned)blocks, 256, 0, s>>>(a.returns, a.n_returns, a.n_pulses,
                                                  a.max_returns, a.noise_sd, a.seed, a.pulse_base);
  return cudaGetLastError();
}

// Packed returns: lengths (= n_returns) and the copy of the used slots.
__global__ void k_ret_len(const uint8_t* __restrict__ nr, uint64_t m, uint64_t* __restrict__ len) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x)
    len[i] = nr[i];
}

__global__ void k_pack_returns(const helios_return* __restrict__ slots,
                               const uint8_t* __restrict__ nr, uint64_t m, uint32_t R,
                               const uint64_t* __restrict__ offs, helios_return* __restrict__ dst,
                               int staged, uint64_t capacity) {
  const uint64_t base = staged ? offs[0] : 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m * R;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = i / R;
    const uint32_t j = (uint32_t)(i - p * R);
    if (j >= nr[p]) continue;
    const uint64_t g = offs[p] + j;
    if (g >= capacity) continue;
    const uint4* src = reinterpret_cast<const uint4*>(slots + i);
    uint4* out = reinterpret_cast<uint4*>(dst + (g - base));
    out[0] = src[0];
    out[1] = src[1];
  }
}

cudaError_t launch_pack_returns(const helios_return* slots, const uint8_t* nr, uint64_t m,
                                uint32_t R, uint64_t* len, uint64_t* offs, void* scan_temp,
                                size_t scan_bytes, helios_return* dst, int staged,
                                uint64_t capacity, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  const unsigned b1 = (unsigned)std::min<uint64_t>((m + 255) / 256, 148ull * 8);
  k_ret_len<<<b1, 256, 0, s>>>(nr, m, len);
  cudaError_t e = cudaGetLastError();
  // offs[1 + i] = offs[0] + sum_{j <= i} len[j] (offs[0]: carry of the previous chunks)
  if (e == cudaSuccess) e = scan_u64(len, offs + 1, m, true, scan_temp, scan_bytes, s, offs);
  if (e != cudaSuccess) return e;
  const unsigned b2 = (unsigned)std::min<uint64_t>((m * R + 255) / 256, 148ull * 16);
  k_pack_returns<<<b2, 256, 0, s>>>(slots, nr, m, R, offs, dst, staged, capacity);
  return cudaGetLastError();
}

cudaError_t launch_waveform(const WaveArgs& a, const WavePlan& pl, double* scratch,
                            cudaStream_t s) {
  if (a.n_pulses == 0) return cudaSuccess;
  if (pl.warps == 0 || !a.wide_list || !a.wide_count) return cudaErrorInvalidValue;
  uint64_t want = (a.n_pulses + pl.warps - 1) / pl.warps;
  uint64_t grid = pl.grid;
  if (pl.grid_cap && pl.grid_cap < grid) grid = pl.grid_cap;
  if (want < grid) grid = want;
  cudaError_t e = cudaMemsetAsync(a.wide_count, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  const unsigned g = (unsigned)grid, t = (unsigned)pl.warps * 32;
  const int R = a.N <= 96 ? (int)((a.N + 31) / 32) : 0;
  switch (R + (a.fit ? 4 : 0)) {
    case 1: k_waveform<0, false, 1><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 2: k_waveform<0, false, 2><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 3: k_waveform<0, false, 3><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 4: k_waveform<0, true, 0><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 5: k_waveform<0, true, 1><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 6: k_waveform<0, true, 2><<<g, t, pl.smem, s>>>(a, scratch); break;
    case 7: k_waveform<0, true, 3><<<g, t, pl.smem, s>>>(a, scratch); break;
    default: k_waveform<0, false, 0><<<g, t, pl.smem, s>>>(a, scratch); break;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // the pulses the main pass deferred (support > kWCap bins), same stream
  const unsigned gw = (unsigned)std::min<uint64_t>(pl.wide_grid, want);
  const unsigned tw = (unsigned)pl.wide_warps * 32;
  if (pl.scratch_bytes == 0) {
    if (a.fit)
      k_waveform<1, true, 0><<<gw, tw, pl.wide_smem, s>>>(a, scratch);
    else
      k_waveform<1, false, 0><<<gw, tw, pl.wide_smem, s>>>(a, scratch);
  } else {
    if (a.fit)
      k_waveform<2, true, 0><<<gw, tw, pl.wide_smem, s>>>(a, scratch);
    else
      k_waveform<2, false, 0><<<gw, tw, pl.wide_smem, s>>>(a, scratch);
  }
  return cudaGetLastError();
}

cudaError_t launch_fit(const WaveArgs& a, cudaStream_t s) {
  if (a.n_pulses == 0 || !a.fit) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t jobs_max = a.n_pulses * a.max_returns;
  const uint64_t fb = std::min<uint64_t>((jobs_max + 63) / 64, (uint64_t)sms * 32);
  k_fit<<<(unsigned)fb, 64, 0, s>>>(a.fit_jobs, a.fit_y, a.fit_stride, a.fit_count, a.fit_half,
                                    a.delta_ns, a.fit_s0, a.returns);
  return cudaGetLastError();
}

}  // namespace helios
