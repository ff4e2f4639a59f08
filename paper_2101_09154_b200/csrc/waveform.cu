// waveform.cu -- K7: full-waveform binning + local-maximum peaks -> returns.
//
// One warp per pulse (grid-stride).  The pulse's subray records (16 B each,
// written by K6) are read once; the waveform is accumulated in shared memory
// in fp64 ("the recorded power for each bin is taken as the sum of the
// subray's waveforms, shifted according to the different ranges"), strictly
// in subray order -- no atomics, so the sum is deterministic and its
// decisions (max, local maxima, threshold) are taken in the same precision as
// the oracle's.  The dense row is stored as fp32.
//
//   k_s  = floor(2 R_s / c / Delta)                  (R8, R9; same fp64 ops as the oracle)
//   k0   = min_s k_s                                  (window anchor, R9)
//   W[k] = sum_s A_s p[k - (k_s - k0)],  p[j] = f((j + 1/2) Delta / tau),
//          f(x) = x^2 e^-x  (Eq. 3),  j < L_p = ceil(20 tau / Delta)
//   peak at k in [1, n_bins-2]: W[k] > W[k-1], W[k] > W[k+1], W[k] >= thr max W
//   (P:215 local-maximum filter; R11), earliest max_returns kept,
//   range (c/2)(k0 + k - j* + 1/2) Delta (R12), prim = argmax_s contribution (R13).
#include <math.h>

#include "internal.cuh"

namespace helios {
namespace {

constexpr int kMaxWarps = 8;
constexpr size_t kSmemCap = 200 * 1024;

__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}
__device__ __forceinline__ int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(kMaxWarps * 32) k_waveform(const WaveArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t N = a.N, nb = a.n_bins, taps = a.taps;
  // smem: kernel[taps] | per warp: W[nb] (double), off[N] (int), amp[N] (float)
  double* ker = reinterpret_cast<double*>(smem_raw);
  const size_t ker_d = (taps + 1) & ~1u;
  const size_t per_warp_d = nb + ((N + 1) / 2) + ((N + 1) / 2);
  double* W = ker + ker_d + warp * per_warp_d;
  int* off = reinterpret_cast<int*>(W + nb);
  float* amp = reinterpret_cast<float*>(W + nb + (N + 1) / 2);

  for (uint32_t j = threadIdx.x; j < taps; j += blockDim.x) ker[j] = a.kernel[j];
  __syncthreads();

  for (uint64_t p = (uint64_t)blockIdx.x * nw + warp; p < a.n_pulses;
       p += (uint64_t)gridDim.x * nw) {
    const helios_subray_hit* rec = a.rec + p * N;
    // pass 1: bins k_s (fp64, the oracle's operation order) and k0
    long long kmin = LLONG_MAX;
    for (uint32_t s = lane; s < N; s += 32) {
      const helios_subray_hit r = rec[s];
      long long k = -1;
      if (r.prim_id != 0xFFFFFFFFu) {
        k = (long long)floor(2.0 * r.range_m / kC / (a.delta_ns * 1e-9));
        kmin = k < kmin ? k : kmin;
      }
      off[s] = (int)(k < 0 ? -1 : k);  // absolute bin for now (fits: R < 3e8 m)
      amp[s] = r.amplitude;
    }
    __syncwarp();
    const long long k0 = warp_min_ll(kmin);
    uint8_t nret = 0;
    helios_return* slots = a.returns + p * a.max_returns;
    float* row = a.waveform ? a.waveform + p * (uint64_t)nb : nullptr;
    if (k0 == LLONG_MAX) {  // no hit (R23): empty row, no returns
      if (lane == 0) {
        a.first_bin[p] = -1;
        a.n_returns[p] = 0;
      }
      for (uint32_t q = lane; q < a.max_returns * 4u; q += 32)
        reinterpret_cast<double*>(slots)[q] = 0.0;
      if (row)
        for (uint32_t k = lane; k < nb; k += 32) row[k] = 0.0f;
      continue;
    }
    // offsets relative to the window; support length S
    int maxoff = 0;
    for (uint32_t s = lane; s < N; s += 32) {
      int o = off[s];
      if (o >= 0) {
        o = (int)((long long)o - k0);
        if (o >= (int)nb) o = -2;  // beyond maxFullwaveRange: discarded
        else maxoff = max(maxoff, o);
        off[s] = o;
      }
    }
    maxoff = warp_max_i(maxoff);
    const uint32_t S = min(nb, (uint32_t)maxoff + taps);
    for (uint32_t k = lane; k < S; k += 32) W[k] = 0.0;
    __syncwarp();
    // accumulate in subray order (deterministic)
    for (uint32_t s = 0; s < N; ++s) {
      const int o = off[s];
      if (o < 0) continue;
      const double A = (double)amp[s];
      for (uint32_t j = lane; j < taps; j += 32) {
        const uint32_t k = (uint32_t)o + j;
        if (k < S) W[k] += A * ker[j];
      }
      __syncwarp();
    }
    // maximum
    double M = 0.0;
    for (uint32_t k = lane; k < S; k += 32) M = fmax(M, W[k]);
    M = warp_max_d(M);
    const double thr = (double)a.thr * M;
    // local maxima in time order (ballot over 32 consecutive bins)
    for (uint32_t base = 0; base < S && nret < a.max_returns; base += 32) {
      const uint32_t k = base + lane;
      bool pk = false;
      if (k >= 1 && k + 1 < nb && k < S) {
        const double w = W[k], wl = W[k - 1], wr = (k + 1 < S) ? W[k + 1] : 0.0;
        pk = w > wl && w > wr && w >= thr;
      }
      unsigned m = __ballot_sync(0xffffffffu, pk);
      while (m && nret < a.max_returns) {
        const uint32_t kk = base + (__ffs(m) - 1);
        m &= m - 1;
        // attribution (R13): largest contribution A_s p[kk - o_s], ties -> lowest s
        double bc = -1.0;
        uint32_t bs = 0xFFFFFFFFu;
        for (uint32_t s = lane; s < N; s += 32) {
          const int o = off[s];
          if (o < 0) continue;
          const int j = (int)kk - o;
          if (j < 0 || j >= (int)taps) continue;
          const double c = (double)amp[s] * ker[j];
          if (c > bc) {
            bc = c;
            bs = s;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double c2 = __shfl_xor_sync(0xffffffffu, bc, o);
          const uint32_t s2 = __shfl_xor_sync(0xffffffffu, bs, o);
          if (c2 > bc || (c2 == bc && s2 < bs)) {
            bc = c2;
            bs = s2;
          }
        }
        if (lane == 0) {
          helios_return r;
          r.range_m = 0.5 * kC * ((double)(k0 + (long long)kk - (long long)a.jstar) + 0.5) *
                      a.delta_ns * 1e-9;
          r.gps_time_s = a.time_s ? a.time_s[p] : 0.0;
          r.intensity = (float)W[kk];
          r.prim_id = rec[bs].prim_id;
          r.return_number = (uint8_t)(nret + 1);
          r.n_returns = 0;  // patched below once the count is known
          for (int q = 0; q < 6; ++q) r.pad[q] = 0;
          slots[nret] = r;
        }
        ++nret;
      }
    }
    __syncwarp();
    // patch n_returns into the slots, zero the unused ones
    for (uint32_t r = lane; r < a.max_returns; r += 32) {
      if (r < nret) {
        slots[r].n_returns = nret;
      } else {
        double* q = reinterpret_cast<double*>(slots + r);
        q[0] = 0.0;
        q[1] = 0.0;
        q[2] = 0.0;
        q[3] = 0.0;
      }
    }
    if (lane == 0) {
      a.first_bin[p] = k0;
      a.n_returns[p] = nret;
      if (a.counters) atomicAdd(a.counters + 1, (unsigned long long)nret);
    }
    if (a.counters) {
      unsigned h = 0;
      for (uint32_t s = lane; s < N; s += 32) h += (rec[s].prim_id != 0xFFFFFFFFu);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
      if (lane == 0) atomicAdd(a.counters + 0, (unsigned long long)h);
    }
    if (row)
      for (uint32_t k = lane; k < nb; k += 32) row[k] = k < S ? (float)W[k] : 0.0f;
    __syncwarp();
  }
}

}  // namespace

static size_t smem_for(uint32_t n_bins, uint32_t N, uint32_t taps, int warps) {
  const size_t ker_d = (taps + 1) & ~1u;
  const size_t per_warp_d = n_bins + ((N + 1) / 2) + ((N + 1) / 2);
  return 8 * (ker_d + (size_t)warps * per_warp_d);
}

// warps per block that fit the shared-memory budget (0 = does not fit)
int waveform_warps(uint32_t n_bins, uint32_t N, uint32_t taps) {
  for (int w = kMaxWarps; w >= 1; --w)
    if (smem_for(n_bins, N, taps, w) <= kSmemCap) return w;
  return 0;
}

cudaError_t launch_waveform(const WaveArgs& a, cudaStream_t s) {
  if (a.n_pulses == 0) return cudaSuccess;
  const int warps = waveform_warps(a.n_bins, a.N, a.taps);
  if (warps == 0) return cudaErrorInvalidValue;
  const size_t smem = smem_for(a.n_bins, a.N, a.taps, warps);
  cudaError_t e = cudaFuncSetAttribute(k_waveform, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_waveform, warps * 32, smem);
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t want = (a.n_pulses + warps - 1) / warps;
  uint64_t grid = (uint64_t)sms * per_sm;
  if (want < grid) grid = want;
  k_waveform<<<(unsigned)grid, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace helios
