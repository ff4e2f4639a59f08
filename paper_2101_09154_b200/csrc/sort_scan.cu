// sort_scan.cu -- the build's and the runtime's data-parallel primitives,
// hand-written for sm_100a (no CUB on the build or hot path):
//
//   * inclusive / exclusive prefix sums of u32 / u64 arrays: reduce-then-scan
//     over 2048-element tiles (tile sums -> one-block scan of the tile sums ->
//     tile scans seeded with their offset, plus an optional device-resident
//     seed: the carry of the previous chunks of a call).  Integer sums: exact, so the
//     result does not depend on the tiling.
//   * LSD radix sort of (u64 key, u32 value) pairs, 8 bits per pass (the
//     63-bit Morton codes of helios_build_accel, K2 of DESIGN.md s.7): per
//     pass a digit histogram per tile (stored digit-major, so ONE exclusive
//     scan of the [256][tiles] table gives every (digit, tile) its global
//     offset), then a stable scatter: within a tile, keys are ranked round by
//     round (32 consecutive keys per warp round, peers of a digit found with
//     __match_any_sync, per-warp digit counters in shared memory), warps are
//     ordered by a per-digit prefix over the block's warps.  Every pass is
//     stable, so the sort is stable: equal keys keep their input order (the
//     BVH build is deterministic and equals a stable sort of the codes).
//
// Exposed through include/helios_util.h for the tests (cross-checked there
// against numpy's stable argsort and cumsum).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "internal.cuh"

namespace helios {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// exclusive scan of one value per thread over the block (kScanThreads);
// returns the exclusive prefix, *total = the block sum
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T wsum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < kScanThreads / 32 ? wsum[lane] : T(0);
    x = warp_incl_scan(x);
    if (lane < kScanThreads / 32) wsum[lane] = x;
  }
  __syncthreads();
  const T before = w > 0 ? wsum[w - 1] : T(0);
  *total = wsum[kScanThreads / 32 - 1];
  __syncthreads();  // wsum reusable by the next call
  return before + inc - v;
}

// phase A: sum of every tile
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sum(const T* __restrict__ in, uint64_t n,
                                                          T* __restrict__ part) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kScanThreads + threadIdx.x;  // coalesced
    if (k < n) s += in[k];
  }
  T tot;
  block_excl_scan(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// phase B: exclusive scan of the tile sums in one block (chunks of
// kScanThreads x kScanItems with a running carry)
template <class T>
__global__ void __launch_bounds__(kScanThreads) k_scan_parts(T* __restrict__ part, uint64_t m) {
  T carry = 0;
  for (uint64_t c = 0; c < m; c += kScanTile) {
    T v[kScanItems];
    T s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const uint64_t k = c + (uint64_t)threadIdx.x * kScanItems + i;
      v[i] = k < m ? part[k] : T(0);
      s += v[i];
    }
    T tot;
    T run = block_excl_scan(s, &tot) + carry;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const uint64_t k = c + (uint64_t)threadIdx.x * kScanItems + i;
      if (k < m) part[k] = run;
      run += v[i];
    }
    carry += tot;
  }
}

// phase C: scan of every tile seeded with its offset (inclusive or exclusive)
template <class T, bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* __restrict__ in, uint64_t n,
                                                           const T* __restrict__ part,
                                                           const T* __restrict__ seed,
                                                           T* __restrict__ out) {
  __shared__ T tile[kScanTile];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  // coalesced load, then each thread scans kScanItems consecutive elements
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kScanThreads + threadIdx.x;
    tile[i * kScanThreads + threadIdx.x] = k < n ? in[k] : T(0);
  }
  __syncthreads();
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = tile[threadIdx.x * kScanItems + i];
    s += v[i];
  }
  T tot;
  T run = block_excl_scan(s, &tot) + part[blockIdx.x] + (seed ? *seed : T(0));
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (INCLUSIVE) run += v[i];
    tile[threadIdx.x * kScanItems + i] = run;
    if (!INCLUSIVE) run += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t k = base + (uint64_t)i * kScanThreads + threadIdx.x;
    if (k < n) out[k] = tile[i * kScanThreads + threadIdx.x];
  }
}

template <class T>
cudaError_t scan_impl(const T* in, T* out, uint64_t n, bool inclusive, void* temp,
                      size_t temp_bytes, cudaStream_t s, const T* seed = nullptr) {
  if (n == 0) return cudaSuccess;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (temp_bytes < tiles * sizeof(T) || tiles > 0x7FFFFFFFull) return cudaErrorInvalidValue;
  T* part = static_cast<T*>(temp);
  k_tile_sum<T><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, part);
  k_scan_parts<T><<<1, kScanThreads, 0, s>>>(part, tiles);
  if (inclusive)
    k_tile_scan<T, true><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, part, seed, out);
  else
    k_tile_scan<T, false><<<(unsigned)tiles, kScanThreads, 0, s>>>(in, n, part, seed, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- radix sort
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortRounds = 8;                       // 32-key rounds per warp
constexpr int kSortWarpKeys = 32 * kSortRounds;      // 256
constexpr int kSortTile = kSortWarps * kSortWarpKeys;  // 2048
constexpr int kRadix = 256;

// digit histogram of every tile, digit-major: hist[d * tiles + tile]
__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const uint64_t* __restrict__ keys,
                                                            uint64_t n, int shift, uint32_t dmask,
                                                            uint32_t* __restrict__ hist,
                                                            uint32_t tiles) {
  __shared__ uint32_t h[kRadix];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
#pragma unroll
  for (int i = 0; i < kSortTile / kSortThreads; ++i) {
    const uint64_t k = base + (uint64_t)i * kSortThreads + threadIdx.x;
    if (k < n) atomicAdd(&h[(uint32_t)(keys[k] >> shift) & dmask], 1u);
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

// stable scatter of one tile: key j of the tile (j = warp * 256 + round * 32
// + lane) goes to offs[d * tiles + tile] + (keys of digit d in earlier warps
// of the tile) + (keys of digit d earlier in this warp)
__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(
    const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t n, int shift,
    uint32_t dmask, const uint32_t* __restrict__ offs, uint32_t tiles, uint64_t* __restrict__ kout,
    uint32_t* __restrict__ vout) {
  __shared__ uint32_t cnt[kSortWarps][kRadix];  // per-warp digit counts -> warp offsets
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kSortWarps * kRadix; i += kSortThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kSortTile + (uint64_t)w * kSortWarpKeys;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t key[kSortRounds];
  uint32_t val[kSortRounds], rank[kSortRounds];
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t k = base + (uint64_t)r * 32 + lane;
    const bool in = k < n;
    key[r] = in ? kin[k] : 0ull;
    val[r] = in ? vin[k] : 0u;
    const uint32_t d = in ? (uint32_t)(key[r] >> shift) & dmask : 0x100u;  // 0x100: no key
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    // only this warp's lanes touch cnt[w][*]: read, then the group's highest
    // lane adds the group size (after every lane has read)
    const uint32_t before = d < kRadix ? cnt[w][d] : 0u;
    rank[r] = before + __popc(peers & lt);
    __syncwarp();
    if (d < kRadix && (peers >> lane) == 1u) cnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over the warps (thread = digit)
  {
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < kSortWarps; ++q) {
      const uint32_t c = cnt[q][d];
      cnt[q][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortRounds; ++r) {
    const uint64_t k = base + (uint64_t)r * 32 + lane;
    if (k >= n) continue;
    const uint32_t d = (uint32_t)(key[r] >> shift) & dmask;
    const uint64_t dst = (uint64_t)offs[(uint64_t)d * tiles + blockIdx.x] + cnt[w][d] + rank[r];
    kout[dst] = key[r];
    vout[dst] = val[r];
  }
}

}  // namespace

size_t scan_temp_bytes(uint64_t n, size_t elem) {
  return std::max<size_t>(256, ((n + kScanTile - 1) / kScanTile) * elem);
}

cudaError_t scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, bool inclusive, void* temp,
                     size_t temp_bytes, cudaStream_t s, const uint64_t* seed) {
  return scan_impl<unsigned long long>(reinterpret_cast<const unsigned long long*>(in),
                                       reinterpret_cast<unsigned long long*>(out), n, inclusive,
                                       temp, temp_bytes, s,
                                       reinterpret_cast<const unsigned long long*>(seed));
}

cudaError_t scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, bool inclusive, void* temp,
                     size_t temp_bytes, cudaStream_t s) {
  return scan_impl<uint32_t>(in, out, n, inclusive, temp, temp_bytes, s);
}

size_t sort_temp_bytes(uint64_t n) {
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
  const uint64_t h = tiles * kRadix;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  // ping-pong keys + values, the digit table, its scan temp
  return al(8 * n) + al(4 * n) + al(4 * h) + al(scan_temp_bytes(h, 4));
}

cudaError_t sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int bits, void* temp,
                           size_t temp_bytes, cudaStream_t s) {
  if (n <= 1 || bits <= 0) return cudaSuccess;
  if (n >= (1ull << 32) || bits > 64 || temp_bytes < sort_temp_bytes(n))
    return cudaErrorInvalidValue;
  const uint64_t tiles = (n + kSortTile - 1) / kSortTile;
  const uint64_t h = tiles * kRadix;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  char* t = static_cast<char*>(temp);
  uint64_t* k2 = reinterpret_cast<uint64_t*>(t);
  uint32_t* v2 = reinterpret_cast<uint32_t*>(t + al(8 * n));
  uint32_t* hist = reinterpret_cast<uint32_t*>(t + al(8 * n) + al(4 * n));
  void* stemp = t + al(8 * n) + al(4 * n) + al(4 * h);
  const size_t sbytes = al(scan_temp_bytes(h, 4));
  uint64_t* ka = keys;
  uint32_t* va = vals;
  uint64_t* kb = k2;
  uint32_t* vb = v2;
  const int passes = (bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    // the last pass sees only the key bits below `bits`
    const uint32_t dmask = bits - shift >= 8 ? 0xFFu : (1u << (bits - shift)) - 1u;
    k_digit_hist<<<(unsigned)tiles, kSortThreads, 0, s>>>(ka, n, shift, dmask, hist,
                                                          (uint32_t)tiles);
    cudaError_t e = scan_u32(hist, hist, h, false, stemp, sbytes, s);
    if (e != cudaSuccess) return e;
    k_digit_scatter<<<(unsigned)tiles, kSortThreads, 0, s>>>(ka, va, n, shift, dmask, hist,
                                                              (uint32_t)tiles, kb, vb);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  // an odd number of passes leaves the result in the temp buffers
  if (ka != keys) {
    cudaMemcpyAsync(keys, ka, 8 * n, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(vals, va, 4 * n, cudaMemcpyDeviceToDevice, s);
  }
  return cudaGetLastError();
}

}  // namespace helios

// ---- utility ABI (include/helios_util.h): the same primitives on caller buffers
extern "C" {

int helios_util_sort_pairs_u64(uint64_t* d_keys, uint32_t* d_vals, uint64_t n, int key_bits,
                               void* stream) {
  if (n == 0) return 0;
  if (!d_keys || !d_vals || key_bits < 1 || key_bits > 64 || n >= (1ull << 32)) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  void* temp = nullptr;
  const size_t tb = helios::sort_temp_bytes(n);
  if (helios::dev_alloc(&temp, tb, s) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  cudaError_t e = helios::sort_pairs_u64(d_keys, d_vals, n, key_bits, temp, tb, s);
  cudaFreeAsync(temp, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 3;
  }
  return 0;
}

int helios_util_scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t n, int inclusive,
                         void* stream) {
  if (n == 0) return 0;
  if (!d_in || !d_out) return 1;
  const cudaStream_t s = (cudaStream_t)stream;
  void* temp = nullptr;
  const size_t tb = helios::scan_temp_bytes(n, 8);
  if (helios::dev_alloc(&temp, tb, s) != cudaSuccess) {
    cudaGetLastError();
    return 2;
  }
  cudaError_t e = helios::scan_u64(d_in, d_out, n, inclusive != 0, temp, tb, s);
  cudaFreeAsync(temp, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 3;
  }
  return 0;
}

}  // extern "C"
