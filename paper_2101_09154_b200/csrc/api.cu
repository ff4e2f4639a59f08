// api.cu -- the C ABI of libhelios.so (include/helios.h) and its host runtime:
// argument validation, scene ownership, the beam-pattern tables, scratch
// management (a library-private stream-ordered memory pool), host<->device
// staging, the chunk pipeline over one or more pulse batches, and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <list>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace helios;

// ---- library-private device memory pool (one per device): every library
// allocation is stream-ordered from it, and its release threshold is raised
// so freed blocks stay mapped across synchronisations -- without touching the
// device's default pool, which other libraries in the process share.
namespace {
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};
}  // namespace

namespace helios {
std::atomic<uint64_t> g_fault_alloc{0};  // helios_tuning.fault_alloc_bytes (0 = off)
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t s) {
  const uint64_t lim = g_fault_alloc.load(std::memory_order_relaxed);
  if (lim && bytes > lim) {
    *p = nullptr;
    return cudaErrorMemoryAllocation;  // injected (tests of the out-of-memory paths)
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (!g_pool[dev]) {
      cudaMemPoolProps pp{};
      pp.allocType = cudaMemAllocationTypePinned;
      pp.handleTypes = cudaMemHandleTypeNone;
      pp.location.type = cudaMemLocationTypeDevice;
      pp.location.id = dev;
      e = cudaMemPoolCreate(&g_pool[dev], &pp);
      if (e != cudaSuccess) return e;
      uint64_t keep = std::numeric_limits<uint64_t>::max();
      cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = g_pool[dev];
  }
  return cudaMallocFromPoolAsync(p, bytes ? bytes : 256, pool, s);
}
}  // namespace helios

// ---- process-wide tuning switches (helios_set_tuning), seeded once from the
// environment at first use; every call takes a snapshot when it starts
namespace {
std::mutex g_tune_mu;
bool g_tune_init = false;
helios_tuning g_tune{};

helios_tuning tuning_defaults() {
  helios_tuning t{};
  t.beam_prepass = -1;
  t.builder = 0;
  t.lane_order = 1;
  t.pad_lanes = -1;
  t.serialize = 0;
  t.trace_spans = 0;
  t.chunk_pulses = 0;
  t.fault_alloc_bytes = 0;
  return t;
}

helios_tuning tuning_snapshot() {
  std::lock_guard<std::mutex> g(g_tune_mu);
  if (!g_tune_init) {
    g_tune = tuning_defaults();
    auto env = [](const char* name, int64_t* v) {
      const char* s = getenv(name);
      if (s && *s) *v = atoll(s);
      return s != nullptr;
    };
    int64_t v;
    if (env("HELIOS_BEAM", &v)) g_tune.beam_prepass = (int32_t)v;
    if (const char* b = getenv("HELIOS_BUILDER")) g_tune.builder = strcmp(b, "lbvh") == 0 ? 1 : 0;
    if (env("HELIOS_LANE_ORDER", &v)) g_tune.lane_order = (int32_t)v;
    if (env("HELIOS_PAD_LANES", &v)) g_tune.pad_lanes = (int32_t)v;
    if (env("HELIOS_SERIALIZE", &v)) g_tune.serialize = (int32_t)v;
    if (env("HELIOS_TRACE_SPANS", &v)) g_tune.trace_spans = (int32_t)v;
    if (env("HELIOS_CHUNK_PULSES", &v)) g_tune.chunk_pulses = (uint64_t)std::max<int64_t>(0, v);
    g_tune_init = true;
  }
  return g_tune;
}
}  // namespace

struct helios_scene_s {
  uint32_t n_tris = 0;
  float* d_xyz = nullptr;   // original order (build input)
  float* d_refl = nullptr;
  float* d_pad = nullptr;
  uint8_t* d_bricks = nullptr;  // 4^3-brick occupancy of the grid
  uint32_t nbx = 0, nby = 0, nbz = 0;
  uint32_t nx = 0, ny = 0, nz = 0;
  double origin[3] = {0, 0, 0};
  double vs = 0;
  float* d_lut = nullptr;
  uint32_t n_lut = 0;
  uint32_t voxel_mode = HELIOS_VOXEL_TRANSMISSIVE;  // R31
  double voxel_refl = 0.5, pad_max = 1.0, scale_alpha = 1.0;
  uint32_t scale_shift = 0;
  bool built = false;
  BuildResult bvh{};
  int device = 0;

  // Scratch cache: one device buffer (+ the call's internal streams and a
  // pinned mirror) per caller stream, grown on demand and reused by later
  // calls on that stream.  Idle entries beyond kMaxIdle are evicted, least
  // recently used first; destroy frees the rest.  Only streams the library
  // created are ever synchronised here (never a caller's stream, which may
  // no longer exist).
  struct Slot {
    cudaStream_t key;  // caller stream (not owned, never used after the call)
    char* ptr;
    size_t bytes;
    bool busy;
    uint64_t last_use;
    cudaStream_t copy_in, copy_out, wave, fit, trace2;  // owned, created lazily
    uint64_t* pinned;  // 4 kSlots words: per chunk slot (first, last) packed offsets
  };
  static constexpr int kMaxIdle = 4;
  std::mutex mu;
  std::list<Slot> slots;  // stable addresses: a call keeps its Slot* while others acquire
  uint64_t use_clock = 0;

  static void release_slot(Slot& sl) {
    cudaStream_t own[5] = {sl.copy_in, sl.copy_out, sl.wave, sl.fit, sl.trace2};
    for (cudaStream_t x : own)
      if (x) cudaStreamSynchronize(x);
    if (sl.ptr) {
      // freed on an owned stream (or synchronously): the last use of the
      // buffer was ordered before the end of the call that used it
      if (sl.wave) {
        cudaFreeAsync(sl.ptr, sl.wave);
        cudaStreamSynchronize(sl.wave);
      } else {
        cudaFree(sl.ptr);
      }
    }
    for (cudaStream_t x : own)
      if (x) cudaStreamDestroy(x);
    if (sl.pinned) cudaFreeHost(sl.pinned);
    cudaGetLastError();
  }

  cudaError_t acquire(cudaStream_t s, size_t bytes, Slot** out) {
    std::lock_guard<std::mutex> g(mu);
    Slot* use = nullptr;
    for (Slot& sl : slots)
      if (sl.key == s && !sl.busy) {
        use = &sl;
        break;
      }
    if (!use) {
      // evict the least recently used idle entries first (keeps the cache bounded)
      int idle = 0;
      for (const Slot& sl : slots) idle += !sl.busy;
      while (idle >= kMaxIdle) {
        auto lru = slots.end();
        for (auto it = slots.begin(); it != slots.end(); ++it)
          if (!it->busy && (lru == slots.end() || it->last_use < lru->last_use)) lru = it;
        release_slot(*lru);
        slots.erase(lru);
        --idle;
      }
      slots.push_back(Slot{s, nullptr, 0, false, 0, nullptr, nullptr, nullptr, nullptr, nullptr,
                           nullptr});
      use = &slots.back();
    }
    if (use->bytes < bytes) {
      if (use->ptr) cudaFreeAsync(use->ptr, s);
      use->ptr = nullptr;
      use->bytes = 0;
      cudaError_t e = dev_alloc((void**)&use->ptr, bytes, s);
      if (e != cudaSuccess) return e;
      use->bytes = bytes;
    }
    auto make = [](cudaStream_t* st, int prio_hi) -> cudaError_t {
      if (*st) return cudaSuccess;
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      return cudaStreamCreateWithPriority(st, cudaStreamNonBlocking, prio_hi ? hi : lo);
    };
    cudaError_t e;
    // K7 (and the scans, fits and copies it feeds) at high priority: its
    // blocks are scheduled ahead of the queued blocks of the next chunks' K6
    // grids, so a chunk's outputs do not wait for them to drain
    if ((e = make(&use->wave, 1)) != cudaSuccess) return e;
    if ((e = make(&use->copy_in, 0)) != cudaSuccess) return e;
    if ((e = make(&use->copy_out, 0)) != cudaSuccess) return e;
    if ((e = make(&use->fit, 0)) != cudaSuccess) return e;
    if ((e = make(&use->trace2, 0)) != cudaSuccess) return e;
    if (!use->pinned) {
      e = cudaMallocHost((void**)&use->pinned, 4 * kSlots * sizeof(uint64_t));
      if (e != cudaSuccess) return e;
    }
    use->busy = true;
    use->last_use = ++use_clock;
    *out = use;
    return cudaSuccess;
  }
  void release(Slot* sl) {
    std::lock_guard<std::mutex> g(mu);
    sl->busy = false;
  }
  void free_slots() {
    std::lock_guard<std::mutex> g(mu);
    for (Slot& sl : slots) release_slot(sl);
    slots.clear();
  }
};

namespace {

thread_local std::string g_err;

double now_ms() {
  return 1e3 * (double)std::chrono::duration_cast<std::chrono::nanoseconds>(
                   std::chrono::steady_clock::now().time_since_epoch()).count() * 1e-9;
}

helios_status fail(helios_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

helios_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation)
    return fail(HELIOS_ERR_OUT_OF_MEMORY, "%s: out of device memory", what);
  return fail(HELIOS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool device_accessible(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// page-locked host memory (cudaMallocHost / cudaHostRegister): an async copy
// into it does not block the host
bool pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// ---- subray pattern (P:199 / R1): paper rule floor(2 pi i), or hexagonal 6i
struct Pattern {
  int q = -1;
  bool hex = false;
};
Pattern resolve_pattern(uint32_t count) {
  Pattern pt;
  uint64_t total = 1;
  for (int q = 0; q <= 64 && total <= count; ++q) {
    if (q > 0) total += (uint64_t)std::floor(2.0 * kPi * (double)q);
    if (total == count) {
      pt.q = q;
      return pt;
    }
  }
  for (int q = 0; q <= 64; ++q) {
    if (1ull + 3ull * (uint64_t)q * (uint64_t)(q + 1) == count) {
      pt.q = q;
      pt.hex = true;
      return pt;
    }
  }
  return pt;
}

std::vector<SubrayConst> subray_table(uint32_t count, double beta, Pattern pt) {
  std::vector<SubrayConst> t;
  t.reserve(count);
  const double tb = std::tan(beta);
  auto push = [&](double theta, double phi) {
    SubrayConst c{};
    const double st = std::sin(theta);
    c.cos_t = std::cos(theta);
    c.sin_t = st;
    c.cos_p = std::cos(phi);
    c.sin_p = std::sin(phi);
    c.w_far = theta == 0.0 ? 1.0 : std::exp(-2.0 * st * st / (tb * tb));
    t.push_back(c);
  };
  push(0.0, 0.0);  // central subray
  for (int i = 1; i <= pt.q; ++i) {
    const int n = pt.hex ? 6 * i : (int)std::floor(2.0 * kPi * (double)i);
    const double theta = (double)i / (double)pt.q * beta;  // R2
    for (int j = 0; j < n; ++j) push(theta, 2.0 * kPi * (double)j / (double)n);  // R4
  }
  for (uint32_t s = 0; s < (uint32_t)t.size(); ++s) t[s].index = s;
  return t;
}

// Lane order of the subrays in K6 (a permutation of the table; each entry
// keeps its index s, which alone defines the subray: directions, Philox
// counters and output slots are unchanged).  R4's order runs ring by ring, so
// any 32 consecutive subrays of a 91-subray pulse span a whole annulus and
// their warp walks every leaf of the footprint.  Ordered along a Hilbert curve
// over the footprint disc instead, consecutive subrays form compact patches:
// each warp visits the leaves of its patch only.
uint32_t hilbert_d(uint32_t n, uint32_t x, uint32_t y) {
  uint32_t d = 0;
  for (uint32_t s = n / 2; s > 0; s /= 2) {
    const uint32_t rx = (x & s) > 0, ry = (y & s) > 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = n - 1 - x;
        y = n - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}
std::vector<SubrayConst> lane_order(const std::vector<SubrayConst>& t) {
  double rmax = 0.0;
  for (const SubrayConst& c : t) rmax = std::max(rmax, c.sin_t);
  std::vector<std::pair<uint32_t, uint32_t>> key;
  const uint32_t G = 256;
  for (const SubrayConst& c : t) {
    const double x = rmax > 0.0 ? c.sin_t * c.cos_p / rmax : 0.0;  // [-1, 1]
    const double y = rmax > 0.0 ? c.sin_t * c.sin_p / rmax : 0.0;
    const uint32_t gx = std::min(G - 1, (uint32_t)((x + 1.0) * 0.5 * G));
    const uint32_t gy = std::min(G - 1, (uint32_t)((y + 1.0) * 0.5 * G));
    key.emplace_back(hilbert_d(G, gx, gy), c.index);
  }
  std::stable_sort(key.begin(), key.end());
  std::vector<SubrayConst> o;
  for (const auto& k : key) o.push_back(t[k.second]);
  return o;
}

struct Derived {
  uint32_t n_bins = 0, taps = 0, jstar = 0;
  std::vector<double> kernel;
  Pattern pt;
};

helios_status validate_params(const helios_scanner_params* p, Derived* d) {
  if (!p) return fail(HELIOS_ERR_INVALID_ARGUMENT, "params is NULL");
  if (!(p->divergence_rad > 0.0 && p->divergence_rad < 0.1))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "divergence_rad must be in (0, 0.1)");
  d->pt = resolve_pattern(p->subray_count);
  if (d->pt.q < 0 || p->subray_count > (uint32_t)kMaxSubrays)
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "subray_count %u is neither 1+sum floor(2 pi i) nor 1+3q(q+1)", p->subray_count);
  if (!(p->pulse_length_ns > 0.0) || !std::isfinite(p->pulse_length_ns))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulse_length_ns must be > 0");
  if (!(p->bin_width_ns > 0.0) || !std::isfinite(p->bin_width_ns))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "bin_width_ns must be > 0");
  if (!(p->max_fullwave_range_ns >= p->bin_width_ns) || !std::isfinite(p->max_fullwave_range_ns))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "max_fullwave_range_ns must be >= bin_width_ns");
  if (!(p->detection_threshold > 0.0f && p->detection_threshold <= 1.0f))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "detection_threshold must be in (0, 1]");
  if (p->max_returns < 1 || p->max_returns > 255)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "max_returns must be in [1, 255]");
  if (!(p->range_noise_sd_m >= 0.0) || !std::isfinite(p->range_noise_sd_m))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "range_noise_sd_m must be finite and >= 0");
  if (p->fit_echo_width > 1 || p->reserved_ != 0)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "fit_echo_width must be 0 or 1, reserved_ 0");
  if (!(p->peak_power_w > 0.0) || !std::isfinite(p->peak_power_w))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "peak_power_w must be > 0");
  if (!(p->efficiency >= 0.0) || !(p->receiver_diameter_m >= 0.0) ||
      !std::isfinite(p->efficiency) || !std::isfinite(p->receiver_diameter_m))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "efficiency / receiver_diameter_m must be >= 0");
  if (!(p->beam_waist_m >= 0.0) || !(p->focus_range_m >= 0.0))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "beam_waist_m / focus_range_m must be >= 0");
  if (p->beam_waist_m > 0.0 && !(p->wavelength_nm > 0.0))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "wavelength_nm must be > 0 with Eq. 2 (beam_waist_m > 0)");
  const double nb = std::ceil(p->max_fullwave_range_ns / p->bin_width_ns);  // R9
  const double tau = p->pulse_length_ns / 1.75;
  const double taps = std::ceil(20.0 * tau / p->bin_width_ns);               // R9
  if (nb > 1e6) return fail(HELIOS_ERR_INVALID_ARGUMENT, "too many waveform bins (%g)", nb);
  if (taps > kMaxTaps || taps < 1)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulse kernel of %g taps out of range", taps);
  d->n_bins = (uint32_t)nb;
  d->taps = (uint32_t)taps;
  if (!waveform_fits(d->n_bins, p->subray_count, d->taps))
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "pulse kernel / subray tables do not fit shared memory");
  d->kernel.resize(d->taps);
  double best = -1.0;
  for (uint32_t j = 0; j < d->taps; ++j) {
    const double x = ((double)j + 0.5) * p->bin_width_ns / tau;  // bin centre (R9)
    d->kernel[j] = x * x * std::exp(-x);                             // Eq. 3 shape
    if (d->kernel[j] > best) {
      best = d->kernel[j];
      d->jstar = j;
    }
  }
  return HELIOS_OK;
}

// ---- 4^3-brick occupancy of the voxel grid (1 = some voxel has PAD > 0)
__global__ void k_bricks(const float* __restrict__ pad, uint32_t nx, uint32_t ny, uint32_t nz,
                         uint32_t nbx, uint32_t nby, uint8_t* __restrict__ bricks) {
  const uint64_t n = (uint64_t)nx * ny * nz;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!(pad[i] > 0.0f)) continue;
    const uint32_t x = (uint32_t)(i % nx), y = (uint32_t)((i / nx) % ny), z = (uint32_t)(i / ((uint64_t)nx * ny));
    bricks[(x >> kBrickShift) + nbx * ((y >> kBrickShift) + nby * (z >> kBrickShift))] = 1;
  }
}

// ---- validation kernel for scene arrays (finite vertices, rho in [0,1], PAD >= 0)
__global__ void k_check_scene(const float* __restrict__ xyz, uint64_t n_xyz,
                              const float* __restrict__ refl, uint64_t n_refl,
                              const float* __restrict__ pad, uint64_t n_pad,
                              unsigned* __restrict__ bad) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_xyz; i += stride)
    if (!isfinite(xyz[i])) atomicOr(bad, 1u);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_refl; i += stride) {
    const float r = refl[i];
    if (!(r >= 0.0f && r <= 1.0f)) atomicOr(bad, 2u);
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += stride) {
    const float v = pad[i];
    if (!(v >= 0.0f) || !isfinite(v)) atomicOr(bad, 4u);
  }
}


template <class T>
cudaError_t copy_in(T** dst, const T* src, size_t count, cudaStream_t s) {
  cudaError_t e = dev_alloc((void**)dst, sizeof(T) * (count ? count : 1), s);
  if (e != cudaSuccess) return e;
  if (count) e = cudaMemcpyAsync(*dst, src, sizeof(T) * count, cudaMemcpyDefault, s);
  return e;
}

// ---- serialised acceleration structure (helios_accel_export / _import)
constexpr uint64_t kAccelMagic = 0x31304343414C5848ull;  // "HXLACC01" little-endian
constexpr uint32_t kAccelVersion = 1;
struct AccelHeader {
  uint64_t magic;
  uint32_t version, header_bytes;
  uint32_t n_tris, n_nodes;
  int32_t root;
  uint32_t max_depth;
  uint64_t scene_hash;    // fingerprint of the triangle soup + reflectances
  uint64_t tri_bytes;     // each of the two triangle record arrays
  uint64_t node_bytes;
  uint32_t record_sizes;  // sizeof(TriRecord) | sizeof(Node) << 16
  uint32_t leaf_max;
  uint64_t reserved[8];
};
static_assert(sizeof(AccelHeader) % 16 == 0, "keeps the record arrays 16-B aligned");

// order-sensitive 64-bit fingerprint: the sum mod 2^64 of a mixed hash of
// (word index, word) over every word (deterministic in any summation order)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fingerprint(const uint32_t* __restrict__ w, uint64_t n, uint64_t salt,
                              unsigned long long* __restrict__ acc) {
  uint64_t sum = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    sum += mix64((i + salt) * 0x9E3779B97F4A7C15ull ^ (uint64_t)w[i]);
  for (int d = 16; d; d >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, d);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, (unsigned long long)sum);
}

cudaError_t scene_fingerprint(helios_scene sc, cudaStream_t s, uint64_t* out) {
  unsigned long long* d = nullptr;
  cudaError_t e = helios::dev_alloc((void**)&d, sizeof(*d), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d, 0, sizeof(*d), s);
  const uint64_t n9 = 9ull * sc->n_tris, n1 = sc->n_tris;
  auto run = [&](const void* p, uint64_t n, uint64_t salt) {
    if (e != cudaSuccess || !p || !n) return;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
    k_fingerprint<<<blocks, 256, 0, s>>>(static_cast<const uint32_t*>(p), n, salt, d);
    e = cudaGetLastError();
  };
  run(sc->d_xyz, n9, 0x51ull);
  run(sc->d_refl, n1, 0xA7ull << 40);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(d, s);
  *out = (uint64_t)h ^ ((uint64_t)sc->n_tris << 1);
  return e;
}

cudaError_t accel_header(helios_scene sc, cudaStream_t s, AccelHeader* h, bool tree = true) {
  *h = AccelHeader{};
  h->magic = kAccelMagic;
  h->version = kAccelVersion;
  h->header_bytes = sizeof(AccelHeader);
  h->n_tris = sc->n_tris;
  h->record_sizes = (uint32_t)sizeof(TriRecord) | ((uint32_t)sizeof(Node) << 16);
  h->leaf_max = kLeafMax;
  if (tree) {
    h->n_nodes = sc->bvh.n_nodes;
    h->root = sc->bvh.root;
    h->max_depth = sc->bvh.max_depth;
    h->tri_bytes = (uint64_t)sc->n_tris * sizeof(TriRecord);
    h->node_bytes = (uint64_t)sc->bvh.n_nodes * sizeof(Node);
  }
  return scene_fingerprint(sc, s, &h->scene_hash);
}

void free_scene(helios_scene sc, cudaStream_t s) {
  sc->free_slots();
  cudaFreeAsync(sc->d_xyz, s);
  cudaFreeAsync(sc->d_refl, s);
  cudaFreeAsync(sc->d_pad, s);
  cudaFreeAsync(sc->d_lut, s);
  cudaFreeAsync(sc->d_bricks, s);
  cudaFreeAsync(sc->bvh.tris, s);
  cudaFreeAsync(sc->bvh.filt, s);
  cudaFreeAsync(sc->bvh.nodes, s);
  cudaStreamSynchronize(s);
}

}  // namespace

extern "C" {

const char* helios_last_error(void) { return g_err.c_str(); }

const char* helios_version(void) { return "helios-b200 0.2 sm_100a"; }

helios_status helios_scene_create(const helios_scene_desc* desc, helios_stream stream,
                                  helios_scene* out) {
  helios::NvtxRange nvtx_("helios_scene_create");
  g_err.clear();
  if (!desc || !out) return fail(HELIOS_ERR_INVALID_ARGUMENT, "desc/out is NULL");
  *out = nullptr;
  const cudaStream_t s = (cudaStream_t)stream;
  if (desc->n_tris > 0 && !desc->p_tri_xyz)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_tri_xyz is NULL with n_tris = %u", desc->n_tris);
  if (desc->n_tris >= (1u << 28))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "n_tris >= 2^28 is not supported");
  const bool grid = desc->p_voxel_pad != nullptr;
  uint64_t nvox = 0;
  if (grid) {
    if (desc->nx == 0 || desc->ny == 0 || desc->nz == 0)
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "voxel grid dims must be > 0");
    if (!(desc->voxel_size > 0.0) || !std::isfinite(desc->voxel_size))
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "voxel_size must be > 0");
    for (int a = 0; a < 3; ++a)
      if (!std::isfinite(desc->grid_origin[a]))
        return fail(HELIOS_ERR_INVALID_ARGUMENT, "grid_origin must be finite");
    nvox = (uint64_t)desc->nx * desc->ny * desc->nz;
    if ((uint64_t)desc->n_tris + nvox >= 0xFFFFFFFFull)
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "n_tris + nx*ny*nz must be < 2^32 - 1");
  }
  if (desc->n_tris == 0 && !grid)
    return fail(HELIOS_ERR_EMPTY_SCENE, "scene has no triangles and no voxel grid");
  if (desc->voxel_mode > HELIOS_VOXEL_SCALED)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "unknown voxel_mode %u", desc->voxel_mode);
  if (desc->reserved_ != 0) return fail(HELIOS_ERR_INVALID_ARGUMENT, "reserved_ must be 0");
  if (desc->voxel_mode != HELIOS_VOXEL_TRANSMISSIVE &&
      !(desc->voxel_reflectance >= 0.0f && desc->voxel_reflectance <= 1.0f))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "voxel_reflectance must be in [0, 1]");
  if (desc->voxel_mode == HELIOS_VOXEL_SCALED &&
      (!(desc->pad_max > 0.0) || !std::isfinite(desc->pad_max) || !(desc->scale_alpha >= 0.0) ||
       !std::isfinite(desc->scale_alpha) || desc->scale_shift > 1))
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "scaled voxels need pad_max > 0, scale_alpha >= 0, scale_shift 0/1");
  if (desc->n_lut == 1 || desc->n_lut > (uint32_t)kMaxLut)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "n_lut must be 0 or in [2, %d]", kMaxLut);
  if (desc->n_lut > 0 && !desc->h_g_lut)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "h_g_lut is NULL with n_lut > 0");
  for (uint32_t k = 0; k < desc->n_lut; ++k)
    if (!(desc->h_g_lut[k] >= 0.0f) || !std::isfinite(desc->h_g_lut[k]))
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "h_g_lut[%u] must be finite and >= 0", k);

  helios_scene sc = new (std::nothrow) helios_scene_s();
  if (!sc) return fail(HELIOS_ERR_OUT_OF_MEMORY, "host allocation failed");
  cudaGetDevice(&sc->device);
  sc->n_tris = desc->n_tris;
  cudaError_t e = cudaSuccess;
  unsigned* d_bad = nullptr;
  unsigned bad = 0;
  do {
    if (desc->n_tris) {
      if ((e = copy_in(&sc->d_xyz, desc->p_tri_xyz, 9ull * desc->n_tris, s)) != cudaSuccess) break;
      if (desc->p_tri_reflectance &&
          (e = copy_in(&sc->d_refl, desc->p_tri_reflectance, desc->n_tris, s)) != cudaSuccess)
        break;
    }
    if (grid) {
      sc->nx = desc->nx;
      sc->ny = desc->ny;
      sc->nz = desc->nz;
      for (int a = 0; a < 3; ++a) sc->origin[a] = desc->grid_origin[a];
      sc->vs = desc->voxel_size;
      sc->voxel_mode = desc->voxel_mode;
      sc->voxel_refl = desc->voxel_reflectance;
      sc->pad_max = desc->pad_max;
      sc->scale_alpha = desc->scale_alpha;
      sc->scale_shift = desc->scale_shift;
      if ((e = copy_in(&sc->d_pad, desc->p_voxel_pad, nvox, s)) != cudaSuccess) break;
      // brick occupancy for empty-space skipping in the march
      sc->nbx = (sc->nx + (1u << kBrickShift) - 1) >> kBrickShift;
      sc->nby = (sc->ny + (1u << kBrickShift) - 1) >> kBrickShift;
      sc->nbz = (sc->nz + (1u << kBrickShift) - 1) >> kBrickShift;
      const size_t nbr = (size_t)sc->nbx * sc->nby * sc->nbz;
      if ((e = dev_alloc((void**)&sc->d_bricks, nbr, s)) != cudaSuccess) break;
      if ((e = cudaMemsetAsync(sc->d_bricks, 0, nbr, s)) != cudaSuccess) break;
      k_bricks<<<(unsigned)std::min<uint64_t>((nvox + 255) / 256, 148ull * 32), 256, 0, s>>>(
          sc->d_pad, sc->nx, sc->ny, sc->nz, sc->nbx, sc->nby, sc->d_bricks);
      if ((e = cudaGetLastError()) != cudaSuccess) break;
    }
    if (desc->n_lut) {
      sc->n_lut = desc->n_lut;
      if ((e = copy_in(&sc->d_lut, desc->h_g_lut, desc->n_lut, s)) != cudaSuccess) break;
    }
    if ((e = dev_alloc((void**)&d_bad, sizeof(unsigned), s)) != cudaSuccess) break;
    if ((e = cudaMemsetAsync(d_bad, 0, sizeof(unsigned), s)) != cudaSuccess) break;
    k_check_scene<<<148 * 4, 256, 0, s>>>(sc->d_xyz, 9ull * sc->n_tris, sc->d_refl,
                                         sc->d_refl ? sc->n_tris : 0, sc->d_pad,
                                         grid ? nvox : 0, d_bad);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(&bad, d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      break;
    e = cudaStreamSynchronize(s);
  } while (0);
  cudaFreeAsync(d_bad, s);
  if (e != cudaSuccess) {
    free_scene(sc, s);
    delete sc;
    return cuda_fail(e, "helios_scene_create");
  }
  if (bad) {
    free_scene(sc, s);
    delete sc;
    if (bad & 1u) return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_tri_xyz has a non-finite vertex");
    if (bad & 2u) return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_tri_reflectance outside [0, 1]");
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_voxel_pad has a negative or non-finite value");
  }
  *out = sc;
  return HELIOS_OK;
}

helios_status helios_build_accel(helios_scene sc, helios_stream stream) {
  helios::NvtxRange nvtx_("helios_build_accel");
  g_err.clear();
  if (!sc) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (sc->built) return HELIOS_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  char err[256] = {0};
  const helios_tuning tu = tuning_snapshot();
  cudaError_t e = build_lbvh(sc->d_xyz, sc->d_refl, sc->n_tris, tu.builder, s, &sc->bvh, err,
                             sizeof(err));
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation)
      return fail(HELIOS_ERR_OUT_OF_MEMORY, "helios_build_accel: %s", err);
    return fail(HELIOS_ERR_CUDA, "helios_build_accel: %s", err);
  }
  sc->built = true;
  return HELIOS_OK;
}

helios_status helios_accel_export(helios_scene sc, void* buffer, uint64_t* bytes,
                                  helios_stream stream) {
  helios::NvtxRange nvtx_("helios_accel_export");
  g_err.clear();
  if (!sc || !bytes) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene/bytes is NULL");
  if (!sc->built) return fail(HELIOS_ERR_NOT_BUILT, "helios_accel_export: scene not built");
  const cudaStream_t s = (cudaStream_t)stream;
  AccelHeader h{};
  cudaError_t e = accel_header(sc, s, &h);
  if (e != cudaSuccess) return cuda_fail(e, "helios_accel_export");
  const uint64_t total = h.header_bytes + 2 * h.tri_bytes + h.node_bytes;
  if (!buffer) {
    *bytes = total;
    return HELIOS_OK;
  }
  if (*bytes < total)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "helios_accel_export: buffer of %llu bytes < %llu",
                (unsigned long long)*bytes, (unsigned long long)total);
  char* out = static_cast<char*>(buffer);
  e = cudaMemcpyAsync(out, &h, sizeof(h), cudaMemcpyDefault, s);
  uint64_t at = h.header_bytes;
  if (e == cudaSuccess && h.tri_bytes)
    e = cudaMemcpyAsync(out + at, sc->bvh.tris, h.tri_bytes, cudaMemcpyDefault, s);
  at += h.tri_bytes;
  if (e == cudaSuccess && h.tri_bytes)
    e = cudaMemcpyAsync(out + at, sc->bvh.filt, h.tri_bytes, cudaMemcpyDefault, s);
  at += h.tri_bytes;
  if (e == cudaSuccess && h.node_bytes)
    e = cudaMemcpyAsync(out + at, sc->bvh.nodes, h.node_bytes, cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "helios_accel_export");
  *bytes = total;
  return HELIOS_OK;
}

helios_status helios_accel_import(helios_scene sc, const void* buffer, uint64_t bytes,
                                  helios_stream stream) {
  helios::NvtxRange nvtx_("helios_accel_import");
  g_err.clear();
  if (!sc || !buffer) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene/buffer is NULL");
  const cudaStream_t s = (cudaStream_t)stream;
  AccelHeader h{};
  if (bytes < sizeof(h)) return fail(HELIOS_ERR_INVALID_ARGUMENT, "helios_accel_import: not an accel blob");
  cudaError_t e = cudaMemcpyAsync(&h, buffer, sizeof(h), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "helios_accel_import");
  AccelHeader mine{};
  e = accel_header(sc, s, &mine, /*tree=*/false);
  if (e != cudaSuccess) return cuda_fail(e, "helios_accel_import");
  const uint64_t n = h.n_tris;
  if (h.magic != kAccelMagic || h.version != kAccelVersion || h.header_bytes != sizeof(h) ||
      h.record_sizes != mine.record_sizes || h.leaf_max != mine.leaf_max ||
      h.tri_bytes != n * sizeof(TriRecord) || h.node_bytes != (uint64_t)h.n_nodes * sizeof(Node) ||
      bytes < h.header_bytes + 2 * h.tri_bytes + h.node_bytes)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "helios_accel_import: not a valid accel blob");
  if (h.n_tris != sc->n_tris || h.scene_hash != mine.scene_hash)
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "helios_accel_import: the blob was exported from other triangles");
  helios::BuildResult r{};
  r.n_nodes = h.n_nodes;
  r.root = h.root;
  r.max_depth = h.max_depth;
  r.ms = 0.f;
  const char* in = static_cast<const char*>(buffer);
  if (n) {
    e = helios::dev_alloc((void**)&r.tris, h.tri_bytes, s);
    if (e == cudaSuccess) e = helios::dev_alloc((void**)&r.filt, h.tri_bytes, s);
    if (e == cudaSuccess && h.n_nodes) e = helios::dev_alloc((void**)&r.nodes, h.node_bytes, s);
    uint64_t at = h.header_bytes;
    if (e == cudaSuccess) e = cudaMemcpyAsync(r.tris, in + at, h.tri_bytes, cudaMemcpyDefault, s);
    at += h.tri_bytes;
    if (e == cudaSuccess) e = cudaMemcpyAsync(r.filt, in + at, h.tri_bytes, cudaMemcpyDefault, s);
    at += h.tri_bytes;
    if (e == cudaSuccess && h.n_nodes)
      e = cudaMemcpyAsync(r.nodes, in + at, h.node_bytes, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      cudaFreeAsync(r.tris, s);
      cudaFreeAsync(r.filt, s);
      cudaFreeAsync(r.nodes, s);
      cudaStreamSynchronize(s);
      cudaGetLastError();
      return e == cudaErrorMemoryAllocation
                 ? fail(HELIOS_ERR_OUT_OF_MEMORY, "helios_accel_import: out of device memory")
                 : cuda_fail(e, "helios_accel_import");
    }
  }
  // replace the previous tree (no call may be running on this scene)
  sc->free_slots();
  cudaFreeAsync(sc->bvh.tris, s);
  cudaFreeAsync(sc->bvh.filt, s);
  cudaFreeAsync(sc->bvh.nodes, s);
  cudaStreamSynchronize(s);
  sc->bvh = r;
  sc->built = true;
  return HELIOS_OK;
}

helios_status helios_scene_destroy(helios_scene sc) {
  g_err.clear();
  if (!sc) return HELIOS_OK;
  free_scene(sc, nullptr);
  delete sc;
  return HELIOS_OK;
}

helios_status helios_scene_get_info(helios_scene sc, helios_scene_info* out) {
  g_err.clear();
  if (!sc || !out) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene/out is NULL");
  out->n_tris = sc->n_tris;
  out->n_nodes = sc->bvh.n_nodes;
  out->max_depth = sc->bvh.max_depth;
  out->leaf_max = kLeafMax;
  out->node_bytes = (uint64_t)sc->bvh.n_nodes * sizeof(Node);
  out->tri_bytes = 2ull * sc->n_tris * sizeof(TriRecord);  // exact + filter records
  out->grid_bytes = (uint64_t)sc->nx * sc->ny * sc->nz * sizeof(float);
  out->build_ms = sc->bvh.ms;
  return HELIOS_OK;
}

uint32_t helios_waveform_bins(const helios_scanner_params* params) {
  g_err.clear();
  Derived d;
  return validate_params(params, &d) == HELIOS_OK ? d.n_bins : 0;
}

uint32_t helios_pulse_taps(const helios_scanner_params* params) {
  g_err.clear();
  Derived d;
  return validate_params(params, &d) == HELIOS_OK ? d.taps : 0;
}

}  // extern "C"

namespace {

helios_status validate_survey(const helios_survey* v) {
  if (!v) return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey is NULL");
  if (!v->h_waypoints || v->n_waypoints < 1)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey needs >= 1 waypoint");
  for (uint32_t i = 0; i < 3 * v->n_waypoints; ++i)
    if (!std::isfinite(v->h_waypoints[i]))
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey waypoint %u is not finite", i / 3);
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(v->mount[i])) return fail(HELIOS_ERR_INVALID_ARGUMENT, "mount not finite");
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(v->mount_offset[i]))
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "mount_offset not finite");
  if (v->n_waypoints > 1 && !(v->speed_m_s > 0.0 && std::isfinite(v->speed_m_s)))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "speed_m_s must be > 0 with > 1 waypoint");
  if (!(v->pulse_freq_hz > 0.0) || !std::isfinite(v->pulse_freq_hz))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulse_freq_hz must be > 0");
  if (!(v->scan_freq_hz > 0.0) || !std::isfinite(v->scan_freq_hz))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "scan_freq_hz must be > 0");
  const double amax = v->deflector == HELIOS_DEFLECTOR_PALMER ? 0.5 * kPi : kPi;
  if (!(v->scan_angle_rad >= 0.0 && v->scan_angle_rad < amax))
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "scan_angle_rad must be in [0, pi) (Palmer: [0, pi/2))");
  if (!std::isfinite(v->t0_s) || !std::isfinite(v->head_rotation_rad_s))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "t0_s / head_rotation_rad_s not finite");
  if (v->deflector > HELIOS_DEFLECTOR_PALMER)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "unknown deflector %u", v->deflector);
  if (v->deflector == HELIOS_DEFLECTOR_FIBRE && v->n_fibres == 0)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "n_fibres must be >= 1 with FIBRE");
  if (v->reserved_ != 0) return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey reserved_ must be 0");
  return HELIOS_OK;
}


// ---------------------------------------------------------------------------
// The chunk pipeline.  One call simulates one or more pulse batches ("jobs":
// helios_simulate = 1, helios_simulate_batches = n, helios_simulate_survey =
// 1 generated on the device).  Every job is cut into chunks; the chunks of all
// jobs form ONE pipeline over kSlots rotating scratch slots, so the head of a
// batch (its first K6a + K6) overlaps the tail of the previous one (its last
// K7 and copy-outs).  Per chunk c (slot = c % kSlots):
//   s  (or ts2 for odd c) : [wait inputs]  K0 (survey)  K6a  K6        -> t_done
//   ws (high priority)    : wait t_done    support scan  K7  [noise]   -> w_done
//   fs                    : echo-width fits (optional)                 -> w_done
//   cs                    : H2D of chunk c+1's host inputs             -> in_done
//   co                    : D2H of chunk c-2's host outputs            -> out_done
// ---------------------------------------------------------------------------
struct Job {
  const helios_pulses* pulses;
  const helios_outputs* out;
};

enum Arr { A_ORIGIN = 0, A_DIR, A_TIME, A_NRET, A_RET, A_K0, A_WF, A_HITS, A_COUNT };

helios_status simulate_impl(helios_scene sc, const helios_scanner_params* params,
                            const Job* jobs, uint32_t n_jobs, const helios_survey* survey,
                            uint64_t first_pulse, helios_stream stream, helios_stats* stats) {
  NvtxRange nvtx_(survey ? "helios_simulate_survey" : (n_jobs > 1 ? "helios_simulate_batches" : "helios_simulate"));
  g_err.clear();
  if (!sc) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!jobs || n_jobs == 0) return fail(HELIOS_ERR_INVALID_ARGUMENT, "no pulse batch given");
  for (uint32_t j = 0; j < n_jobs; ++j)
    if (!jobs[j].pulses || !jobs[j].out)
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulses/outputs of batch %u is NULL", j);
  if (survey) {
    const helios_status vs = validate_survey(survey);
    if (vs != HELIOS_OK) return vs;
  }
  Derived d;
  helios_status st = validate_params(params, &d);
  if (st != HELIOS_OK) return st;
  if (!sc->built) return fail(HELIOS_ERR_NOT_BUILT, "helios_build_accel has not been called");
  const helios_tuning tu = tuning_snapshot();
  const bool counters = stats && stats->collect_counters;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->collect_counters = counters ? 1u : 0u;
  }
  const uint32_t N = params->subray_count;
  const uint32_t R = params->max_returns;
  const bool gen = survey != nullptr;
  uint64_t total_n = 0;
  for (uint32_t j = 0; j < n_jobs; ++j) {
    const helios_pulses* P = jobs[j].pulses;
    const helios_outputs* O = jobs[j].out;
    if (P->n_pulses == 0) continue;
    total_n += P->n_pulses;
    if (!gen && (!P->p_origin || !P->p_direction))
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_origin/p_direction of batch %u is NULL", j);
    if (!O->p_n_returns || !O->p_wf_first_bin || (!O->p_returns && !O->p_returns_packed))
      return fail(HELIOS_ERR_INVALID_ARGUMENT,
                  "batch %u: p_n_returns/p_wf_first_bin and p_returns or p_returns_packed must "
                  "not be NULL", j);
    if (O->p_returns_packed && !O->p_return_offset)
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "batch %u: p_returns_packed needs p_return_offset", j);
    if (O->p_wf_compact && !O->p_wf_offset)
      return fail(HELIOS_ERR_INVALID_ARGUMENT, "batch %u: p_wf_compact needs p_wf_offset", j);
  }
  if (total_n == 0) return HELIOS_OK;
  const cudaStream_t s = (cudaStream_t)stream;

  // ---- per-job argument arrays: device-accessible as given, else staged
  // per chunk through the slot's scratch buffers
  const size_t per_pulse[A_COUNT] = {12, 12, 8, 1, sizeof(helios_return) * R, 8, 4ull * d.n_bins,
                                     sizeof(helios_subray_hit) * N};
  const bool is_in[A_COUNT] = {!gen, !gen, !gen, false, false, false, false, false};
  std::vector<const void*> user(n_jobs * A_COUNT);
  std::vector<char> staged(n_jobs * A_COUNT, 0);
  std::vector<char> want_offs(n_jobs), compact_staged(n_jobs), packed(n_jobs),
      packed_staged(n_jobs), job_staged(n_jobs), woff_pinned(n_jobs), roff_pinned(n_jobs);
  bool stage_any[A_COUNT] = {false};
  bool any_staged = false, any_offs = false, any_packed = false, any_cstaged = false,
       any_pstaged = false, any_opin = false;
  for (uint32_t j = 0; j < n_jobs; ++j) {
    const helios_pulses* P = jobs[j].pulses;
    const helios_outputs* O = jobs[j].out;
    const void* u[A_COUNT] = {gen ? (const void*)O->p_beam_origin : P->p_origin,
                              gen ? (const void*)O->p_beam_direction : P->p_direction,
                              gen ? (const void*)O->p_beam_time : P->p_time_s,
                              O->p_n_returns, O->p_returns, O->p_wf_first_bin, O->p_waveform,
                              O->p_subray_hits};
    for (int a = 0; a < A_COUNT; ++a) {
      user[j * A_COUNT + a] = u[a];
      if (P->n_pulses && u[a] && !device_accessible(u[a])) {
        staged[j * A_COUNT + a] = 1;
        stage_any[a] = true;
        job_staged[j] = 1;
      }
    }
    want_offs[j] = O->p_wf_offset != nullptr;
    compact_staged[j] = O->p_wf_compact && !device_accessible(O->p_wf_compact);
    packed[j] = O->p_returns_packed != nullptr;
    packed_staged[j] = packed[j] && !device_accessible(O->p_returns_packed);
    job_staged[j] |= compact_staged[j] | packed_staged[j];
    // offset arrays in pinned host memory leave chunk by chunk (drain_offsets)
    woff_pinned[j] = pinned_host(O->p_wf_offset);
    roff_pinned[j] = O->p_returns_packed && pinned_host(O->p_return_offset);
    any_opin |= woff_pinned[j] || roff_pinned[j];
    any_offs |= want_offs[j] != 0;
    any_packed |= packed[j] != 0;
    any_cstaged |= compact_staged[j] != 0;
    any_pstaged |= packed_staged[j] != 0;
    any_staged |= job_staged[j] != 0;
  }
  // arrays the kernels need although the caller passed none: generated pulses
  // without an export (survey), fixed return slots with packed returns only
  auto internal = [&](uint32_t j, int a) {
    return !user[(size_t)j * A_COUNT + a] && ((gen && a <= A_TIME) || a == A_RET);
  };
  bool internal_any[A_COUNT] = {false};
  for (uint32_t j = 0; j < n_jobs; ++j)
    for (int a = 0; a < A_COUNT; ++a) internal_any[a] |= jobs[j].pulses->n_pulses && internal(j, a);

  // ---- beam pre-pass K6a (packet traversal from per-pulse entry lists; trees
  // with internal nodes, beams of >= 7 subrays) unless switched off
  const bool beam_ok = N >= 7 && sc->n_tris > 0 && !ref_is_leaf(sc->bvh.root);
  const bool beam = beam_ok && tu.beam_prepass != 0;

  // ---- chunks.  Without the pre-pass: the K6 -> K7 records (12 B per subray)
  // stay L2-resident.  With it (or a voxel grid), per-chunk tails dominate:
  // >= 2 chunks per batch of <= 64 Mi subrays (>= 4 when it has host outputs)
  struct Chunk {
    uint32_t job;
    uint64_t b, m;
  };
  std::vector<Chunk> chunks;
  uint64_t chunk_max = 0;
  for (uint32_t j = 0; j < n_jobs; ++j) {
    const uint64_t n = jobs[j].pulses->n_pulses;
    if (n == 0) continue;
    uint64_t chunk = std::min<uint64_t>(n, std::max<uint64_t>(1024, (48ull << 20) / (12ull * N)));
    if (beam || sc->d_pad != nullptr) {
      // a batch of a multi-batch call with device outputs may be one chunk
      // of <= 128 Mi subrays: the batches themselves overlap in the pipeline,
      // and fewer, longer launches lose less to launch tails (C5 +1.2 %, C3
      // +2.6 %, profiles/r02s3_chunk_ab.txt); alone, or with host outputs,
      // >= 2 chunks of <= 64 Mi so that K6a / copies overlap within the batch
      // (a single batch too when its pulses have >= 64 subrays: K6a's
      // per-pulse walk is then small next to K6, so overlapping it with a
      // previous chunk buys less than one launch tail costs)
      const bool one_ok = !job_staged[j] && (n_jobs > 1 || N >= 64);
      const uint64_t kBeamChunkSubrays = one_ok ? (128ull << 20) : (64ull << 20);
      uint64_t k = std::max<uint64_t>(one_ok ? 1 : 2,
                                      (n * N + kBeamChunkSubrays - 1) / kBeamChunkSubrays);
      // host staging: >= 4 chunks per batch so copies overlap compute within a
      // single batch; a multi-batch call overlaps them across batches, and 2
      // chunks per batch measured faster there (C5 e2e 12.67 -> 12.46 ms per
      // 1 M pulses, tools/e2e_repro.py)
      if (job_staged[j]) k = std::max<uint64_t>(k, n_jobs > 1 ? 2 : 4);
      chunk = std::max(chunk, (n + k - 1) / k);
    }
    if (tu.chunk_pulses >= 1024) chunk = std::min<uint64_t>(n, tu.chunk_pulses);
    for (uint64_t b = 0; b < n; b += chunk) chunks.push_back({j, b, std::min(chunk, n - b)});
    chunk_max = std::max(chunk_max, chunk);
  }
  // per-job bases of the call-wide offset arrays (packed outputs)
  std::vector<uint64_t> job_off(n_jobs + 1, 0);
  for (uint32_t j = 0; j < n_jobs; ++j) job_off[j + 1] = job_off[j] + jobs[j].pulses->n_pulses + 1;

  // ---- host tables
  const std::vector<SubrayConst> tab = subray_table(N, params->divergence_rad, d.pt);
  const std::vector<SubrayConst> lanes = tu.lane_order ? lane_order(tab) : tab;
  const double beta = params->divergence_rad;
  const double K = params->efficiency * params->receiver_diameter_m * params->receiver_diameter_m /
                   (4.0 * kPi * beta * beta);  // Eq. 7 (R14)
  WavePlan plan = plan_waveform(d.n_bins, N, d.taps);
  if (plan.warps == 0)
    return fail(HELIOS_ERR_CUDA, "helios_simulate: waveform kernel cannot be configured");

  // ---- scratch layout
  size_t total = 0;
  auto carve = [&](size_t bytes) {
    const size_t at = total;
    total += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const uint64_t C = chunk_max;
  const size_t o_tab = carve(sizeof(SubrayConst) * N);
  const size_t o_ker = carve(sizeof(double) * d.taps);
  const size_t o_err = carve(sizeof(unsigned));
  const size_t o_cnt = carve(sizeof(unsigned long long) * 16);
  const size_t o_ws = carve(plan.scratch_bytes);
  const size_t o_wlist = carve(sizeof(uint32_t) * chunk_max);  // K7 wide-pass list (one stream)
  const size_t o_wcnt = carve(sizeof(unsigned));
  size_t o_wrec[kSlots], o_prim[kSlots], o_arr[A_COUNT][kSlots] = {}, o_ent[kSlots],
      o_frm[kSlots], o_fjob[kSlots], o_fy[kSlots], o_cst[kSlots], o_rst[kSlots];
  for (int k = 0; k < kSlots; ++k) {
    o_wrec[k] = carve(sizeof(WaveRec) * N * C);
    o_prim[k] = carve(sizeof(uint32_t) * N * C);
  }
  for (int a = 0; a < A_COUNT; ++a)
    if (stage_any[a] || internal_any[a])
      for (int k = 0; k < kSlots; ++k) o_arr[a][k] = carve(per_pulse[a] * C);
  const size_t o_wp = carve(gen ? sizeof(double) * 3 * survey->n_waypoints : 0);
  for (int k = 0; k < kSlots; ++k) {
    o_ent[k] = carve(beam ? sizeof(int2) * kEntryStride * C : 0);
    o_frm[k] = carve(beam ? sizeof(double) * 10 * C : 0);
  }
  const size_t scan_bytes = scan_temp_bytes(C, sizeof(uint64_t));
  const size_t o_len = carve(any_offs ? sizeof(uint64_t) * C : 0);
  const size_t o_offs = carve(any_offs ? sizeof(uint64_t) * job_off[n_jobs] : 0);
  const size_t o_scan = carve(any_offs ? scan_bytes : 0);
  const uint32_t fit_stride = 2u * (uint32_t)std::ceil(3.0 * params->pulse_length_ns /
                                                        params->bin_width_ns) + 1u;
  const bool fit = params->fit_echo_width != 0;
  for (int k = 0; k < kSlots; ++k) {
    o_fjob[k] = carve(fit ? sizeof(FitJob) * C * R : 0);
    o_fy[k] = carve(fit ? sizeof(double) * fit_stride * C * R : 0);
    o_cst[k] = carve(any_cstaged ? 4ull * d.n_bins * C : 0);
    o_rst[k] = carve(any_pstaged ? sizeof(helios_return) * R * C : 0);
  }
  const size_t o_fcnt = carve(fit ? kSlots * sizeof(unsigned) : 0);
  const size_t o_rlen = carve(any_packed ? sizeof(uint64_t) * C : 0);
  const size_t o_roffs = carve(any_packed ? sizeof(uint64_t) * job_off[n_jobs] : 0);
  const size_t o_rscan = carve(any_packed ? scan_bytes : 0);

  helios_scene_s::Slot* slot_ = nullptr;
  cudaError_t e = sc->acquire(s, total, &slot_);
  if (e != cudaSuccess) return cuda_fail(e, "helios_simulate (scratch)");
  char* buf = slot_->ptr;
  uint64_t* pin = slot_->pinned;
  const bool serial_all = tu.serialize != 0;
  // K7 overlaps K6 on its own stream, except on voxel scenes: there K6 is
  // ALU-bound (fp64 DDA + Philox) and a concurrent K7 costs more than it hides
  // (measured: profiles/r01_overlap_ab.txt); serialize = 1 puts every kernel
  // on the caller's stream (exclusive per-kernel times for the roofline)
  const bool serial = serial_all || sc->d_pad != nullptr;
  const cudaStream_t ws = serial ? s : slot_->wave;
  const cudaStream_t fs = serial ? s : slot_->fit;
  const cudaStream_t ts2 = serial ? s : slot_->trace2;  // K6 of odd chunks
  const cudaStream_t cs = slot_->copy_in, co = slot_->copy_out;
  auto sync_all = [&]() {
    cudaStreamSynchronize(s);
    cudaStreamSynchronize(ws);
    cudaStreamSynchronize(fs);
    cudaStreamSynchronize(ts2);
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(co);
  };
  SubrayConst* d_tab = reinterpret_cast<SubrayConst*>(buf + o_tab);
  double* d_ker = reinterpret_cast<double*>(buf + o_ker);
  unsigned* d_err = reinterpret_cast<unsigned*>(buf + o_err);
  unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(buf + o_cnt);
  double* d_wscratch = reinterpret_cast<double*>(buf + o_ws);
  uint64_t* d_len = reinterpret_cast<uint64_t*>(buf + o_len);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(buf + o_offs);
  uint64_t* d_rlen = reinterpret_cast<uint64_t*>(buf + o_rlen);
  uint64_t* d_roffs = reinterpret_cast<uint64_t*>(buf + o_roffs);
  e = cudaMemcpyAsync(d_tab, lanes.data(), sizeof(SubrayConst) * N, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_ker, d.kernel.data(), sizeof(double) * d.taps, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 16, s);
  // offs[job base] = 0: the carry the first chunk of each batch starts from
  for (uint32_t j = 0; j < n_jobs && e == cudaSuccess; ++j) {
    if (any_offs) e = cudaMemsetAsync(d_offs + job_off[j], 0, sizeof(uint64_t), s);
    if (e == cudaSuccess && any_packed)
      e = cudaMemsetAsync(d_roffs + job_off[j], 0, sizeof(uint64_t), s);
  }
  SurveyArgs sa{};
  if (e == cudaSuccess && gen) {
    sa.waypoints = reinterpret_cast<const double*>(buf + o_wp);
    e = cudaMemcpyAsync(buf + o_wp, survey->h_waypoints, sizeof(double) * 3 * survey->n_waypoints,
                        cudaMemcpyHostToDevice, s);
    sa.n_waypoints = survey->n_waypoints;
    sa.deflector = survey->deflector;
    sa.speed = survey->speed_m_s;
    for (int i = 0; i < 9; ++i) sa.mount[i] = survey->mount[i];
    for (int i = 0; i < 3; ++i) sa.offset[i] = survey->mount_offset[i];
    sa.head = survey->head_rotation_rad_s;
    sa.prf = survey->pulse_freq_hz;
    sa.t0 = survey->t0_s;
    sa.f = survey->scan_freq_hz;
    sa.A = survey->scan_angle_rad;
    sa.n_fibres = survey->n_fibres;
  }
  if (e != cudaSuccess) {
    sync_all();
    sc->release(slot_);
    return cuda_fail(e, "helios_simulate (setup)");
  }

  TraceArgs ta{};
  ta.tris = sc->bvh.tris;
  ta.filt = sc->bvh.filt;
  ta.nodes = sc->bvh.nodes;
  ta.root = sc->bvh.root;
  ta.n_tris = sc->n_tris;
  ta.pad = sc->d_pad;
  ta.nx = sc->nx;
  ta.ny = sc->ny;
  ta.nz = sc->nz;
  ta.gx0 = sc->origin[0];
  ta.gy0 = sc->origin[1];
  ta.gz0 = sc->origin[2];
  ta.vs = sc->vs;
  ta.g_lut = sc->d_lut;
  ta.n_lut = sc->n_lut;
  ta.voxel_mode = sc->voxel_mode;
  ta.bricks = sc->d_bricks;
  ta.nbx = sc->nbx;
  ta.nby = sc->nby;
  ta.voxel_refl = sc->voxel_refl;
  ta.pad_max = sc->pad_max;
  ta.scale_alpha = sc->scale_alpha;
  ta.scale_shift = sc->scale_shift;
  ta.sub = d_tab;
  ta.N = N;
  {
    // pad a pulse to whole warps when that wastes <= 6 % of the lanes (91 -> 96):
    // every warp then walks one pulse's patch
    const uint32_t padded = (N + 31u) / 32u * 32u;
    const bool pad = tu.pad_lanes < 0 ? (padded - N) * 100u <= 6u * N : tu.pad_lanes != 0;
    ta.lanes = pad ? padded : N;
  }
  ta.seed = params->seed;
  ta.K = K;
  ta.I0 = params->peak_power_w;
  ta.eq2 = params->beam_waist_m > 0.0 ? 1 : 0;
  ta.w0 = params->beam_waist_m;
  ta.lambda_m = params->wavelength_nm * 1e-9;
  ta.R0 = params->focus_range_m;
  ta.err_flag = d_err;
  ta.counters = d_cnt;
  ta.delta_ns = params->bin_width_ns;
  ta.inv_bin = 1.0 / (kC * (params->bin_width_ns * 1e-9));
  {
    double smax = 0.0;
    for (const SubrayConst& t : tab) smax = std::max(smax, t.sin_t);
    ta.cone_sin = smax * (1.0 + 1e-9) + 1e-12;  // widened: covers the fp64 subray directions
#ifndef HELIOS_BEAM_K
#define HELIOS_BEAM_K 6.0
#endif
    ta.beam_k = HELIOS_BEAM_K;  // measured (profiles/r01s3_beam_ab.txt, r02_beam_k_ab.txt)
  }

  WaveArgs wa{};
  wa.N = N;
  wa.n_bins = d.n_bins;
  wa.taps = d.taps;
  wa.jstar = d.jstar;
  wa.kernel = d_ker;
  wa.delta_ns = params->bin_width_ns;
  wa.thr = params->detection_threshold;
  wa.max_returns = R;
  // echo-width fit (R28): window half-width and LM start value
  wa.fit = params->fit_echo_width;
  wa.fit_half = (int)std::ceil(3.0 * params->pulse_length_ns / params->bin_width_ns);
  wa.fit_s0 = params->pulse_length_ns / (2.0 * std::sqrt(2.0 * std::log(2.0)));
  wa.counters = counters ? d_cnt + 4 : nullptr;
  wa.noise_sd = params->range_noise_sd_m;
  wa.fit_stride = fit_stride;
  wa.err_flag = d_err;
  wa.seed = params->seed;
  wa.wide_list = reinterpret_cast<uint32_t*>(buf + o_wlist);
  wa.wide_count = reinterpret_cast<unsigned*>(buf + o_wcnt);

  // per-kernel device time (CUDA events on each kernel's stream)
  std::vector<cudaEvent_t> ev_b, ev_t, ev_w;
  auto mark = [&](std::vector<cudaEvent_t>& v, cudaStream_t st) {
    if (!stats) return;
    cudaEvent_t x;
    if (cudaEventCreate(&x) == cudaSuccess) {
      cudaEventRecord(x, st);
      v.push_back(x);
    }
  };
  // trace_spans: device-side spans of the streams (stderr), for diagnosis
  std::vector<std::pair<char, cudaEvent_t>> tev;
  cudaEvent_t tev0 = nullptr;
  auto tmark = [&](char tag, cudaStream_t st) {
    if (!tu.trace_spans) return;
    cudaEvent_t x;
    if (cudaEventCreate(&x) == cudaSuccess) {
      cudaEventRecord(x, st);
      tev.emplace_back(tag, x);
    }
  };
  if (tu.trace_spans && cudaEventCreate(&tev0) == cudaSuccess) cudaEventRecord(tev0, s);
  double host_wait_ms = 0.0;
  const double call_t0 = tu.trace_spans ? now_ms() : 0.0;

  cudaEvent_t in_done[kSlots] = {}, t_done[kSlots] = {}, w_done[kSlots] = {},
              out_done[kSlots] = {}, off_done[kSlots] = {}, cd_done[kSlots] = {},
              k7_done[kSlots] = {}, roff_done[kSlots] = {}, rd_done[kSlots] = {};
  cudaEvent_t ev_setup = nullptr;
  auto mk = [&](cudaEvent_t* x) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(x, cudaEventDisableTiming);
  };
  mk(&ev_setup);
  for (int k = 0; k < kSlots; ++k) {
    mk(&t_done[k]);
    mk(&w_done[k]);
    if (fit) mk(&k7_done[k]);
    if (any_pstaged) {
      mk(&roff_done[k]);
      mk(&rd_done[k]);
    }
    if (any_cstaged) {
      mk(&off_done[k]);
      mk(&cd_done[k]);
    }
    if (any_staged) {
      mk(&in_done[k]);
      mk(&out_done[k]);
    }
  }
  // every other stream starts after the setup work on `s`
  if (e == cudaSuccess) e = cudaEventRecord(ev_setup, s);
  for (cudaStream_t x : {ws, fs, ts2, cs, co})
    if (e == cudaSuccess && x != s) e = cudaStreamWaitEvent(x, ev_setup, 0);

  auto dev_ptr = [&](int a, int slot, const Chunk& ch) -> char* {
    const size_t ix = (size_t)ch.job * A_COUNT + a;
    if (staged[ix] || internal(ch.job, a)) return buf + o_arr[a][slot];
    if (!user[ix]) return nullptr;
    return (char*)user[ix] + per_pulse[a] * ch.b;
  };
  auto copy_in = [&](uint64_t c) -> cudaError_t {
    const Chunk& ch = chunks[c];
    const int slot = (int)(c % kSlots);
    for (int a = 0; a < A_COUNT; ++a) {
      const size_t ix = (size_t)ch.job * A_COUNT + a;
      if (is_in[a] && staged[ix]) {
        cudaError_t r = cudaMemcpyAsync(buf + o_arr[a][slot],
                                        (const char*)user[ix] + per_pulse[a] * ch.b,
                                        per_pulse[a] * ch.m, cudaMemcpyHostToDevice, cs);
        if (r != cudaSuccess) return r;
      }
    }
    return cudaEventRecord(in_done[slot], cs);
  };
  // staged packed rows of chunk c: the host learns the chunk's offset range
  // from the pinned mirror (written on the waveform stream right after the
  // chunk's scan), then queues the copy behind K7(c).  Called kSlots-1 chunks
  // late, so the GPU never waits for the host.
  auto drain_compact = [&](uint64_t c) -> cudaError_t {
    const Chunk& ch = chunks[c];
    if (!compact_staged[ch.job]) return cudaSuccess;
    const int sl = (int)(c % kSlots);
    const double h0 = tu.trace_spans ? now_ms() : 0.0;
    cudaError_t r = cudaEventSynchronize(off_done[sl]);
    if (tu.trace_spans) host_wait_ms += now_ms() - h0;
    if (r != cudaSuccess) return r;
    const helios_outputs* O = jobs[ch.job].out;
    const uint64_t first = pin[2 * sl], last = std::min(pin[2 * sl + 1], O->wf_compact_capacity);
    r = cudaStreamWaitEvent(co, w_done[sl], 0);
    tmark('c', co);
    if (r == cudaSuccess && last > first)
      r = cudaMemcpyAsync(O->p_wf_compact + first, buf + o_cst[sl], sizeof(float) * (last - first),
                          cudaMemcpyDeviceToHost, co);
    tmark('C', co);
    if (r == cudaSuccess) r = cudaEventRecord(cd_done[sl], co);
    return r;
  };
  auto drain_returns = [&](uint64_t c) -> cudaError_t {
    const Chunk& ch = chunks[c];
    if (!packed_staged[ch.job]) return cudaSuccess;
    const int sl = (int)(c % kSlots);
    const double h0 = tu.trace_spans ? now_ms() : 0.0;
    cudaError_t r = cudaEventSynchronize(roff_done[sl]);
    if (tu.trace_spans) host_wait_ms += now_ms() - h0;
    if (r != cudaSuccess) return r;
    const helios_outputs* O = jobs[ch.job].out;
    const uint64_t first = pin[2 * kSlots + 2 * sl],
                   last = std::min(pin[2 * kSlots + 2 * sl + 1], O->returns_capacity);
    r = cudaStreamWaitEvent(co, w_done[sl], 0);
    if (r == cudaSuccess && last > first)
      r = cudaMemcpyAsync(O->p_returns_packed + first, buf + o_rst[sl],
                          sizeof(helios_return) * (last - first), cudaMemcpyDeviceToHost, co);
    if (r == cudaSuccess) r = cudaEventRecord(rd_done[sl], co);
    return r;
  };
  // staged fixed-size outputs of chunk c -> host; out_done marks the slot free
  auto drain_fixed = [&](uint64_t c) -> cudaError_t {
    const Chunk& ch = chunks[c];
    const int sl = (int)(c % kSlots);
    cudaError_t r = cudaStreamWaitEvent(co, w_done[sl], 0);
    tmark('f', co);
    for (int a = 0; a < A_COUNT && r == cudaSuccess; ++a) {
      const size_t ix = (size_t)ch.job * A_COUNT + a;
      if (!is_in[a] && staged[ix])
        r = cudaMemcpyAsync((char*)user[ix] + per_pulse[a] * ch.b, buf + o_arr[a][sl],
                            per_pulse[a] * ch.m, cudaMemcpyDeviceToHost, co);
    }
    tmark('F', co);
    if (r == cudaSuccess) r = cudaEventRecord(out_done[sl], co);
    return r;
  };
  // the chunk's entries [b, b + m] of the call-wide offset arrays -> pinned host
  // arrays as soon as the chunk is done (final after its scans), instead of
  // n + 1 words per batch after the last chunk (C5: 16 MB per 1 M pulses
  // less in the call's tail)
  auto drain_offsets = [&](uint64_t c) -> cudaError_t {
    const Chunk& ch = chunks[c];
    if (!woff_pinned[ch.job] && !roff_pinned[ch.job]) return cudaSuccess;
    const int sl = (int)(c % kSlots);
    const helios_outputs* O = jobs[ch.job].out;
    const size_t bytes = sizeof(uint64_t) * (ch.m + 1);
    cudaError_t r = cudaStreamWaitEvent(co, w_done[sl], 0);
    if (r == cudaSuccess && woff_pinned[ch.job])
      r = cudaMemcpyAsync(O->p_wf_offset + ch.b, d_offs + job_off[ch.job] + ch.b, bytes,
                          cudaMemcpyDeviceToHost, co);
    if (r == cudaSuccess && roff_pinned[ch.job])
      r = cudaMemcpyAsync(O->p_return_offset + ch.b, d_roffs + job_off[ch.job] + ch.b, bytes,
                          cudaMemcpyDeviceToHost, co);
    return r;
  };

  uint32_t launches = 0, trace_launches = 0;
  const uint64_t n_chunks = chunks.size();
  const bool dual_trace = !serial;
  if (any_staged && e == cudaSuccess) e = copy_in(0);
  for (uint64_t c = 0; c < n_chunks && e == cudaSuccess; ++c) {
    const Chunk& ch = chunks[c];
    const helios_pulses* P = jobs[ch.job].pulses;
    const helios_outputs* O = jobs[ch.job].out;
    const uint64_t b = ch.b, m = ch.m;
    const int slot = (int)(c % kSlots);
    const cudaStream_t ts = (dual_trace && (c & 1)) ? ts2 : s;
    const bool reuse = c >= (uint64_t)kSlots;  // the slot's previous user: chunk c - kSlots
    if (any_staged) e = cudaStreamWaitEvent(ts, in_done[slot], 0);
    if (e == cudaSuccess && reuse) e = cudaStreamWaitEvent(ts, w_done[slot], 0);
    // K6 / K0 overwrite staged slot buffers chunk c-K copies out: wait for that
    if (e == cudaSuccess && any_staged && reuse) e = cudaStreamWaitEvent(ts, out_done[slot], 0);
    NvtxRange nvtx_chunk("chunk: K0/K6a/K6 -> K7");
    if (e == cudaSuccess && gen) {
      e = launch_generate(sa, first_pulse + b, m, (float*)dev_ptr(A_ORIGIN, slot, ch),
                          (float*)dev_ptr(A_DIR, slot, ch), (double*)dev_ptr(A_TIME, slot, ch), ts);
      ++launches;
    }
    if (e != cudaSuccess) break;
    ta.origin = (const float*)dev_ptr(A_ORIGIN, slot, ch);
    ta.direction = (const float*)dev_ptr(A_DIR, slot, ch);
    ta.n_pulses = m;
    ta.pulse_base = P->pulse_index_base + b;
    ta.wrec = reinterpret_cast<WaveRec*>(buf + o_wrec[slot]);
    ta.prim = reinterpret_cast<uint32_t*>(buf + o_prim[slot]);
    ta.out = (helios_subray_hit*)dev_ptr(A_HITS, slot, ch);
    ta.entries = nullptr;
    ta.frames = nullptr;
    if (beam) {
      ta.entries = reinterpret_cast<int2*>(buf + o_ent[slot]);
      ta.frames = reinterpret_cast<double*>(buf + o_frm[slot]);
      mark(ev_b, ts);
      tmark('b', ts);
      e = launch_beam(ta, counters, ts);
      tmark('B', ts);
      mark(ev_b, ts);
      ++launches;
    }
    mark(ev_t, ts);
    tmark('t', ts);
    if (e == cudaSuccess) e = launch_trace(ta, counters, ts);
    tmark('T', ts);
    mark(ev_t, ts);
    ++launches;
    ++trace_launches;
    if (e == cudaSuccess) e = cudaEventRecord(t_done[slot], ts);
    if (e == cudaSuccess && ws != ts) e = cudaStreamWaitEvent(ws, t_done[slot], 0);
    if (e == cudaSuccess && any_staged && reuse) e = cudaStreamWaitEvent(ws, out_done[slot], 0);
    if (e == cudaSuccess && any_cstaged && reuse) e = cudaStreamWaitEvent(ws, cd_done[slot], 0);
    uint64_t* offs = want_offs[ch.job] ? d_offs + job_off[ch.job] + b : nullptr;
    if (e == cudaSuccess && offs) {
      // packed rows: support lengths -> inclusive scan into offs[1..m] seeded
      // with offs[0] (the previous chunks of this batch), on K7's stream
      e = launch_support(ta.wrec, N, m, d.n_bins, d.taps, d_len, ws);
      if (e == cudaSuccess) e = scan_u64(d_len, offs + 1, m, true, buf + o_scan, scan_bytes, ws, offs);
      launches += 4;
      if (e == cudaSuccess && compact_staged[ch.job]) {
        e = cudaMemcpyAsync(pin + 2 * slot, offs, sizeof(uint64_t), cudaMemcpyDeviceToHost, ws);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(pin + 2 * slot + 1, offs + m, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, ws);
        if (e == cudaSuccess) e = cudaEventRecord(off_done[slot], ws);
      }
    }
    if (e != cudaSuccess) break;
    wa.rec = ta.wrec;
    wa.prim = ta.prim;
    wa.n_pulses = m;
    wa.pulse_base = ta.pulse_base;
    wa.time_s = (const double*)dev_ptr(A_TIME, slot, ch);
    wa.n_returns = (uint8_t*)dev_ptr(A_NRET, slot, ch);
    wa.returns = (helios_return*)dev_ptr(A_RET, slot, ch);
    wa.first_bin = (int64_t*)dev_ptr(A_K0, slot, ch);
    wa.waveform = (float*)dev_ptr(A_WF, slot, ch);
    wa.offs = offs;
    wa.compact = compact_staged[ch.job] ? reinterpret_cast<float*>(buf + o_cst[slot])
                                        : O->p_wf_compact;
    wa.compact_staged = compact_staged[ch.job] ? 1 : 0;
    wa.capacity = O->p_wf_compact ? O->wf_compact_capacity : 0;
    if (fit) {
      wa.fit_jobs = reinterpret_cast<FitJob*>(buf + o_fjob[slot]);
      wa.fit_y = reinterpret_cast<double*>(buf + o_fy[slot]);
      wa.fit_count = reinterpret_cast<unsigned*>(buf + o_fcnt) + slot;
      e = cudaMemsetAsync(wa.fit_count, 0, sizeof(unsigned), ws);
    }
    mark(ev_w, ws);
    tmark('w', ws);
    if (e == cudaSuccess) e = launch_waveform(wa, plan, d_wscratch, ws);
    tmark('W', ws);
    if (e == cudaSuccess && wa.noise_sd > 0.0) {
      e = launch_range_noise(wa, ws);
      ++launches;
    }
    mark(ev_w, ws);
    launches += 2;  // K7 main + wide pass
    cudaStream_t post = ws;  // the stream that completes the chunk's returns
    if (e == cudaSuccess && fit) {
      // echo-width fits on their own stream (their tail overlaps later chunks)
      if (fs != ws) e = cudaEventRecord(k7_done[slot], ws);
      if (e == cudaSuccess && fs != ws) e = cudaStreamWaitEvent(fs, k7_done[slot], 0);
      if (e == cudaSuccess) e = launch_fit(wa, fs);
      ++launches;
      post = fs;
    }
    if (e == cudaSuccess && packed[ch.job]) {
      // packed returns: scan of the counts, copy of the used slots
      if (packed_staged[ch.job] && reuse) e = cudaStreamWaitEvent(post, rd_done[slot], 0);
      helios_return* dst = packed_staged[ch.job]
                               ? reinterpret_cast<helios_return*>(buf + o_rst[slot])
                               : O->p_returns_packed;
      uint64_t* roffs = d_roffs + job_off[ch.job] + b;
      if (e == cudaSuccess)
        e = launch_pack_returns(wa.returns, wa.n_returns, m, R, d_rlen, roffs, buf + o_rscan,
                                scan_bytes, dst, packed_staged[ch.job] ? 1 : 0,
                                O->returns_capacity, post);
      launches += 5;
      if (e == cudaSuccess && packed_staged[ch.job]) {
        e = cudaMemcpyAsync(pin + 2 * kSlots + 2 * slot, roffs, sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, post);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(pin + 2 * kSlots + 2 * slot + 1, roffs + m, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, post);
        if (e == cudaSuccess) e = cudaEventRecord(roff_done[slot], post);
      }
    }
    if (e == cudaSuccess) e = cudaEventRecord(w_done[slot], post);
    // copy-outs run kSlots-1 chunks behind, so the host never blocks on a
    // chunk whose K7 may still be queued behind the K6 it just enqueued; all
    // copy-outs of a chunk leave in one go, in chunk order
    constexpr uint64_t kLag = kSlots - 1;
    if (c >= kLag) {
      const uint64_t cc = c - kLag;
      if (e == cudaSuccess && any_cstaged) e = drain_compact(cc);
      if (e == cudaSuccess && any_pstaged) e = drain_returns(cc);
      if (e == cudaSuccess && any_staged) e = drain_fixed(cc);
      if (e == cudaSuccess && any_opin) e = drain_offsets(cc);
    }
    // prefetch the next chunk's inputs into its slot once that slot's previous
    // user (chunk c+1-kSlots) is done with it
    if (e == cudaSuccess && any_staged && c + 1 < n_chunks) {
      const int nslot = (int)((c + 1) % kSlots);
      if (c + 1 >= (uint64_t)kSlots) e = cudaStreamWaitEvent(cs, w_done[nslot], 0);
      if (e == cudaSuccess) e = copy_in(c + 1);
    }
  }
  for (uint64_t c = n_chunks > (uint64_t)(kSlots - 1) ? n_chunks - (kSlots - 1) : 0;
       c < n_chunks && e == cudaSuccess; ++c) {
    if (any_cstaged) e = drain_compact(c);
    if (e == cudaSuccess && any_pstaged) e = drain_returns(c);
    if (e == cudaSuccess && any_staged) e = drain_fixed(c);
    if (e == cudaSuccess && any_opin) e = drain_offsets(c);
  }
  // join: the caller's stream is ordered after every kernel and copy of the call
  for (int k = 0; k < kSlots && (uint64_t)k < n_chunks && e == cudaSuccess; ++k)
    e = cudaStreamWaitEvent(s, w_done[k], 0);
  // call-wide offsets of every batch to the caller (device or host memory;
  // pinned host arrays already left chunk by chunk)
  for (uint32_t j = 0; j < n_jobs && e == cudaSuccess; ++j) {
    const helios_outputs* O = jobs[j].out;
    const uint64_t n = jobs[j].pulses->n_pulses;
    if (n == 0) continue;
    if (O->p_wf_offset && !woff_pinned[j])
      e = cudaMemcpyAsync(O->p_wf_offset, d_offs + job_off[j], sizeof(uint64_t) * (n + 1),
                          cudaMemcpyDefault, s);
    if (e == cudaSuccess && O->p_return_offset && !roff_pinned[j])
      e = cudaMemcpyAsync(O->p_return_offset, d_roffs + job_off[j], sizeof(uint64_t) * (n + 1),
                          cudaMemcpyDefault, s);
  }
  unsigned herr = 0;
  unsigned long long hcnt[16] = {0};
  std::vector<uint64_t> htot(n_jobs, 0), hrtot(n_jobs, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  for (uint32_t j = 0; j < n_jobs && e == cudaSuccess; ++j) {
    const uint64_t n = jobs[j].pulses->n_pulses;
    if (n == 0) continue;
    if (want_offs[j])
      e = cudaMemcpyAsync(&htot[j], d_offs + job_off[j] + n, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && packed[j])
      e = cudaMemcpyAsync(&hrtot[j], d_roffs + job_off[j] + n, 8, cudaMemcpyDeviceToHost, s);
  }
  if (e == cudaSuccess && counters)
    e = cudaMemcpyAsync(hcnt, d_cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(co);
  if (tu.trace_spans && tev0) {
    std::string line;
    for (auto& pr : tev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev0, pr.second);
      char bb[32];
      snprintf(bb, sizeof bb, " %c%.2f", pr.first, ms);
      line += bb;
      cudaEventDestroy(pr.second);
    }
    cudaEventDestroy(tev0);
    fprintf(stderr, "helios_simulate spans (ms from call start; b/B K6a, t/T K6, w/W K7, f/F "
                    "fixed copy-out, c/C rows copy-out):%s\n", line.c_str());
    fprintf(stderr, "helios_simulate: %llu pulses, %u batches, %llu chunks, host %.3f ms, "
                    "blocked in drains %.3f ms\n", (unsigned long long)total_n, n_jobs,
            (unsigned long long)n_chunks, now_ms() - call_t0, host_wait_ms);
  }
  auto sum_ms = [](std::vector<cudaEvent_t>& v) {
    double t = 0.0;
    for (size_t i = 0; i + 1 < v.size(); i += 2) {
      float a = 0.f;
      if (cudaEventElapsedTime(&a, v[i], v[i + 1]) == cudaSuccess) t += a;
    }
    for (cudaEvent_t x : v) cudaEventDestroy(x);
    return t;
  };
  const double t_beam = sum_ms(ev_b), t_trace = sum_ms(ev_t), t_wave = sum_ms(ev_w);
  for (cudaEvent_t* arr : {in_done, t_done, w_done, out_done, off_done, cd_done, k7_done,
                           roff_done, rd_done})
    for (int k = 0; k < kSlots; ++k)
      if (arr[k]) cudaEventDestroy(arr[k]);
  if (ev_setup) cudaEventDestroy(ev_setup);
  cudaGetLastError();
  sync_all();
  sc->release(slot_);
  if (e != cudaSuccess) return cuda_fail(e, "helios_simulate");
  if (stats) {
    stats->pulses = total_n;
    stats->subrays = total_n * N;
    stats->kernel_launches = launches;
    stats->trace_launches = trace_launches;
    stats->beam_nodes = hcnt[7];
    stats->node_bytes = (uint32_t)sizeof(Node);
    stats->trace_ms = t_trace;
    stats->beam_ms = t_beam;
    stats->waveform_ms = t_wave;
    stats->nodes_visited = hcnt[0];
    stats->tris_tested = hcnt[1];
    stats->voxel_steps = hcnt[2];
    stats->voxel_returns = hcnt[3];
    stats->fp64_tests = hcnt[6];
    stats->subray_hits = hcnt[4];
    stats->returns = hcnt[5];
    stats->batches = n_jobs;
    stats->warp_entries = hcnt[8];
    stats->warp_steps = hcnt[9];
    stats->warp_leaf_tris = hcnt[10];
    stats->warp_entries_walked = hcnt[11];
    stats->warp_fp64_in_walk = hcnt[12];
    stats->second_definite_hits = hcnt[13];
    stats->chunks = (uint32_t)n_chunks;
  }
  if (herr & 4u) return fail(HELIOS_ERR_CUDA, "internal: compact row length mismatch");
  if (herr & 1u) return fail(HELIOS_ERR_INVALID_ARGUMENT, "a pulse direction has zero length");
  for (uint32_t j = 0; j < n_jobs; ++j) {
    const helios_outputs* O = jobs[j].out;
    if (packed[j] && hrtot[j] > O->returns_capacity)
      return fail(HELIOS_ERR_CAPACITY, "batch %u: packed returns need %llu slots, capacity %llu",
                  j, (unsigned long long)hrtot[j], (unsigned long long)O->returns_capacity);
    if (O->p_wf_compact && htot[j] > O->wf_compact_capacity)
      return fail(HELIOS_ERR_CAPACITY, "batch %u: compact waveform needs %llu floats, capacity %llu",
                  j, (unsigned long long)htot[j], (unsigned long long)O->wf_compact_capacity);
  }
  return HELIOS_OK;
}

}  // namespace

extern "C" {

helios_status helios_simulate(helios_scene sc, const helios_scanner_params* params,
                              const helios_pulses* pulses, const helios_outputs* outputs,
                              helios_stream stream, helios_stats* stats) {
  g_err.clear();
  if (!pulses || !outputs) return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulses/outputs is NULL");
  const Job j{pulses, outputs};
  return simulate_impl(sc, params, &j, 1, nullptr, 0, stream, stats);
}

helios_status helios_simulate_batches(helios_scene sc, const helios_scanner_params* params,
                                      const helios_pulses* pulses, const helios_outputs* outputs,
                                      uint32_t n_batches, helios_stream stream,
                                      helios_stats* stats) {
  g_err.clear();
  if (n_batches == 0) return HELIOS_OK;
  if (!pulses || !outputs) return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulses/outputs is NULL");
  std::vector<Job> jobs(n_batches);
  for (uint32_t i = 0; i < n_batches; ++i) jobs[i] = Job{pulses + i, outputs + i};
  return simulate_impl(sc, params, jobs.data(), n_batches, nullptr, 0, stream, stats);
}

// Non-blocking calls: a worker thread per call runs the blocking pipeline on
// the scene's device (the scratch cache is per caller stream and locked, so
// calls on distinct streams run concurrently).
struct helios_call_s {
  std::thread worker;
  helios_scanner_params params{};
  std::vector<helios_pulses> pulses;
  std::vector<helios_outputs> outputs;
  helios_stats stats{};
  bool has_stats = false;
  helios_status status = HELIOS_OK;
  std::string err;
};

helios_status helios_simulate_batches_async(helios_scene sc, const helios_scanner_params* params,
                                            const helios_pulses* pulses,
                                            const helios_outputs* outputs, uint32_t n_batches,
                                            helios_stream stream, const helios_stats* stats,
                                            helios_call* call) {
  g_err.clear();
  if (!call) return fail(HELIOS_ERR_INVALID_ARGUMENT, "call is NULL");
  *call = nullptr;
  if (!sc) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!params) return fail(HELIOS_ERR_INVALID_ARGUMENT, "params is NULL");
  if (n_batches && (!pulses || !outputs))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulses/outputs is NULL");
  helios_call_s* c = new (std::nothrow) helios_call_s;
  if (!c) return fail(HELIOS_ERR_OUT_OF_MEMORY, "helios_simulate_batches_async: no memory");
  c->params = *params;
  c->pulses.assign(pulses, pulses + n_batches);
  c->outputs.assign(outputs, outputs + n_batches);
  c->has_stats = stats != nullptr;
  if (stats) c->stats = *stats;
  const int dev = sc->device;
  try {
    c->worker = std::thread([c, sc, stream, dev]() {
      cudaSetDevice(dev);
      const uint32_t n = (uint32_t)c->pulses.size();
      std::vector<Job> jobs(n);
      for (uint32_t i = 0; i < n; ++i) jobs[i] = Job{&c->pulses[i], &c->outputs[i]};
      g_err.clear();
      c->status = n ? simulate_impl(sc, &c->params, jobs.data(), n, nullptr, 0, stream,
                                    c->has_stats ? &c->stats : nullptr)
                    : HELIOS_OK;
      c->err = g_err;
    });
  } catch (...) {
    delete c;
    return fail(HELIOS_ERR_OUT_OF_MEMORY, "helios_simulate_batches_async: cannot start a worker");
  }
  *call = c;
  return HELIOS_OK;
}

helios_status helios_call_wait(helios_call c, helios_stats* stats) {
  g_err.clear();
  if (!c) return fail(HELIOS_ERR_INVALID_ARGUMENT, "call is NULL");
  c->worker.join();
  const helios_status st = c->status;
  if (stats) *stats = c->stats;
  if (st != HELIOS_OK) g_err = c->err;
  delete c;
  return st;
}

helios_status helios_simulate_survey(helios_scene sc, const helios_scanner_params* params,
                                     const helios_survey* survey, uint64_t first_pulse,
                                     uint64_t n_pulses, uint64_t pulse_index_base,
                                     const helios_outputs* outputs, helios_stream stream,
                                     helios_stats* stats) {
  g_err.clear();
  if (!survey) return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey is NULL");
  if (!outputs) return fail(HELIOS_ERR_INVALID_ARGUMENT, "outputs is NULL");
  helios_pulses p{};
  p.n_pulses = n_pulses;
  p.pulse_index_base = pulse_index_base;
  const Job j{&p, outputs};
  return simulate_impl(sc, params, &j, 1, survey, first_pulse, stream, stats);
}

helios_status helios_get_tuning(helios_tuning* out) {
  g_err.clear();
  if (!out) return fail(HELIOS_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = tuning_snapshot();
  return HELIOS_OK;
}

helios_status helios_set_tuning(const helios_tuning* t) {
  g_err.clear();
  if (!t) return fail(HELIOS_ERR_INVALID_ARGUMENT, "tuning is NULL");
  if (t->beam_prepass < -1 || t->beam_prepass > 1 || t->builder < 0 || t->builder > 1 ||
      t->lane_order < 0 || t->lane_order > 1 || t->pad_lanes < -1 || t->pad_lanes > 1 ||
      t->serialize < 0 || t->serialize > 1 || t->trace_spans < 0 || t->trace_spans > 1 ||
      (t->chunk_pulses != 0 && t->chunk_pulses < 1024))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "tuning value out of range");
  tuning_snapshot();  // seed from the environment first, then override
  std::lock_guard<std::mutex> g(g_tune_mu);
  g_tune = *t;
  helios::g_fault_alloc.store(t->fault_alloc_bytes, std::memory_order_relaxed);
  return HELIOS_OK;
}

}  // extern "C"
