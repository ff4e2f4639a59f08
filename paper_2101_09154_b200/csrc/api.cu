// api.cu -- the C ABI of libhelios.so (include/helios.h) and its host runtime:
// argument validation, scene ownership, the beam-pattern tables, scratch
// management (stream-ordered cudaMallocAsync), host<->device staging, pulse
// chunking so the K6->K7 subray records stay L2-resident, and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "internal.cuh"

using namespace helios;

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

  // Scratch cache: one device buffer per stream, grown on demand, reused by
  // later calls on the same stream, freed by helios_scene_destroy.
  struct Slot {
    cudaStream_t stream;
    char* ptr;
    size_t bytes;
    bool busy;
    cudaStream_t copy;  // non-blocking host->device copy stream for host staging (lazy)
    cudaStream_t copy_out;  // device->host copies (own stream: PCIe is full duplex)
    cudaStream_t wave;  // non-blocking stream for K7, overlapping K6 (lazy)
    cudaStream_t fit;   // non-blocking stream for the echo-width fits (lazy)
    cudaStream_t trace2;  // second K6 stream: odd chunks, so a chunk's K6 fills the SMs
                          // while the previous one's last wave drains (lazy)
    cudaStream_t beam[2];  // K6a streams (normal / high priority; HELIOS_BEAM_STREAM, lazy)
    uint64_t* pinned;   // 4 kSlots pinned words: per chunk slot (first, last) offsets of
                        // the packed waveform rows [0, 2 kSlots) and packed returns (lazy)
  };
  std::mutex mu;
  std::vector<Slot> slots;

  cudaError_t acquire(cudaStream_t s, size_t bytes, char** out, cudaStream_t* copy,
                      cudaStream_t* wave, uint64_t** pinned = nullptr,
                      cudaStream_t* fit = nullptr, cudaStream_t* trace2 = nullptr,
                      cudaStream_t* beam = nullptr, int beam_prio = 0) {
    std::lock_guard<std::mutex> g(mu);
    Slot* use = nullptr;
    for (Slot& sl : slots)
      if (sl.stream == s && !sl.busy) {
        use = &sl;
        break;
      }
    if (!use) {
      slots.push_back(Slot{s, nullptr, 0, false, nullptr, nullptr, nullptr, nullptr, nullptr,
                           {nullptr, nullptr}, nullptr});
      use = &slots.back();
    }
    if (use->bytes < bytes) {
      if (use->ptr) cudaFreeAsync(use->ptr, s);
      use->ptr = nullptr;
      use->bytes = 0;
      cudaError_t e = cudaMallocAsync((void**)&use->ptr, bytes ? bytes : 256, s);
      if (e != cudaSuccess) return e;
      use->bytes = bytes;
    }
    if (copy) {
      if (!use->copy) {
        cudaError_t e = cudaStreamCreateWithFlags(&use->copy, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      if (!use->copy_out) {
        cudaError_t e = cudaStreamCreateWithFlags(&use->copy_out, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      copy[0] = use->copy;
      copy[1] = use->copy_out;
    }
    if (!use->wave) {
      // K7 (and the packed-output scans, fits and copies it feeds) at high
      // priority: its blocks are scheduled ahead of the queued blocks of the
      // next chunks' K6 grids, so a chunk's outputs do not wait for them to
      // drain (HELIOS_WAVE_PRIO=0: normal priority, A/B)
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      int prio = hi;
      if (const char* v = getenv("HELIOS_WAVE_PRIO")) prio = atoi(v) ? hi : lo;
      cudaError_t e = cudaStreamCreateWithPriority(&use->wave, cudaStreamNonBlocking, prio);
      if (e != cudaSuccess) return e;
    }
    *wave = use->wave;
    if (fit) {
      if (!use->fit) {
        cudaError_t e = cudaStreamCreateWithFlags(&use->fit, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      *fit = use->fit;
    }
    if (trace2) {
      if (!use->trace2) {
        cudaError_t e = cudaStreamCreateWithFlags(&use->trace2, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
      }
      *trace2 = use->trace2;
    }
    if (beam) {
      cudaStream_t& b = use->beam[beam_prio ? 1 : 0];
      if (!b) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi: numerically lowest = highest
        cudaError_t e = cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, beam_prio ? hi : lo);
        if (e != cudaSuccess) return e;
      }
      *beam = b;
    }
    if (!use->pinned) {
      cudaError_t e = cudaMallocHost((void**)&use->pinned, 4 * kSlots * sizeof(uint64_t));
      if (e != cudaSuccess) return e;
    }
    use->busy = true;
    *out = use->ptr;
    if (pinned) *pinned = use->pinned;
    return cudaSuccess;
  }
  void release(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    for (Slot& sl : slots)
      if (sl.stream == s && sl.busy) {
        sl.busy = false;
        return;
      }
  }
  void free_slots() {
    std::lock_guard<std::mutex> g(mu);
    for (Slot& sl : slots) {
      cudaStreamSynchronize(sl.stream);
      if (sl.copy) {
        cudaStreamSynchronize(sl.copy);
        cudaStreamDestroy(sl.copy);
      }
      if (sl.copy_out) {
        cudaStreamSynchronize(sl.copy_out);
        cudaStreamDestroy(sl.copy_out);
      }
      if (sl.wave) {
        cudaStreamSynchronize(sl.wave);
        cudaStreamDestroy(sl.wave);
      }
      if (sl.fit) {
        cudaStreamSynchronize(sl.fit);
        cudaStreamDestroy(sl.fit);
      }
      if (sl.trace2) {
        cudaStreamSynchronize(sl.trace2);
        cudaStreamDestroy(sl.trace2);
      }
      for (cudaStream_t b : sl.beam)
        if (b) {
          cudaStreamSynchronize(b);
          cudaStreamDestroy(b);
        }
      cudaFree(sl.ptr);
      if (sl.pinned) cudaFreeHost(sl.pinned);
    }
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

#define TRY_CUDA(expr, what)                        \
  do {                                              \
    cudaError_t e_ = (expr);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

bool device_accessible(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Kernels may store straight into page-locked host memory mapped into the
// device address space (UVA: the same address).  Used for the packed
// outputs, whose per-chunk extent is only known on the device: the packing
// kernels write them over PCIe with coalesced 128-byte stores, and the host
// never has to learn a chunk's range before its copy.  Opt-in
// (HELIOS_DIRECT_HOST=1): measured slower than the staged copies (C2 e2e
// 7.9 -> 9.4 ms per 1 M pulses, profiles/r01s2_e2e.txt).
bool kernel_writable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) return true;
  const char* v = getenv("HELIOS_DIRECT_HOST");  // opt-in: measured slower than staging
  if (!v || !atoi(v)) return false;
  return at.type == cudaMemoryTypeHost && at.devicePointer == p;
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
  cudaError_t e = cudaMallocAsync((void**)dst, sizeof(T) * (count ? count : 1), s);
  if (e != cudaSuccess) return e;
  if (count) e = cudaMemcpyAsync(*dst, src, sizeof(T) * count, cudaMemcpyDefault, s);
  return e;
}

void free_scene(helios_scene sc, cudaStream_t s) {
  sc->free_slots();
  cudaFreeAsync(sc->d_xyz, s);
  cudaFreeAsync(sc->d_refl, s);
  cudaFreeAsync(sc->d_pad, s);
  cudaFreeAsync(sc->d_lut, s);
  cudaFreeAsync(sc->d_bricks, s);
  cudaFreeAsync(sc->bvh.tris, s);
  cudaFreeAsync(sc->bvh.nodes, s);
  cudaFreeAsync(sc->bvh.nodes4, s);
  cudaStreamSynchronize(s);
}

// one argument array: device-accessible as given, or staged through scratch
struct Staged {
  void* dev = nullptr;
  bool owned = false;
};

}  // namespace

extern "C" {

const char* helios_last_error(void) { return g_err.c_str(); }

const char* helios_version(void) { return "helios-b200 0.1 sm_100a"; }

helios_status helios_scene_create(const helios_scene_desc* desc, helios_stream stream,
                                  helios_scene* out) {
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
  {
    // keep stream-ordered allocations mapped across synchronisations
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, sc->device) == cudaSuccess) {
      uint64_t keep = std::numeric_limits<uint64_t>::max();
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
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
      if ((e = cudaMallocAsync((void**)&sc->d_bricks, nbr, s)) != cudaSuccess) break;
      if ((e = cudaMemsetAsync(sc->d_bricks, 0, nbr, s)) != cudaSuccess) break;
      k_bricks<<<(unsigned)std::min<uint64_t>((nvox + 255) / 256, 148ull * 32), 256, 0, s>>>(
          sc->d_pad, sc->nx, sc->ny, sc->nz, sc->nbx, sc->nby, sc->d_bricks);
      if ((e = cudaGetLastError()) != cudaSuccess) break;
    }
    if (desc->n_lut) {
      sc->n_lut = desc->n_lut;
      if ((e = copy_in(&sc->d_lut, desc->h_g_lut, desc->n_lut, s)) != cudaSuccess) break;
    }
    if ((e = cudaMallocAsync((void**)&d_bad, sizeof(unsigned), s)) != cudaSuccess) break;
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
  g_err.clear();
  if (!sc) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (sc->built) return HELIOS_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  char err[256] = {0};
  cudaError_t e = build_lbvh(sc->d_xyz, sc->d_refl, sc->n_tris, s, &sc->bvh, err, sizeof(err));
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation)
      return fail(HELIOS_ERR_OUT_OF_MEMORY, "helios_build_accel: %s", err);
    return fail(HELIOS_ERR_CUDA, "helios_build_accel: %s", err);
  }
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
  out->tri_bytes = (uint64_t)sc->n_tris * sizeof(TriRecord);
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

// helios_simulate (survey == nullptr: pulses from the caller's arrays) and
// helios_simulate_survey (pulses generated on the device, survey pulse
// first_pulse + i for pulse i of the call).
helios_status simulate_impl(helios_scene sc, const helios_scanner_params* params,
                            const helios_pulses* pulses, const helios_survey* survey,
                            uint64_t first_pulse, const helios_outputs* outputs,
                            helios_stream stream, helios_stats* stats) {
  g_err.clear();
  if (!sc) return fail(HELIOS_ERR_INVALID_ARGUMENT, "scene is NULL");
  if (!pulses || !outputs) return fail(HELIOS_ERR_INVALID_ARGUMENT, "pulses/outputs is NULL");
  if (survey) {
    const helios_status vs = validate_survey(survey);
    if (vs != HELIOS_OK) return vs;
  }
  Derived d;
  helios_status st = validate_params(params, &d);
  if (st != HELIOS_OK) return st;
  if (!sc->built) return fail(HELIOS_ERR_NOT_BUILT, "helios_build_accel has not been called");
  const bool counters = stats && stats->collect_counters;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->collect_counters = counters ? 1u : 0u;
  }
  const uint64_t n = pulses->n_pulses;
  if (n == 0) return HELIOS_OK;
  if (!survey && (!pulses->p_origin || !pulses->p_direction))
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_origin/p_direction is NULL");
  if (!outputs->p_n_returns || !outputs->p_wf_first_bin ||
      (!outputs->p_returns && !outputs->p_returns_packed))
    return fail(HELIOS_ERR_INVALID_ARGUMENT,
                "p_n_returns/p_wf_first_bin and p_returns or p_returns_packed must not be NULL");
  if (outputs->p_returns_packed && !outputs->p_return_offset)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_returns_packed needs p_return_offset");
  if (outputs->p_wf_compact && !outputs->p_wf_offset)
    return fail(HELIOS_ERR_INVALID_ARGUMENT, "p_wf_compact needs p_wf_offset");
  const uint32_t N = params->subray_count;
  const uint32_t R = params->max_returns;
  const cudaStream_t s = (cudaStream_t)stream;
  const bool want_offs = outputs->p_wf_offset != nullptr;
  const bool compact_staged = outputs->p_wf_compact && !kernel_writable(outputs->p_wf_compact);
  const bool packed = outputs->p_returns_packed != nullptr;
  const bool packed_staged = packed && !kernel_writable(outputs->p_returns_packed);

  // ---- host tables
  const std::vector<SubrayConst> tab = subray_table(N, params->divergence_rad, d.pt);
  std::vector<SubrayConst> lanes;  // K6's lane order of tab (set below)
  const double beta = params->divergence_rad;
  const double K = params->efficiency * params->receiver_diameter_m * params->receiver_diameter_m /
                   (4.0 * kPi * beta * beta);  // Eq. 7 (R14)
  WavePlan plan = plan_waveform(d.n_bins, N, d.taps);
  if (plan.warps == 0)
    return fail(HELIOS_ERR_CUDA, "helios_simulate: waveform kernel cannot be configured");

  // ---- argument arrays: device-accessible as given, or staged per chunk.
  // Per-pulse bytes of each array; chunk-local offsets are (b * per_pulse).
  struct Arr {
    const void* user;
    size_t per_pulse;
    bool in;      // host->device before the chunk's kernels, else device->host after
    bool staged;  // host memory: two chunk buffers in scratch (double buffering)
    size_t off[kSlots];
    bool gen;     // pulse array written by the on-device generator (survey mode), or
                  // any array the kernels need: internal slots when the user passes NULL
  };
  const bool gen = survey != nullptr;
  Arr arrs[] = {
      {gen ? (const void*)outputs->p_beam_origin : pulses->p_origin, 12, !gen, false, {0, 0}, gen},
      {gen ? (const void*)outputs->p_beam_direction : pulses->p_direction, 12, !gen, false,
       {0, 0}, gen},
      {gen ? (const void*)outputs->p_beam_time : pulses->p_time_s, 8, !gen, false, {0, 0}, gen},
      {outputs->p_n_returns, 1, false, false, {0, 0}, false},
      {outputs->p_returns, sizeof(helios_return) * R, false, false, {0, 0}, packed},
      {outputs->p_wf_first_bin, 8, false, false, {0, 0}, false},
      {outputs->p_waveform, 4ull * d.n_bins, false, false, {0, 0}, false},
      {outputs->p_subray_hits, sizeof(helios_subray_hit) * N, false, false, {0, 0}, false},
  };
  bool any_staged = compact_staged || packed_staged;
  bool gen_staged = false;  // a generated array is copied out to host memory
  for (Arr& a : arrs)
    if (a.user && !device_accessible(a.user)) {
      a.staged = any_staged = true;
      gen_staged |= a.gen;
    }

  // beam pre-pass K6a (packet traversal of a tree with internal nodes, beams of
  // >= 7 subrays); HELIOS_BEAM=0/1 forces, HELIOS_BEAM_K sets the hand-over size.
  // (An early version cost 6 % on C6's 1 622 triangles; with the later K6/K6a
  // changes it gains 19 % there: no scene-size threshold.)
  const bool beam_ok = N >= 7 && sc->n_tris > 0 && !ref_is_leaf(sc->bvh.root);
  bool beam = beam_ok;
  if (const char* v = getenv("HELIOS_BEAM")) beam = beam_ok && atoi(v) != 0;
  // Chunk size.  Without the pre-pass: the K6 -> K7 records (16 B per subray)
  // stay L2-resident.  With it, per-chunk tails (K6a's longest cone walks, K6's
  // last wave) dominate: few chunks of up to kBeamChunkSubrays subrays, balanced
  // (measured: profiles/r01s3_beam_ab.txt, C3 +33 %, C5 +13 %).
  uint64_t chunk = std::min<uint64_t>(n, std::max<uint64_t>(1024, (48ull << 20) / (16ull * N)));
  // (the same for voxel scenes, whose K6 and K7 run serially: C4 +7 %)
  if ((beam || sc->d_pad != nullptr) && n > 0) {
    constexpr uint64_t kBeamChunkSubrays = 64ull << 20;
    // at least 2 chunks (K7 of the first overlaps K6 of the second); measured
    // per 1M-pulse call: C5 1/2/3 chunks 7361/7214/7135, C3 2 best (9300),
    // C2 2 best (6703) -- profiles/r01s3_beam_ab.txt item 27
    uint64_t k = std::max<uint64_t>(2, (n * N + kBeamChunkSubrays - 1) / kBeamChunkSubrays);
    // host outputs: at least a few chunks, so copy-outs overlap later chunks'
    // kernels (HELIOS_STAGED_MIN_CHUNKS, default 4)
    if (any_staged) {
      uint64_t kmin = 4;
      if (const char* v = getenv("HELIOS_STAGED_MIN_CHUNKS")) kmin = std::max(1, atoi(v));
      k = std::max(k, kmin);
    }
    chunk = std::max(chunk, (n + k - 1) / k);
  }
  if (const char* v = getenv("HELIOS_CHUNK_PULSES"))  // experiments: chunk size override
    if (atoll(v) >= 1024) chunk = std::min<uint64_t>(n, (uint64_t)atoll(v));
  // chunk c covers pulses [cstart[c], cstart[c+1]).  Option: split the last
  // chunk so its K7, which nothing overlaps, is short (HELIOS_TAIL_FRAC of it
  // last; measured: C5 +2 %, C3 -6 % -> off by default)
  std::vector<uint64_t> cstart;
  for (uint64_t b = 0; b < n; b += chunk) cstart.push_back(b);
  // option: a short first chunk (HELIOS_HEAD_FRAC of a chunk), so the first
  // K6 starts after a short K6a (A/B)
  if (beam && cstart.size() >= 2) {
    double f = 0.0;
    if (const char* v = getenv("HELIOS_HEAD_FRAC")) f = atof(v);
    const uint64_t head = (uint64_t)(f * (double)chunk);
    if (f > 0.0 && head >= 4096 && head < chunk) cstart.insert(cstart.begin() + 1, head);
  }
  if (beam && cstart.size() >= 2) {
    double f = 0.0;
    if (const char* v = getenv("HELIOS_TAIL_FRAC")) f = atof(v);
    const uint64_t last = cstart.back(), len = n - last;
    const uint64_t tail = (uint64_t)(f * (double)len);
    if (f > 0.0 && tail >= 4096 && tail < len) cstart.push_back(n - tail);
  }
  cstart.push_back(n);
  const bool own_rec = outputs->p_subray_hits == nullptr;
  size_t total = 0;
  auto carve = [&](size_t bytes) {
    const size_t at = total;
    total += (bytes + 255) & ~(size_t)255;
    return at;
  };
  const size_t o_tab = carve(sizeof(SubrayConst) * N);
  const size_t o_ker = carve(sizeof(double) * d.taps);
  const size_t o_err = carve(sizeof(unsigned));
  const size_t o_cnt = carve(sizeof(unsigned long long) * 8);
  const size_t o_ws = carve(plan.scratch_bytes);
  // two record buffers: K6 of chunk c+1 overlaps K7 of chunk c
  size_t o_rec[kSlots];
  for (int k = 0; k < kSlots; ++k) o_rec[k] = carve(own_rec ? sizeof(helios_subray_hit) * N * chunk : 0);
  for (Arr& a : arrs)
    if (a.staged || (a.gen && !a.user))  // staged, or generated with no export
      for (int k = 0; k < kSlots; ++k) a.off[k] = carve(a.per_pulse * chunk);
  const size_t o_wp = carve(gen ? sizeof(double) * 3 * survey->n_waypoints : 0);
  size_t o_ent[kSlots];
  for (int k = 0; k < kSlots; ++k) o_ent[k] = carve(beam ? sizeof(int2) * kEntryStride * chunk : 0);
  size_t o_frm[kSlots];  // K6a's pulse frames (10 doubles per pulse)
  for (int k = 0; k < kSlots; ++k) o_frm[k] = carve(beam ? sizeof(double) * 10 * chunk : 0);
  // compact output: per-pulse lengths, call-wide offsets, scan temp, staging
  size_t scan_bytes = 0;
  if (want_offs)
    cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int)chunk, s);
  const size_t o_len = carve(want_offs ? sizeof(uint64_t) * chunk : 0);
  const size_t o_offs = carve(want_offs ? sizeof(uint64_t) * (n + 1) : 0);
  const size_t o_scan = carve(want_offs ? scan_bytes : 0);
  // echo-width jobs of one K7 launch (K7 and k_fit are serial on their stream)
  const uint32_t fit_stride = 2u * (uint32_t)std::ceil(3.0 * params->pulse_length_ns /
                                                        params->bin_width_ns) + 1u;
  const bool fit = params->fit_echo_width != 0;
  // two job buffers: k_fit(c) on its own stream overlaps K7(c+1) and K6(c+2)
  size_t o_fjob[kSlots], o_fy[kSlots], o_cst[kSlots], o_rst[kSlots];
  for (int k = 0; k < kSlots; ++k) o_fjob[k] = carve(fit ? sizeof(FitJob) * chunk * R : 0);
  for (int k = 0; k < kSlots; ++k)
    o_fy[k] = carve(fit ? sizeof(double) * fit_stride * chunk * R : 0);
  const size_t o_fcnt = carve(fit ? kSlots * sizeof(unsigned) : 0);
  for (int k = 0; k < kSlots; ++k) o_cst[k] = carve(compact_staged ? 4ull * d.n_bins * chunk : 0);
  // packed returns: lengths, call-wide offsets, scan temp (own: runs on K7's
  // stream concurrently with the waveform scan), staging
  const size_t o_rlen = carve(packed ? sizeof(uint64_t) * chunk : 0);
  const size_t o_roffs = carve(packed ? sizeof(uint64_t) * (n + 1) : 0);
  size_t rscan_bytes = 0;
  if (packed)
    cub::DeviceScan::InclusiveSum(nullptr, rscan_bytes, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int)chunk, s);
  const size_t o_rscan = carve(packed ? rscan_bytes : 0);
  for (int k = 0; k < kSlots; ++k)
    o_rst[k] = carve(packed_staged ? sizeof(helios_return) * R * chunk : 0);

  char* buf = nullptr;
  cudaStream_t cs = nullptr, co = nullptr, ws = nullptr, fs = nullptr;  // co: D2H copies
  cudaStream_t ts2 = nullptr;  // K6 of odd chunks
  cudaStream_t cpair[2] = {nullptr, nullptr};
  uint64_t* pin = nullptr;  // [slot][first, last] row offsets of a staged compact chunk
  // K6a stream: 0 = the chunk's trace stream (default, measured best), 1 = own
  // stream, 2 = own high-priority stream (HELIOS_BEAM_STREAM, A/B)
  int beam_stream = 0;
  if (const char* v = getenv("HELIOS_BEAM_STREAM")) beam_stream = atoi(v);
  cudaStream_t bs = nullptr;
  cudaError_t e = sc->acquire(s, total, &buf, any_staged ? cpair : nullptr, &ws, &pin,
                              fit ? &fs : nullptr, &ts2, beam && beam_stream ? &bs : nullptr,
                              beam_stream == 2);
  cs = cpair[0];
  co = cpair[1];
  if (e != cudaSuccess) return cuda_fail(e, "helios_simulate (scratch)");
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    cudaStreamSynchronize(ws);
    if (fs) cudaStreamSynchronize(fs);
    if (ts2) cudaStreamSynchronize(ts2);
    if (bs) cudaStreamSynchronize(bs);
    if (cs) cudaStreamSynchronize(cs);
    if (co) cudaStreamSynchronize(co);
    sc->release(s);
  };
  SubrayConst* d_tab = reinterpret_cast<SubrayConst*>(buf + o_tab);
  double* d_ker = reinterpret_cast<double*>(buf + o_ker);
  unsigned* d_err = reinterpret_cast<unsigned*>(buf + o_err);
  unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(buf + o_cnt);
  double* d_wscratch = reinterpret_cast<double*>(buf + o_ws);
  {
    // K6's lane order (HELIOS_SUBRAY_ORDER=0: the table order of R4, A/B)
    bool hil = true;
    if (const char* v = getenv("HELIOS_SUBRAY_ORDER")) hil = atoi(v) != 0;
    lanes = hil ? lane_order(tab) : tab;
  }
  e = cudaMemcpyAsync(d_tab, lanes.data(), sizeof(SubrayConst) * N, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_ker, d.kernel.data(), sizeof(double) * d.taps, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_err, 0, sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * 8, s);
  uint64_t* d_len = reinterpret_cast<uint64_t*>(buf + o_len);
  uint64_t* d_offs = reinterpret_cast<uint64_t*>(buf + o_offs);
  if (e == cudaSuccess && want_offs) e = cudaMemsetAsync(d_offs, 0, sizeof(uint64_t), s);
  uint64_t* d_rlen = reinterpret_cast<uint64_t*>(buf + o_rlen);
  uint64_t* d_roffs = reinterpret_cast<uint64_t*>(buf + o_roffs);
  if (e == cudaSuccess && packed) e = cudaMemsetAsync(d_roffs, 0, sizeof(uint64_t), s);
  if (e != cudaSuccess) {
    cleanup();
    return cuda_fail(e, "helios_simulate (setup)");
  }

  SurveyArgs sa{};
  if (gen && e == cudaSuccess) {
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
    if (e != cudaSuccess) {
      cleanup();
      return cuda_fail(e, "helios_simulate_survey (waypoints)");
    }
  }

  TraceArgs ta{};
  ta.tris = sc->bvh.tris;
  ta.nodes = sc->bvh.nodes;
  ta.root = sc->bvh.root;
  ta.nodes4 = sc->bvh.nodes4;
  ta.root4 = sc->bvh.root4;
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
  if (const char* v = getenv("HELIOS_BRICKS"))  // A/B switch (default on)
    if (!atoi(v)) ta.bricks = nullptr;
  ta.voxel_refl = sc->voxel_refl;
  ta.pad_max = sc->pad_max;
  ta.scale_alpha = sc->scale_alpha;
  ta.scale_shift = sc->scale_shift;
  ta.sub = d_tab;
  ta.N = N;
  {
    // pad a pulse to whole warps when that wastes <= 6 % of the lanes (91 -> 96):
    // every warp then walks one pulse's patch (HELIOS_PAD_LANES=0/1 forces)
    const uint32_t padded = (N + 31u) / 32u * 32u;
    bool pad = (padded - N) * 100u <= 6u * N;
    if (const char* v = getenv("HELIOS_PAD_LANES")) pad = atoi(v) != 0;
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
  {
    double smax = 0.0;
    for (const SubrayConst& t : tab) smax = std::max(smax, t.sin_t);
    ta.cone_sin = smax * (1.0 + 1e-9) + 1e-12;  // widened: covers the fp64 subray directions
    ta.beam_k = 8.0;  // measured (profiles/r01s3_beam_ab.txt)
    if (const char* v = getenv("HELIOS_BEAM_K")) ta.beam_k = atof(v);
    ta.entry_max = kEntryMax;
    ta.beam_budget = 1 << 30;
    if (const char* v = getenv("HELIOS_BEAM_BUDGET")) ta.beam_budget = std::max(1, atoi(v));
    if (const char* v = getenv("HELIOS_BEAM_ENTRIES"))
      ta.entry_max = std::max(2, std::min(kEntryMax, atoi(v)));
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
  wa.compact = compact_staged ? nullptr : outputs->p_wf_compact;
  wa.compact_staged = compact_staged ? 1 : 0;
  wa.capacity = outputs->p_wf_compact ? outputs->wf_compact_capacity : 0;
  wa.err_flag = d_err;
  wa.seed = params->seed;

  // per-kernel device time (CUDA events on each kernel's stream)
  std::vector<cudaEvent_t> ev_t, ev_w;
  auto mark = [&](std::vector<cudaEvent_t>& v, cudaStream_t st) {
    if (!stats) return;
    cudaEvent_t x;
    if (cudaEventCreate(&x) == cudaSuccess) {
      cudaEventRecord(x, st);
      v.push_back(x);
    }
  };
  // Stream graph per chunk c (slot = c % kSlots; "c-K" = the chunk that last used the slot):
  //   s  : [wait in_done]  [wait w_done(c-2)]  K6(c)  -> t_done
  //   ws : wait t_done  [wait out_done(c-2)]   K7(c)  -> w_done
  //   cs : wait w_done(c-1) -> H2D(c+1) -> in_done
  //   co : wait w_done(c) -> D2H(c) -> out_done   (own stream: PCIe is full duplex)
  // so K7(c) runs concurrently with K6(c+1) and the copies with both.
  cudaEvent_t in_done[kSlots] = {}, t_done[kSlots] = {}, w_done[kSlots] = {},
              out_done[kSlots] = {};
  cudaEvent_t off_done[kSlots] = {}, cd_done[kSlots] = {};  // packed rows: range known / drained
  cudaEvent_t k7_done[kSlots] = {};                         // fit: K7 done, jobs listed
  cudaEvent_t b_done[kSlots] = {};                          // K6a done: entry lists ready
  cudaEvent_t roff_done[kSlots] = {}, rd_done[kSlots] = {}; // packed returns: known / drained
  for (int k = 0; k < kSlots && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&t_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess && fit) e = cudaEventCreateWithFlags(&k7_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess && packed_staged) {
      e = cudaEventCreateWithFlags(&roff_done[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rd_done[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess && compact_staged) {
      e = cudaEventCreateWithFlags(&off_done[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cd_done[k], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&w_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess && bs) e = cudaEventCreateWithFlags(&b_done[k], cudaEventDisableTiming);
    if (e == cudaSuccess && any_staged) {
      e = cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming);
    }
  }
  // the copy stream must not start before the setup work on `s`
  if (any_staged && e == cudaSuccess) {
    e = cudaEventRecord(t_done[1], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, t_done[1], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(co, t_done[1], 0);
  }
  auto dev_ptr = [&](const Arr& a, int slot, uint64_t b) -> char* {
    if (a.gen && !a.user) return buf + a.off[slot];
    if (!a.user) return nullptr;
    if (a.staged) return buf + a.off[slot];
    return (char*)a.user + a.per_pulse * b;
  };
  auto copy_in = [&](uint64_t c, int slot) -> cudaError_t {
    const uint64_t b = cstart[c], m = cstart[c + 1] - b;
    for (const Arr& a : arrs)
      if (a.staged && a.in) {
        cudaError_t r = cudaMemcpyAsync(buf + a.off[slot], (const char*)a.user + a.per_pulse * b,
                                        a.per_pulse * m, cudaMemcpyHostToDevice, cs);
        if (r != cudaSuccess) return r;
      }
    return cudaEventRecord(in_done[slot], cs);
  };

  // HELIOS_TRACE_HOST=1: report the host's blocking time per call (stderr)
  const bool host_trace = getenv("HELIOS_TRACE_HOST") != nullptr;
  double host_wait_ms = 0.0;
  const double call_t0 = host_trace ? now_ms() : 0.0;
  // HELIOS_TRACE_HOST: device-side spans of the copy-out stream, the trace
  // streams and K7 (timing events; reported relative to a start event on s)
  std::vector<std::pair<char, cudaEvent_t>> tev;
  cudaEvent_t tev0 = nullptr;
  auto tmark = [&](char tag, cudaStream_t st) {
    if (!host_trace) return;
    cudaEvent_t x;
    if (cudaEventCreate(&x) == cudaSuccess) {
      cudaEventRecord(x, st);
      tev.emplace_back(tag, x);
    }
  };
  if (host_trace && cudaEventCreate(&tev0) == cudaSuccess) cudaEventRecord(tev0, s);
  // staged compact rows of chunk c: the host learns the chunk's offset range
  // from the pinned mirror (written on `s` right after the chunk's scan), then
  // queues the copy behind K7(c) on the copy stream.  Called one iteration
  // late, so the GPU never waits for the host.
  const uint64_t cap = outputs->wf_compact_capacity;
  auto drain_compact = [&](uint64_t c) -> cudaError_t {
    const int sl = (int)(c % kSlots);
    const double h0 = host_trace ? now_ms() : 0.0;
    cudaError_t r = cudaEventSynchronize(off_done[sl]);
    if (host_trace) host_wait_ms += now_ms() - h0;
    if (r != cudaSuccess) return r;
    const uint64_t first = pin[2 * sl], last = std::min(pin[2 * sl + 1], cap);
    r = cudaStreamWaitEvent(co, w_done[sl], 0);
    tmark('c', co);
    if (r == cudaSuccess && last > first)
      r = cudaMemcpyAsync(outputs->p_wf_compact + first, buf + o_cst[sl],
                          sizeof(float) * (last - first), cudaMemcpyDeviceToHost, co);
    tmark('C', co);
    if (r == cudaSuccess) r = cudaEventRecord(cd_done[sl], co);
    return r;
  };

  // staged fixed-size outputs of chunk c (counts, first bins, return slots,
  // dense rows, subray hits, beam export) -> host; out_done marks the slot free
  auto drain_fixed = [&](uint64_t c) -> cudaError_t {
    const int sl = (int)(c % kSlots);
    const uint64_t b = cstart[c], m = cstart[c + 1] - b;
    cudaError_t r = cudaStreamWaitEvent(co, w_done[sl], 0);
    tmark('f', co);
    for (const Arr& a : arrs)
      if (r == cudaSuccess && a.staged && !a.in)
        r = cudaMemcpyAsync((char*)a.user + a.per_pulse * b, buf + a.off[sl], a.per_pulse * m,
                            cudaMemcpyDeviceToHost, co);
    tmark('F', co);
    if (r == cudaSuccess) r = cudaEventRecord(out_done[sl], co);
    return r;
  };

  // staged packed returns of chunk c (same scheme as drain_compact)
  const uint64_t rcap = outputs->returns_capacity;
  auto drain_returns = [&](uint64_t c) -> cudaError_t {
    const int sl = (int)(c % kSlots);
    const double h0 = host_trace ? now_ms() : 0.0;
    cudaError_t r = cudaEventSynchronize(roff_done[sl]);
    if (host_trace) host_wait_ms += now_ms() - h0;
    if (r != cudaSuccess) return r;
    const uint64_t first = pin[2 * kSlots + 2 * sl],
                   last = std::min(pin[2 * kSlots + 2 * sl + 1], rcap);
    r = cudaStreamWaitEvent(co, w_done[sl], 0);
    if (r == cudaSuccess && last > first)
      r = cudaMemcpyAsync(outputs->p_returns_packed + first, buf + o_rst[sl],
                          sizeof(helios_return) * (last - first), cudaMemcpyDeviceToHost, co);
    if (r == cudaSuccess) r = cudaEventRecord(rd_done[sl], co);
    return r;
  };

  // traversal mode: warp-cooperative packets (default) or per-ray threads;
  // HELIOS_TRAVERSAL=ray selects the latter (A/B measurements).
  // traversal: 1 = packet over the binary tree (default, measured best),
  // 2 = packet over the 4-wide tree (needs HELIOS_BVH4=1 at build time),
  // 0 = per-ray threads; HELIOS_TRAVERSAL=packet2|packet4|ray
  int mode = 1;
  if (const char* v = getenv("HELIOS_TRAVERSAL")) {
    if (!strcmp(v, "ray")) mode = 0;
    else if (!strcmp(v, "packet4") && (sc->bvh.nodes4 || ref_is_leaf(sc->bvh.root))) mode = 2;
  }
  // K7 overlaps K6 on its own stream, except on voxel scenes: there K6 is
  // ALU-bound (fp64 DDA + Philox) and a concurrent K7 costs more than it
  // hides (measured: profiles/r01_overlap_ab.txt).  HELIOS_SERIAL=0/1 forces.
  bool serial = sc->d_pad != nullptr;
  if (const char* v = getenv("HELIOS_SERIAL")) serial = atoi(v) != 0;
  if (serial) ws = s;
  // K6 on two alternating streams (HELIOS_DUAL_TRACE=0/1 forces)
  bool dual_trace = !serial;
  if (const char* v = getenv("HELIOS_DUAL_TRACE")) dual_trace = atoi(v) != 0;
  if ((dual_trace || bs) && e == cudaSuccess) {
    // ts2 and bs must not start before the setup work on `s`
    e = cudaEventRecord(t_done[0], s);
    if (e == cudaSuccess && dual_trace) e = cudaStreamWaitEvent(ts2, t_done[0], 0);
    if (e == cudaSuccess && bs) e = cudaStreamWaitEvent(bs, t_done[0], 0);
  }
  if (ws != s) {
    // optional cap on K7's persistent grid while it shares the SMs with K6
    // (HELIOS_WAVE_BLOCKS_PER_SM; default: full grid, measured best)
    int bps = 0;
    if (const char* v = getenv("HELIOS_WAVE_BLOCKS_PER_SM")) bps = atoi(v);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (bps > 0) plan.grid_cap = (uint32_t)(sms * bps);
  }
  uint32_t launches = 0, trace_launches = 0;
  const uint64_t n_chunks = cstart.size() - 1;
  if (any_staged && e == cudaSuccess) e = copy_in(0, 0);
  for (uint64_t c = 0; c < n_chunks && e == cudaSuccess; ++c) {
    const uint64_t b = cstart[c];
    const uint64_t m = cstart[c + 1] - b;
    const int slot = (int)(c % kSlots);
    // K6 of odd chunks on the second trace stream (chunks are independent);
    // voxel scenes stay on one stream (measured: K6 is ALU-bound there)
    const cudaStream_t ts = (dual_trace && (c & 1)) ? ts2 : s;
    // with its own stream, K6a and the chunk's pulse generation only wait for
    // the chunk's inputs and for the slot's previous user (K7 of chunk c-K,
    // hence also its K6)
    const bool use_beam = beam && mode == 1;
    const cudaStream_t gs = (use_beam && bs) ? bs : ts;
    if (gs != ts) {
      if (any_staged) e = cudaStreamWaitEvent(bs, in_done[slot], 0);
      if (e == cudaSuccess && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(bs, w_done[slot], 0);
      if (e == cudaSuccess && any_staged && c >= (uint64_t)kSlots)
        e = cudaStreamWaitEvent(bs, out_done[slot], 0);
    }
    if (e == cudaSuccess && any_staged) e = cudaStreamWaitEvent(ts, in_done[slot], 0);
    if (e == cudaSuccess && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(ts, w_done[slot], 0);
    // K6 writes the staged subray-hit slot chunk c-K used: its copy-out (on the
    // D2H stream, not ordered behind this chunk's H2D) must be done
    if (e == cudaSuccess && any_staged && c >= (uint64_t)kSlots)
      e = cudaStreamWaitEvent(ts, out_done[slot], 0);
    // generated pulses of this chunk (into the slot chunk c-K used: its copy-out
    // must be done when the export is host memory)
    if (e == cudaSuccess && gen) {
      if (gen_staged && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(gs, out_done[slot], 0);
      if (e == cudaSuccess)
        e = launch_generate(sa, first_pulse + b, m, (float*)dev_ptr(arrs[0], slot, b),
                            (float*)dev_ptr(arrs[1], slot, b), (double*)dev_ptr(arrs[2], slot, b),
                            gs);
      ++launches;
    }
    if (e != cudaSuccess) break;
    ta.origin = (const float*)dev_ptr(arrs[0], slot, b);
    ta.direction = (const float*)dev_ptr(arrs[1], slot, b);
    ta.n_pulses = m;
    ta.pulse_base = pulses->pulse_index_base + b;
    ta.out = own_rec ? reinterpret_cast<helios_subray_hit*>(buf + o_rec[slot])
                     : (helios_subray_hit*)dev_ptr(arrs[7], slot, b);
    ta.entries = nullptr;
    ta.frames = nullptr;
    if (use_beam) {
      ta.entries = reinterpret_cast<int2*>(buf + o_ent[slot]);
      ta.frames = reinterpret_cast<double*>(buf + o_frm[slot]);
      mark(ev_t, gs);
      tmark('b', gs);
      if (e == cudaSuccess) e = launch_beam(ta, counters, gs);
      tmark('B', gs);
      ++launches;
      // measurement only: HELIOS_BEAM_REPEAT=k launches K6a k extra times (its
      // marginal cost in the pipeline = step time delta / k)
      if (const char* v = getenv("HELIOS_BEAM_REPEAT"))
        for (int r = 0; r < atoi(v) && e == cudaSuccess; ++r) e = launch_beam(ta, false, gs);
      mark(ev_t, gs);
      if (gs != ts) {
        if (e == cudaSuccess) e = cudaEventRecord(b_done[slot], bs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(ts, b_done[slot], 0);
      }
    }
    mark(ev_t, ts);
    tmark('t', ts);
    if (e == cudaSuccess) e = launch_trace(ta, counters, mode, ts);
    tmark('T', ts);
    ++trace_launches;
    mark(ev_t, ts);
    if (e == cudaSuccess) e = cudaEventRecord(t_done[slot], ts);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ws, t_done[slot], 0);
    if (e == cudaSuccess && any_staged && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(ws, out_done[slot], 0);
    if (e == cudaSuccess && compact_staged && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(ws, cd_done[slot], 0);
    if (e == cudaSuccess && want_offs) {
      // packed rows: lengths -> inclusive scan into offs[b+1 ..] -> + offs[b]
      // (previous chunks), on K7's stream so the next chunk's K6 never waits
      e = launch_support(ta.out, N, m, d.n_bins, d.taps, params->bin_width_ns, d_len, ws);
      size_t tb = scan_bytes;
      if (e == cudaSuccess)
        e = cub::DeviceScan::InclusiveSum(buf + o_scan, tb, d_len, d_offs + b + 1, (int)m, ws);
      if (e == cudaSuccess) e = launch_add_carry(d_offs + b, m, ws);
      launches += 3;
      if (e == cudaSuccess && compact_staged) {
        e = cudaMemcpyAsync(pin + 2 * slot, d_offs + b, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            ws);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(pin + 2 * slot + 1, d_offs + b + m, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, ws);
        if (e == cudaSuccess) e = cudaEventRecord(off_done[slot], ws);
      }
    }
    if (e != cudaSuccess) break;
    wa.rec = ta.out;
    wa.n_pulses = m;
    wa.pulse_base = ta.pulse_base;
    wa.time_s = (const double*)dev_ptr(arrs[2], slot, b);
    wa.n_returns = (uint8_t*)dev_ptr(arrs[3], slot, b);
    wa.returns = (helios_return*)dev_ptr(arrs[4], slot, b);
    wa.first_bin = (int64_t*)dev_ptr(arrs[5], slot, b);
    wa.waveform = (float*)dev_ptr(arrs[6], slot, b);
    wa.offs = want_offs ? d_offs + b : nullptr;
    if (compact_staged) wa.compact = reinterpret_cast<float*>(buf + o_cst[slot]);
    if (fit) {
      wa.fit_jobs = reinterpret_cast<FitJob*>(buf + o_fjob[slot]);
      wa.fit_y = reinterpret_cast<double*>(buf + o_fy[slot]);
      wa.fit_count = reinterpret_cast<unsigned*>(buf + o_fcnt) + slot;
      // the slot's jobs of chunk c-2 must be fitted before they are overwritten
      if (c >= (uint64_t)kSlots && ws != s) e = cudaStreamWaitEvent(ws, w_done[slot], 0);
      if (e == cudaSuccess) e = cudaMemsetAsync(wa.fit_count, 0, sizeof(unsigned), ws);
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
    // the stream that finishes the chunk's returns: fits (own stream) or K7's
    cudaStream_t post = ws;
    if (e == cudaSuccess && fit) {
      // echo-width fits on their own stream (their tail overlaps later chunks);
      // the chunk's outputs are complete once they are done
      cudaStream_t f = ws == s ? s : fs;
      if (f != ws) e = cudaEventRecord(k7_done[slot], ws);
      if (e == cudaSuccess && f != ws) e = cudaStreamWaitEvent(f, k7_done[slot], 0);
      if (e == cudaSuccess) e = launch_fit(wa, f);
      ++launches;
      post = f;
    }
    if (e == cudaSuccess && packed) {
      // packed returns: scan of the counts, copy of the used slots
      if (packed_staged && c >= (uint64_t)kSlots) e = cudaStreamWaitEvent(post, rd_done[slot], 0);
      helios_return* dst = packed_staged ? reinterpret_cast<helios_return*>(buf + o_rst[slot])
                                         : outputs->p_returns_packed;
      if (e == cudaSuccess)
        e = launch_pack_returns(wa.returns, wa.n_returns, m, R, d_rlen, d_roffs + b,
                                buf + o_rscan, rscan_bytes, dst, packed_staged ? 1 : 0, rcap,
                                post);
      launches += 4;
      if (e == cudaSuccess && packed_staged) {
        e = cudaMemcpyAsync(pin + 2 * kSlots + 2 * slot, d_roffs + b, sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, post);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(pin + 2 * kSlots + 2 * slot + 1, d_roffs + b + m, sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, post);
        if (e == cudaSuccess) e = cudaEventRecord(roff_done[slot], post);
      }
    }
    if (e == cudaSuccess) e = cudaEventRecord(w_done[slot], post);
    launches += 2;
    // packed copy-outs run kSlots-1 chunks behind, so the host never blocks on
    // a chunk whose K7 may still be queued behind the K6 it just enqueued
    constexpr uint64_t kLag = kSlots - 1;
    // (the fixed-size staged outputs too: all copy-outs of a chunk leave in
    // one go, in chunk order, so none queues behind a later chunk's K7)
    if (e == cudaSuccess && compact_staged && c >= kLag) e = drain_compact(c - kLag);
    if (e == cudaSuccess && packed_staged && c >= kLag) e = drain_returns(c - kLag);
    if (e == cudaSuccess && any_staged && c >= kLag) e = drain_fixed(c - kLag);
    if (e != cudaSuccess || !any_staged) continue;
    // prefetch the next chunk's inputs into the other slot once chunk c-1's
    // kernels (K6 reads origin/direction, K7 reads time) are done with it
    if (c + 1 < n_chunks) {
      const int nslot = (int)((c + 1) % kSlots);
      if (c + 1 >= (uint64_t)kSlots) e = cudaStreamWaitEvent(cs, w_done[nslot], 0);
      if (e == cudaSuccess) e = copy_in(c + 1, nslot);
    }
  }
  for (uint64_t c = n_chunks > (uint64_t)(kSlots - 1) ? n_chunks - (kSlots - 1) : 0;
       c < n_chunks && e == cudaSuccess; ++c) {
    if (compact_staged) e = drain_compact(c);
    if (e == cudaSuccess && packed_staged) e = drain_returns(c);
    if (e == cudaSuccess && any_staged) e = drain_fixed(c);
  }
  // call-wide offsets to the caller (device or host memory)
  if (e == cudaSuccess && want_offs) {
    for (int k = 0; k < kSlots && (uint64_t)k < n_chunks && e == cudaSuccess && ws != s; ++k)
      e = cudaStreamWaitEvent(s, w_done[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(outputs->p_wf_offset, d_offs, sizeof(uint64_t) * (n + 1),
                          cudaMemcpyDefault, s);
  }
  if (e == cudaSuccess && packed) {
    for (int k = 0; k < kSlots && (uint64_t)k < n_chunks && e == cudaSuccess; ++k)
      e = cudaStreamWaitEvent(s, w_done[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(outputs->p_return_offset, d_roffs, sizeof(uint64_t) * (n + 1),
                          cudaMemcpyDefault, s);
  }
  // join: the caller's stream is ordered after every kernel of this call
  if (e == cudaSuccess && ws != s && n_chunks > 0)
    for (int k = 0; k < kSlots && (uint64_t)k < n_chunks && e == cudaSuccess; ++k)
      e = cudaStreamWaitEvent(s, w_done[k], 0);
  unsigned herr = 0;
  unsigned long long hcnt[8] = {0};
  uint64_t htotal = 0, hrtotal = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && want_offs)
    e = cudaMemcpyAsync(&htotal, d_offs + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && packed)
    e = cudaMemcpyAsync(&hrtotal, d_roffs + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && counters)
    e = cudaMemcpyAsync(hcnt, d_cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && cs) e = cudaStreamSynchronize(cs);
  if (e == cudaSuccess && co) e = cudaStreamSynchronize(co);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ws);
  if (e == cudaSuccess && fs) e = cudaStreamSynchronize(fs);
  if (host_trace && tev0) {
    std::string line;
    for (auto& pr : tev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev0, pr.second);
      char b[32];
      snprintf(b, sizeof b, " %c%.2f", pr.first, ms);
      line += b;
      cudaEventDestroy(pr.second);
    }
    cudaEventDestroy(tev0);
    fprintf(stderr, "helios_simulate spans (ms from call start; b/B K6a, t/T K6, w/W K7, f/F fixed copy-out, c/C rows copy-out):%s\n", line.c_str());
  }
  if (host_trace)
    fprintf(stderr, "helios_simulate: %llu pulses, %llu chunks, host %.3f ms, blocked in drains %.3f ms\n",
            (unsigned long long)n, (unsigned long long)n_chunks, now_ms() - call_t0, host_wait_ms);
  double t_trace = 0.0, t_wave = 0.0;
  for (size_t i = 0; i + 1 < ev_t.size(); i += 2) {
    float a = 0.f;
    if (cudaEventElapsedTime(&a, ev_t[i], ev_t[i + 1]) == cudaSuccess) t_trace += a;
  }
  for (size_t i = 0; i + 1 < ev_w.size(); i += 2) {
    float a = 0.f;
    if (cudaEventElapsedTime(&a, ev_w[i], ev_w[i + 1]) == cudaSuccess) t_wave += a;
  }
  for (cudaEvent_t x : ev_t) cudaEventDestroy(x);
  for (cudaEvent_t x : ev_w) cudaEventDestroy(x);
  for (int k = 0; k < kSlots; ++k) {
    if (in_done[k]) cudaEventDestroy(in_done[k]);
    if (t_done[k]) cudaEventDestroy(t_done[k]);
    if (w_done[k]) cudaEventDestroy(w_done[k]);
    if (out_done[k]) cudaEventDestroy(out_done[k]);
    if (off_done[k]) cudaEventDestroy(off_done[k]);
    if (cd_done[k]) cudaEventDestroy(cd_done[k]);
    if (roff_done[k]) cudaEventDestroy(roff_done[k]);
    if (rd_done[k]) cudaEventDestroy(rd_done[k]);
    if (k7_done[k]) cudaEventDestroy(k7_done[k]);
    if (b_done[k]) cudaEventDestroy(b_done[k]);
  }
  cudaGetLastError();
  cleanup();
  if (e != cudaSuccess) return cuda_fail(e, "helios_simulate");
  if (stats) {
    stats->pulses = n;
    stats->subrays = n * N;
    stats->kernel_launches = launches;
    stats->trace_launches = trace_launches;
    stats->beam_nodes = hcnt[7];
    stats->node_bytes = mode == 2 ? (uint32_t)sizeof(Node4) : (uint32_t)sizeof(Node);
    stats->trace_ms = t_trace;
    stats->waveform_ms = t_wave;
    stats->nodes_visited = hcnt[0];
    stats->tris_tested = hcnt[1];
    stats->voxel_steps = hcnt[2];
    stats->voxel_returns = hcnt[3];
    stats->fp64_tests = hcnt[6];
    stats->subray_hits = hcnt[4];
    stats->returns = hcnt[5];
  }
  if (herr & 4u) return fail(HELIOS_ERR_CUDA, "internal: compact row length mismatch");
  if (herr & 1u) return fail(HELIOS_ERR_INVALID_ARGUMENT, "a pulse direction has zero length");
  if (packed && hrtotal > outputs->returns_capacity)
    return fail(HELIOS_ERR_CAPACITY, "packed returns need %llu slots, capacity %llu",
                (unsigned long long)hrtotal, (unsigned long long)outputs->returns_capacity);
  if (outputs->p_wf_compact && htotal > outputs->wf_compact_capacity)
    return fail(HELIOS_ERR_CAPACITY, "compact waveform needs %llu floats, capacity %llu",
                (unsigned long long)htotal, (unsigned long long)outputs->wf_compact_capacity);
  return HELIOS_OK;
}

}  // namespace

extern "C" {

helios_status helios_simulate(helios_scene sc, const helios_scanner_params* params,
                              const helios_pulses* pulses, const helios_outputs* outputs,
                              helios_stream stream, helios_stats* stats) {
  return simulate_impl(sc, params, pulses, nullptr, 0, outputs, stream, stats);
}

helios_status helios_simulate_survey(helios_scene sc, const helios_scanner_params* params,
                                     const helios_survey* survey, uint64_t first_pulse,
                                     uint64_t n_pulses, uint64_t pulse_index_base,
                                     const helios_outputs* outputs, helios_stream stream,
                                     helios_stats* stats) {
  g_err.clear();
  if (!survey) return fail(HELIOS_ERR_INVALID_ARGUMENT, "survey is NULL");
  helios_pulses p{};
  p.n_pulses = n_pulses;
  p.pulse_index_base = pulse_index_base;
  return simulate_impl(sc, params, &p, survey, first_pulse, outputs, stream, stats);
}

}  // extern "C"

