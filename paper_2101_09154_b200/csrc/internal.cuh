// internal.cuh -- shared declarations of libhelios (not part of the ABI).
//
// Layout in HBM (DESIGN.md s.6):
//   triangles  : TriRecord[n_tris] in LBVH leaf order, 48 B = 3 x float4
//                { v0.xyz, bits(original id) } { v1.xyz, reflectance } { v2.xyz, 0 }
//   filter recs: TriRecord[n_tris], same order, 48 B: { v0.xyz, A B } { e1.xyz, A }
//                { e2.xyz, B } (fp32 edges, A = |e1|_1, B = |e2|_1): the fp32
//                Moller-Trumbore filter reads only these, the fp64 test the above
//   nodes      : Node[n_tris - 1] child-pair nodes, 64 B = 4 x float4
//                { c0.lo.x, c0.hi.x, c0.lo.y, c0.hi.y }
//                { c1.lo.x, c1.hi.x, c1.lo.y, c1.hi.y }
//                { c0.lo.z, c0.hi.z, c1.lo.z, c1.hi.z }
//                { bits(ref0), bits(ref1), 0, 0 }
//                ref >= 0: internal node index; ref < 0: leaf, see leaf_ref().
//   voxel grid : PAD float[nz][ny][nx] (x fastest).
//   subray rec : helios_subray_hit[n_pulses][N] (16 B), K6 -> K7.
#pragma once
#include <assert.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/helios.h"
#include "../../include/helios_util.h"

namespace helios {

// NVTX ranges (header-only NVTX3: no cost unless a profiler is attached) around
// the ABI calls, the build phases and each chunk's kernel launches, so a timeline shows K6a / K6 /
// K7 / copies per chunk under the call that issued them
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Device-side invariant checks of the debug build (build.py --debug ->
// libhelios_debug.so, -DHELIOS_DEBUG): a failed check traps the kernel
// (cudaErrorAssert); compiled out of the release library.
#ifdef HELIOS_DEBUG
#define HELIOS_DASSERT(x) assert(x)
#else
#define HELIOS_DASSERT(x) ((void)0)
#endif

// stream-ordered allocation from the library's private pool (api.cu)
cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t s);

constexpr int kMaxSubrays = 512;      // >= largest supported count (279)
constexpr int kStackSize = 64;        // LBVH depth bound (checked at build)
#ifndef HELIOS_LEAF_MAX
#define HELIOS_LEAF_MAX 2  // measured best (profiles/r01_leaf_ab.txt)
#endif
constexpr int kLeafMax = HELIOS_LEAF_MAX;  // triangles per collapsed leaf (<= 8)
constexpr int kMortonBits = 21;       // per axis (63-bit codes)
constexpr int kMaxLut = 4096;
constexpr int kBrickShift = 2;        // 4^3-voxel bricks for empty-space skipping
#ifndef HELIOS_SLOTS
#define HELIOS_SLOTS 3
#endif
constexpr int kSlots = HELIOS_SLOTS;  // chunk buffers in flight (records, staging, jobs)
constexpr int kMaxTaps = 8192;        // L_p bound (validated)
// beam entry lists (K6a k_beam -> K6): per pulse one 256-B row of int2,
// row[0].x = entry count, row[1 .. count] = (subtree ref, bits of a float lower
// bound on every subray's entry distance into its box), near-first order
constexpr int kEntryStride = 32;
constexpr int kEntryMax = kEntryStride - 1;  // list cap of K6a
static_assert(kEntryMax <= 32, "K6a keeps its emit flags in 32 bits");
constexpr double kC = 299792458.0;    // m/s
constexpr double kPi = 3.14159265358979323846;

struct __align__(16) TriRecord {
  float4 a, b, c;
};
struct __align__(16) Node {
  float4 xy0, xy1, z01, ref;
};
// K6 -> K7 waveform record, 8 B per subray: the absolute bin
// k_s = floor(2 R_s / (c Delta)) (R8, R9; -1 = no event) and the fp32
// amplitude A_s (Eq. 7).  The prim ids travel in a separate uint32 array that
// K7 reads only to attribute a return (R13).
struct __align__(8) WaveRec {
  int32_t k;
  float amp;
};

// Absolute bin k_s = floor(2 R / c / (Delta 1e-9)) -- the oracle's two
// correctly rounded divisions, bit for bit -- at the cost of one multiply:
// q = 2R * inv_bin (inv_bin = 1 / (c Delta 1e-9)) is within a few ulp of the
// same exact quotient, so its floor is the oracle's whenever q is farther than
// 1e-13 q from an integer; only then (never, in practice) the divisions run.
__device__ __forceinline__ long long bin_of(double range_m, double delta_ns, double inv_bin) {
  const double q = 2.0 * range_m * inv_bin;
  const double f = floor(q);
  if (q - f > 1e-13 * q && (f + 1.0) - q > 1e-13 * q) return (long long)f;
  return (long long)floor(2.0 * range_m / 299792458.0 / (delta_ns * 1e-9));
}

// leaf reference: bit 31 set, bits [3,31) = first triangle, bits [0,3) = count-1
__host__ __device__ inline int32_t leaf_ref(uint32_t first, uint32_t count) {
  return (int32_t)(0x80000000u | (first << 3) | (count - 1u));
}
__host__ __device__ inline bool ref_is_leaf(int32_t r) { return r < 0; }
__host__ __device__ inline uint32_t leaf_first(int32_t r) {
  return ((uint32_t)r & 0x7FFFFFFFu) >> 3;
}
__host__ __device__ inline uint32_t leaf_count(int32_t r) { return ((uint32_t)r & 7u) + 1u; }
constexpr int32_t kEmptyRef = 0x7FFFFFFF;  // never-hit child (box is inverted)

// Per-subray constants of the beam pattern (R2, R4, R5), fp64.
struct SubrayConst {
  double cos_t;     // cos(theta_i)
  double sin_t;     // sin(theta_i)  (also r = R sin theta_i)
  double cos_p;     // cos(phi)
  double sin_p;     // sin(phi)
  double w_far;     // far-field weight exp(-2 sin^2 theta / tan^2 beta) (R5)
  uint32_t index;   // the subray's index s (R4 order: Philox counter word, output slot)
  uint32_t pad32_;
  double pad_[2];
};
static_assert(sizeof(SubrayConst) == 64, "SubrayConst layout");

// Everything a trace launch needs, passed by value (kernel parameter space).
struct TraceArgs {
  const TriRecord* tris;
  const TriRecord* filt;   // filter records (BuildResult::filt)
  const Node* nodes;
  int32_t root;          // root node ref (internal index or leaf ref)
  uint32_t n_tris;
  const float* pad;      // voxel grid or nullptr
  uint32_t nx, ny, nz;
  double gx0, gy0, gz0, vs;
  const float* g_lut;
  uint32_t n_lut;
  const uint8_t* bricks; // [nbz][nby][nbx] 1 = the 4^3 brick holds a voxel with PAD > 0
  uint32_t nbx, nby;
  uint32_t voxel_mode;   // HELIOS_VOXEL_* (R31)
  double voxel_refl, pad_max, scale_alpha;
  uint32_t scale_shift;
  const SubrayConst* sub;
  uint32_t N;            // subrays per pulse
  uint32_t lanes;        // K6 threads per pulse: N, or N padded to whole warps
  const float* origin;   // [n][3]
  const float* direction;
  uint64_t n_pulses;
  uint64_t pulse_base;
  uint64_t seed;
  double K;              // lambda alpha^2 / (4 pi beta^2)    (Eq. 7)
  double I0;
  int eq2;               // 1: Eq. 2 beam width; 0: far field
  double w0, lambda_m, R0;
  WaveRec* wrec;          // [n][N] K6 -> K7 records (k_s, A_s)
  uint32_t* prim;         // [n][N] prim id per subray (UINT32_MAX: no event)
  helios_subray_hit* out; // [n][N] optional export, or nullptr
  double delta_ns;        // bin width Delta (k_s in K6)
  double inv_bin;         // 1 / (c Delta 1e-9)
  unsigned int* err_flag;  // set on zero-length direction
  unsigned long long* counters;  // instrumented variant: [nodes, tris, voxel steps, voxel returns]
  // beam pre-pass (K6a): per-pulse cone over all subrays; nullptr = K6 starts at the root
  int2* entries;         // [n_pulses][kEntryStride] (K6a writes, K6 reads)
  double* frames;        // [n_pulses][10] pulse frames d, u, v + valid flag (K6a writes) or nullptr
  double cone_sin;       // sin of the (widened) cone half-angle: max_i sin(theta_i)
  double beam_k;         // a node is handed to K6 once extent <= beam_k * cone radius
};

// One echo-width fit job (R28), appended by K7, solved by k_fit.
struct FitJob {
  uint32_t slot;  // return slot index p * max_returns + j within the launch
  int16_t lo;     // first window bin relative to the peak bin (<= 0)
  uint16_t n;     // window bins
  double peak;    // W[k] (LM start amplitude)
};

struct WaveArgs {
  const WaveRec* rec;            // [n][N] (k_s, A_s) from K6
  const uint32_t* prim;          // [n][N] prim ids (attribution only)
  uint32_t N;
  uint64_t n_pulses;
  uint32_t n_bins;
  uint32_t taps;                 // L_p
  uint32_t jstar;                // argmax of the binned pulse (R12)
  const double* kernel;          // p[j], j < taps
  double delta_ns;               // bin width Delta
  float thr;
  uint32_t max_returns;
  const double* time_s;          // may be nullptr
  uint8_t* n_returns;
  helios_return* returns;
  int64_t* first_bin;
  float* waveform;               // may be nullptr
  unsigned long long* counters;  // [subray hits, returns] or nullptr
  uint32_t fit;                  // 1: Gaussian echo-width fit per return (R28)
  FitJob* fit_jobs;              // [n_pulses * max_returns] job list (fit only)
  double* fit_y;                 // [n_pulses * max_returns][fit_stride] window values
  uint32_t fit_stride;           // 2 fit_half + 1
  unsigned* fit_count;           // jobs appended (zeroed before each launch)
  int fit_half;                  // window half-width ceil(3 pulse_length / Delta) bins
  double fit_s0;                 // LM start sigma = pulse_length / (2 sqrt(2 ln 2)) ns
  float* compact;                // packed support rows or nullptr
  const uint64_t* offs;          // [n_pulses + 1] call-relative row offsets (nullptr: none)
  int compact_staged;            // 1: `compact` is a chunk staging slot based at offs[0]
  uint64_t capacity;             // floats available in the caller's compact buffer
  unsigned int* err_flag;        // bit 2: internal length mismatch
  double noise_sd;               // ranging error sigma (R29), 0 = none
  uint64_t seed;                 // Philox key
  uint64_t pulse_base;           // global id of pulse 0 of this launch
  uint32_t* wide_list;           // [n_pulses] pulses deferred to the wide pass (support > kWCap)
  unsigned* wide_count;          // their count (zeroed by launch_waveform)
};

// On-device pulse generation (survey.cu; NEXT f2, R30).  Plain values copied
// from helios_survey; waypoints in device memory.
struct SurveyArgs {
  const double* waypoints;  // [n_waypoints][3] device
  uint32_t n_waypoints;
  uint32_t deflector;       // helios_deflector
  double speed;
  double mount[9];
  double offset[3];
  double head;              // head rotation rad/s
  double prf, t0, f, A;
  uint32_t n_fibres;
};
cudaError_t launch_generate(const SurveyArgs& a, uint64_t first, uint64_t n, float* origin,
                            float* direction, double* time, cudaStream_t s);

// launchers (trace.cu / waveform.cu)
cudaError_t launch_trace(const TraceArgs& a, bool instrumented, cudaStream_t s);
// K6a: per-pulse beam entry lists into a.entries (before launch_trace, same stream)
cudaError_t launch_beam(const TraceArgs& a, bool instrumented, cudaStream_t s);

struct WavePlan {
  int warps;            // warps per block (0 = does not fit)
  size_t smem;          // dynamic shared memory per block
  uint32_t grid;        // persistent grid (SMs x occupancy)
  size_t scratch_bytes; // per-warp global rows of the wide pass (0: rows in shared memory)
  uint32_t wide_grid;   // blocks of the wide pass
  int wide_warps;       // warps per block of the wide pass
  size_t wide_smem;     // its dynamic shared memory per block
  uint32_t grid_cap;    // 0 = full persistent grid; else max blocks (overlap with K6)
};
WavePlan plan_waveform(uint32_t n_bins, uint32_t N, uint32_t taps);
// support length len_p of every pulse's waveform (for the compact output)
cudaError_t launch_support(const WaveRec* rec, uint32_t N, uint64_t n_pulses, uint32_t n_bins,
                           uint32_t taps, uint64_t* len, cudaStream_t s);
// echo-width fits of the jobs one K7 launch appended (after it; any stream)
cudaError_t launch_fit(const WaveArgs& a, cudaStream_t s);
// ranging error on the returns of one launch (after K7, same stream)
cudaError_t launch_range_noise(const WaveArgs& a, cudaStream_t s);
// packed returns of one launch: len = n_returns, inclusive scan into
// offs[1..m] seeded with the carry offs[0], copy of the used slots to dst
// (staged: dst is a chunk buffer based at offs[0]); entries at or past
// `capacity` are skipped
cudaError_t launch_pack_returns(const helios_return* slots, const uint8_t* nr, uint64_t m,
                                uint32_t R, uint64_t* len, uint64_t* offs, void* scan_temp,
                                size_t scan_bytes, helios_return* dst, int staged,
                                uint64_t capacity, cudaStream_t s);
bool waveform_fits(uint32_t n_bins, uint32_t N, uint32_t taps);
cudaError_t launch_waveform(const WaveArgs& a, const WavePlan& pl, double* scratch,
                            cudaStream_t s);

// prefix sums and the radix sort (sort_scan.cu): temp sizes, then the calls
// (stream-ordered; in == out allowed for the scans)
size_t scan_temp_bytes(uint64_t n, size_t elem);
// seed (device, nullable): *seed is added to every output (chunk carry)
cudaError_t scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, bool inclusive, void* temp,
                     size_t temp_bytes, cudaStream_t s, const uint64_t* seed = nullptr);
cudaError_t scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, bool inclusive, void* temp,
                     size_t temp_bytes, cudaStream_t s);
size_t sort_temp_bytes(uint64_t n);
// stable LSD radix sort of (keys, vals) in place by the low `bits` bits of the keys
cudaError_t sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int bits, void* temp,
                           size_t temp_bytes, cudaStream_t s);

// LBVH build (lbvh.cu)
struct BuildResult {
  TriRecord* tris;   // device, leaf order
  TriRecord* filt;   // device, leaf order: K6's fp32 filter record of each triangle
                     // {v0.xyz, |e1|_1 |e2|_1} {e1.xyz, |e1|_1} {e2.xyz, |e2|_1},
                     // e1 = v1 - v0, e2 = v2 - v0 rounded to fp32 (the values the
                     // filter used to recompute per test, bit for bit)
  Node* nodes;       // device
  uint32_t n_nodes;
  int32_t root;
  uint32_t max_depth;
  float ms;
};
// builder: 0 = PLOC over Morton order (default), 1 = Karras LBVH
cudaError_t build_lbvh(const float* d_tri_xyz, const float* d_refl, uint32_t n, int builder,
                       cudaStream_t s, BuildResult* out, char* err, size_t err_len);

}  // namespace helios
