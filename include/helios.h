/*
 * helios.h -- C ABI of libhelios.so, the B200 (sm_100a) hot path of
 * HELIOS++-style virtual laser scanning (Winiwarter et al., arXiv 2101.09154).
 *
 * Citations: "P:n" = line n of the paper text, with the section /
 * equation named; "R<k>" = reading k of DESIGN.md s.3 (where the paper is
 * silent, ambiguous or garbled).
 *
 * The problem, as the paper states it:
 *   - a scene is a set of primitives S = {P1..Pn} (Sec. 5.1): here
 *     triangles (meshes and DTM rasters) and one grid of
 *     transmissive voxels carrying plant area density;
 *   - every emitted pulse is fanned out into subrays on concentric rings
 *     (Fig. 6), each cast independently to its first hit
 *     (P:197);
 *   - each hit's power follows the Gaussian beam profile (Eq. 1; Eq. 2,
 *     P:193) and the radar equation (Eq. 7);
 *   - the subray returns are binned into the pulse's full waveform with the
 *     pulse shape of Eq. 3 and a local-maximum filter
 *     turns it into discrete returns, linked to the waveform by the
 *     pulse index ("fullwaveIndex").
 *
 * Conventions for every call:
 *   - d_* = CUDA device pointer (cudaMalloc / torch CUDA tensor), h_* = host.
 *     Pointers named "p_*" may be either: the library asks the driver
 *     (cudaPointerGetAttributes) and stages host memory through device
 *     scratch itself (host <-> device copies are then part of the call).
 *   - Every call returns helios_status.  No C++ exception or abort crosses
 *     the ABI.  On failure helios_last_error() names the offending field.
 *   - Calls never read or write host memory asynchronously after returning.
 */
#ifndef HELIOS_H_
#define HELIOS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* helios_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  HELIOS_OK = 0,
  HELIOS_ERR_INVALID_ARGUMENT = 1, /* bad pointer / value; see helios_last_error()      */
  HELIOS_ERR_OUT_OF_MEMORY = 2,    /* device allocation failed                          */
  HELIOS_ERR_CUDA = 3,             /* any other CUDA runtime error                      */
  HELIOS_ERR_NOT_BUILT = 4,        /* helios_simulate before helios_build_accel         */
  HELIOS_ERR_EMPTY_SCENE = 5,      /* n_tris == 0 and no voxel grid                     */
  HELIOS_ERR_CAPACITY = 6          /* p_wf_compact too small: p_wf_offset[n_pulses] holds
                                      the floats needed; every other output is complete */
} helios_status;

/* Thread-local, NUL-terminated description of the last failure on this
 * thread ("" after a success).  Valid until the next helios_* call on the
 * same thread. */
const char* helios_last_error(void);

/* Library version string, e.g. "helios-b200 0.1 sm_100a". */
const char* helios_version(void);

/* ------------------------------------------------------------------------
 * Scene (Sec. 5.1; P:272 mixed-model scenes).
 * ---------------------------------------------------------------------- */
typedef struct helios_scene_s* helios_scene; /* opaque, library-owned */

typedef struct {
  /* Triangles.  [n_tris][3 vertices][xyz] fp32, row-major.
   * Primitive id = row index.  May be NULL iff n_tris == 0.                */
  const float* p_tri_xyz;
  /* [n_tris] Lambertian reflectance rho in [0,1] ("dependent on the
   * material", R14).  NULL -> 0.5 for every triangle.                      */
  const float* p_tri_reflectance;
  uint32_t n_tris;
  /* Transmissive voxel grid.  [nz][ny][nx] fp32
   * plant area density (m^2/m^3) >= 0; NULL -> no grid.  Voxel id
   * = ix + nx*(iy + ny*iz); reported as prim id n_tris + voxel id.          */
  const float* p_voxel_pad;
  uint32_t nx, ny, nz;
  double grid_origin[3]; /* min corner (m)   */
  double voxel_size;     /* edge (m), > 0    */
  /* G(|d_z|) for sigma = PAD * G (Eq. 4 / Table 2, R15): n_lut values at
   * |d_z| = k/(n_lut-1), linear interpolation.  NULL / 0 -> spherical LAD,
   * G = 0.5.  n_lut == 1 is invalid; n_lut <= 4096.                         */
  const float* h_g_lut;
  uint32_t n_lut;
  /* How the grid is interpreted (reading R31):
   *   HELIOS_VOXEL_TRANSMISSIVE  extinction + Beer-Lambert draws (default)
   *   HELIOS_VOXEL_OPAQUE        every voxel with PAD > 0 is a solid cube
   *   HELIOS_VOXEL_SCALED        solid cube of side a = a0 min(1, PAD/pad_max)^scale_alpha
   *                              (Eq. 5) centred in its voxel, optionally shifted
   *                              by a reproducible random offset (scale_shift = 1)
   * Opaque / scaled cubes return at their entry point with sigma_eff =
   * voxel_reflectance |cos| of the entry face (Lambertian).                  */
  uint32_t voxel_mode;
  float voxel_reflectance;  /* [0, 1] (opaque / scaled)                            */
  double pad_max;           /* > 0 (scaled)                                        */
  double scale_alpha;       /* >= 0 (scaled)                                       */
  uint32_t scale_shift;     /* 0 or 1 (scaled)                                     */
  uint32_t reserved_;       /* must be 0                                           */
} helios_scene_desc;

enum { HELIOS_VOXEL_TRANSMISSIVE = 0, HELIOS_VOXEL_OPAQUE = 1, HELIOS_VOXEL_SCALED = 2 };

/* Copy the scene into library-owned device memory (the caller may free its
 * arrays on return; the stream is synchronised).
 * Errors: INVALID_ARGUMENT (NULL desc/out, NULL triangles with n_tris > 0,
 * non-finite vertex, reflectance outside [0,1], PAD < 0 or non-finite,
 * voxel_size <= 0, n_tris + nx*ny*nz >= 2^32 - 1, n_lut == 1 or > 4096,
 * n_tris >= 2^28, unknown voxel_mode, voxel_reflectance outside [0,1],
 * scaled mode with pad_max <= 0 or scale_alpha < 0, scale_shift > 1,
 * reserved_ != 0); EMPTY_SCENE (no triangles and no grid);
 * OUT_OF_MEMORY; CUDA. */
helios_status helios_scene_create(const helios_scene_desc* desc, helios_stream stream,
                                  helios_scene* out);

/* Build the acceleration structure on the device (replaces the paper's
 * kd-tree, "prior art, not the blueprint"): a binary BVH over the
 * triangles -- 63-bit Morton codes of the centroids on an ISOTROPIC grid (21
 * bits per axis; the north star's 30-bit per-axis codes measured 2.3x slower
 * on C5, DESIGN.md s.7.1), a stable LSD radix sort (hand-written), then the
 * hierarchy: PLOC agglomerative clustering (default) or the Karras LBVH
 * (helios_tuning.builder = 1) with bottom-up AABB refit; 64-B child-pair
 * nodes, subtrees of <= 2 triangles collapsed into leaves, triangles permuted
 * to depth-first leaf order (48 B each).  Deterministic (same arrays -> same
 * tree).  Idempotent.  Synchronises the stream.
 * Errors: INVALID_ARGUMENT (NULL scene), OUT_OF_MEMORY, CUDA (incl. a tree
 * deeper than the 64-entry traversal stack). */
helios_status helios_build_accel(helios_scene scene, helios_stream stream);

/* Saving and loading a built acceleration structure ("Saving and
 * loading already built scenes is relying on boost serialisation"): the
 * tree and both triangle record arrays of a built scene as one
 * self-describing blob, so a later process skips helios_build_accel.
 *   helios_accel_export: buffer == NULL -> *bytes = the blob's size; else
 *     writes the blob (host or device memory, *bytes >= that size) and sets
 *     *bytes to it.  Synchronises the stream.
 *   helios_accel_import: installs a blob into a scene created from the SAME
 *     triangle soup and reflectances (checked by a 64-bit fingerprint of both
 *     arrays stored in the blob) in place of helios_build_accel; the scene is
 *     then built (results bitwise those of the exporting scene).  Replaces an
 *     existing tree.  Synchronises the stream.
 * Errors: INVALID_ARGUMENT (NULL scene / bytes, buffer too small, a blob that
 * is not one -- bad magic, version, record sizes, lengths -- or was exported
 * from other triangles), NOT_BUILT (export before a build), OUT_OF_MEMORY, CUDA. */
helios_status helios_accel_export(helios_scene scene, void* buffer, uint64_t* bytes,
                                  helios_stream stream);
helios_status helios_accel_import(helios_scene scene, const void* buffer, uint64_t bytes,
                                  helios_stream stream);

/* Free everything the scene owns.  NULL is a no-op.  Must not race with a
 * helios_simulate on the same scene. */
helios_status helios_scene_destroy(helios_scene scene);

/* Statistics of a built scene (for logs and the roofline accounting). */
typedef struct {
  uint32_t n_tris, n_nodes, max_depth, leaf_max;
  uint64_t node_bytes, tri_bytes, grid_bytes;
  double build_ms; /* device time of the last helios_build_accel */
} helios_scene_info;
helios_status helios_scene_get_info(helios_scene scene, helios_scene_info* out);

/* ------------------------------------------------------------------------
 * Scanner / beam / detector parameters.
 * ---------------------------------------------------------------------- */
typedef struct {
  double divergence_rad;  /* beta: 1/e^2 HALF-angle of the beam (R3), in (0, 0.1)   */
  uint32_t subray_count;  /* paper rule 1 + sum floor(2 pi i):
                             {1,7,19,37,62,93,130,173,223,279}; or hexagonal
                             1 + 3q(q+1) (R1): {61,91,127,169,217,271}          */
  double pulse_length_ns; /* tau = pulse_length_ns / 1.75, > 0            */
  double bin_width_ns;    /* Delta, binWidth_ns, > 0               */
  double max_fullwave_range_ns; /* maxFullwaveRange_ns, >= bin width;
                                   n_bins = ceil(window / Delta) (R9)            */
  float detection_threshold;    /* fraction of the pulse's waveform max (R11), (0,1] */
  uint32_t max_returns;         /* 1..255; earliest returns kept (R11)           */
  double peak_power_w;          /* I0 of Eq. 1 (> 0)                             */
  double efficiency;            /* lambda of Eq. 7 (atmosphere x efficiency), >= 0 */
  double receiver_diameter_m;   /* alpha of Eq. 7 (R14), >= 0                    */
  double wavelength_nm;         /* lambda of Eq. 2, > 0 when beam_waist_m > 0    */
  double beam_waist_m;          /* w0 of Eq. 2; 0 -> far field w = R tan(beta) (R5) */
  double focus_range_m;         /* R0 of Eq. 2, >= 0                             */
  uint64_t seed;                /* Philox-4x32-10 key for transmission draws (R19) */
  uint32_t fit_echo_width;      /* 0 or 1: fit a Gaussian to every return's echo
                                   ("Optionally, a Gaussian may be fitted ...
                                   to get a measure of echo width", P:280 non-linear
                                   least squares; reading R28: Levenberg-Marquardt
                                   over bins k +- ceil(3 pulse_length / Delta))      */
  uint32_t reserved_;           /* must be 0                                         */
  double range_noise_sd_m;      /* >= 0: sigma of the normal ranging error added to
                                   every return's range (reading R29:
                                   Box-Muller on Philox stream tag 1, counter
                                   (pulse, return number)); 0 -> noiseless       */
} helios_scanner_params;

/* Number of waveform bins, ceil(max_fullwave_range_ns / bin_width_ns);
 * 0 if the parameters are invalid. */
uint32_t helios_waveform_bins(const helios_scanner_params* params);

/* Kernel length L_p = ceil(20 tau / Delta) of the binned outgoing pulse (R9). */
uint32_t helios_pulse_taps(const helios_scanner_params* params);

/* ------------------------------------------------------------------------
 * Pulses and outputs.
 * ---------------------------------------------------------------------- */
typedef struct {
  const float* p_origin;    /* [n_pulses][3] fp32 (m)                               */
  const float* p_direction; /* [n_pulses][3] fp32, non-zero; normalised in fp64 (R24) */
  const double* p_time_s;   /* [n_pulses] GPS time, copied into returns; may be NULL */
  uint64_t n_pulses;
  uint64_t pulse_index_base; /* global id of element 0: Philox counter and output
                                pulse id ("fullwaveIndex").  Splitting a run
                                into batches with matching bases is bitwise
                                identical to one call.                           */
} helios_pulses;

/* One discrete return (P:215, P:276 LAS point format 1 fields; echo width
 * P:280). 32 bytes. */
typedef struct {
  double range_m;        /* (c/2)(k0 + k - j* + 1/2) Delta (R12)                */
  double gps_time_s;     /* the pulse's time                                    */
  float intensity;       /* waveform value at the peak bin                      */
  uint32_t prim_id;      /* generating primitive (R13): triangle row, or
                            n_tris + voxel id                                   */
  uint8_t return_number; /* 1-based, time order                                 */
  uint8_t n_returns;     /* returns of this pulse                               */
  uint8_t pad[2];        /* zero                                                */
  float echo_width_ns;   /* fitted Gaussian sigma (ns) when fit_echo_width = 1
                            (R28); NaN when not requested or when
                            the fit did not converge                           */
} helios_return;

/* One subray's event (debug / parity export). 16 bytes.
 * Miss: range NaN, amplitude 0, prim UINT32_MAX. */
typedef struct {
  double range_m;  /* ray parameter of the event (m)  */
  float amplitude; /* A_s = K sigma_eff I_s / R^4 (Eq. 1, 7) */
  uint32_t prim_id;
} helios_subray_hit;

typedef struct {
  uint8_t* p_n_returns;        /* [n_pulses]                                        */
  helios_return* p_returns;    /* [n_pulses][max_returns]; unused slots zeroed;
                                  may be NULL when p_returns_packed is given       */
  int64_t* p_wf_first_bin;     /* [n_pulses] absolute bin k0 of waveform[0]; -1 = no hit */
  float* p_waveform;           /* [n_pulses][n_bins] or NULL (binning still runs) */
  helios_subray_hit* p_subray_hits; /* [n_pulses][subray_count] or NULL              */
  /* Compact (sparse-support) waveform output, lossless: the bins of row p
   * that can be non-zero, W[0 .. len_p), packed back to back in pulse order.
   * len_p = min(n_bins, max_s (k_s - k0) + L_p) over the subrays whose bin
   * lies in the window (R9), 0 for a pulse without hit; every dense bin at or
   * beyond len_p is exactly 0.  Row p occupies
   * p_wf_compact[p_wf_offset[p] .. p_wf_offset[p+1]), p_wf_offset[0] = 0
   * (offsets relative to this call).  p_wf_offset is required with
   * p_wf_compact and may be given alone (lengths only).  If
   * p_wf_offset[n_pulses] > wf_compact_capacity the call returns
   * HELIOS_ERR_CAPACITY after completing everything else; rows past the
   * capacity are then not (or not completely) written.                      */
  float* p_wf_compact;         /* [wf_compact_capacity] or NULL                     */
  uint64_t* p_wf_offset;       /* [n_pulses + 1] or NULL                            */
  uint64_t wf_compact_capacity;
  /* Beam export of helios_simulate_survey ("the beam origin and the
   * beam direction" of every beam): the generated pulses as simulated.
   * Ignored by helios_simulate (the caller has its pulses).                 */
  float* p_beam_origin;        /* [n_pulses][3] or NULL                             */
  float* p_beam_direction;     /* [n_pulses][3] or NULL                             */
  double* p_beam_time;         /* [n_pulses] or NULL                                */
  /* Packed returns: the used return slots only, pulse after pulse (pulse p's
   * returns are p_returns_packed[p_return_offset[p] .. p_return_offset[p+1]),
   * p_return_offset[0] = 0, offsets relative to this call).  With packed
   * returns p_returns may be NULL.  If p_return_offset[n_pulses] >
   * returns_capacity the call returns HELIOS_ERR_CAPACITY (everything else
   * complete; returns past the capacity not written).                       */
  helios_return* p_returns_packed; /* [returns_capacity] or NULL                    */
  uint64_t* p_return_offset;       /* [n_pulses + 1]; required with p_returns_packed */
  uint64_t returns_capacity;
} helios_outputs;

/* Optional per-call accounting.  Inputs: collect_counters.  Everything else
 * is written by helios_simulate. */
typedef struct {
  uint32_t collect_counters; /* in: 1 -> run the instrumented traversal variant
                                (node / triangle / voxel-step counters; slower:
                                for roofline byte accounting only)               */
  uint32_t kernel_launches;  /* out: kernels launched by this call               */
  uint32_t node_bytes;       /* out: bytes per BVH node of the traversal that ran */
  uint32_t trace_launches;   /* out: K6 launches (one per chunk of pulses)        */
  uint64_t pulses, subrays;
  uint64_t subray_hits, voxel_returns, returns;     /* only with collect_counters */
  uint64_t nodes_visited, tris_tested, voxel_steps; /* only with collect_counters */
  uint64_t fp64_tests; /* triangles the fp32 prefilter could not reject (collect_counters) */
  double trace_ms;    /* out: summed device time of the trace launches (K6), CUDA events */
  double waveform_ms; /* out: summed device time of the waveform launches (K7)          */
  uint64_t beam_nodes; /* BVH nodes tested by the per-pulse beam pre-pass K6a (collect_counters) */
  double beam_ms;     /* out: summed device time of the beam pre-pass launches (K6a)     */
  uint32_t batches;   /* out: pulse batches of the call                                  */
  uint32_t chunks;    /* out: pipeline chunks of the call                                */
  /* warp-level traversal counts of K6 (collect_counters; each once per warp,
     whatever the number of its lanes involved): beam-entry list entries
     examined, entries walked, packet steps (node or leaf visits), triangles
     iterated in leaves -- the cost of the union of the lanes' paths */
  uint64_t warp_entries, warp_entries_walked, warp_steps, warp_leaf_tris;
  /* fp64 tests run inside the walks (counted once per group of lanes running
     one together), and definite fp32 hits that had to be decided at once */
  uint64_t warp_fp64_in_walk, second_definite_hits;
} helios_stats;

/* Simulate n_pulses pulses (the hot path: subray fan-out, nearest hit against
 * triangles and transmissive voxels, radiometry, full waveform, peaks).
 * Enqueues on `stream` and synchronises it before returning (blocking).
 * Pointers in pulses/outputs may be device or host memory (see top).
 * stats may be NULL; when non-NULL the per-kernel device times are measured
 * with CUDA events on `stream`, and with stats->collect_counters = 1 the
 * traversal counters are collected by an instrumented kernel variant.
 * Errors: INVALID_ARGUMENT (NULL args, parameter out of range, a zero-length
 * pulse direction -- detected on the device; that pulse's outputs are then
 * those of a pulse with no hit), NOT_BUILT, OUT_OF_MEMORY, CUDA.
 * n_pulses == 0 is OK and writes nothing. */
helios_status helios_simulate(helios_scene scene, const helios_scanner_params* params,
                              const helios_pulses* pulses, const helios_outputs* outputs,
                              helios_stream stream, helios_stats* stats);

/* Simulate n_batches independent pulse batches in ONE call: pulses[i] with
 * outputs[i] (each exactly as one helios_simulate call: its own pulse ids,
 * its own packed offsets relative to the batch, its own capacities).  The
 * batches run through one chunk pipeline, so the head of a batch overlaps the
 * tail of the previous one and host copies of one batch overlap kernels of
 * the next (pulses are independent).  Results are bitwise those of
 * n_batches separate helios_simulate calls.  Blocking, like helios_simulate.
 * Output arrays of different batches must not overlap.  Errors as
 * helios_simulate (the message names the batch); HELIOS_ERR_CAPACITY is
 * returned if any batch's packed buffer was too small (all other outputs of
 * every batch complete). */
helios_status helios_simulate_batches(helios_scene scene, const helios_scanner_params* params,
                                      const helios_pulses* pulses, const helios_outputs* outputs,
                                      uint32_t n_batches, helios_stream stream,
                                      helios_stats* stats);

/* Non-blocking helios_simulate_batches ("a non-blocking variant
 * is NEXT").  Checks its own arguments, copies the parameter struct and the
 * pulses / outputs descriptors (not the arrays they point to) and returns at
 * once; a library worker thread runs the call (on the scene's device, on
 * `stream`), so the caller's thread is free and calls on distinct streams
 * overlap on the device (one call's pipeline head and tail under another's
 * kernels; pulses are independent).  Results are bitwise those of
 * helios_simulate_batches.  Every array the descriptors point to must stay
 * valid and untouched until helios_call_wait returns; `stats` (may be NULL)
 * is read when the call is submitted (collect_counters) and written by the
 * wait.  Errors: INVALID_ARGUMENT (NULL call, scene or descriptors), or
 * OUT_OF_MEMORY / CUDA if the worker cannot be started; everything else
 * (including argument checks of the call itself) is returned by the wait. */
typedef struct helios_call_s* helios_call;
helios_status helios_simulate_batches_async(helios_scene scene,
                                            const helios_scanner_params* params,
                                            const helios_pulses* pulses,
                                            const helios_outputs* outputs, uint32_t n_batches,
                                            helios_stream stream, const helios_stats* stats,
                                            helios_call* call);
/* Wait for an async call to finish (its stream is then synchronised); returns
 * the call's status -- its message, if any, through helios_last_error on this
 * thread -- copies its statistics into `stats` (may be NULL) and frees the
 * handle.  Each handle must be waited for exactly once. */
helios_status helios_call_wait(helios_call call, helios_stats* stats);

/* ------------------------------------------------------------------------
 * Process-wide tuning / test switches.  Not needed for correct use: every
 * value only changes how the same results are computed (the tests check the
 * outputs bitwise invariant to them).  Read by a call when it starts.  At the
 * first use they are seeded once from the environment (HELIOS_BEAM,
 * HELIOS_BUILDER=lbvh|ploc, HELIOS_LANE_ORDER, HELIOS_PAD_LANES,
 * HELIOS_SERIALIZE, HELIOS_TRACE_SPANS, HELIOS_CHUNK_PULSES; the fault injection
 * fault_alloc_bytes is never seeded).
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t beam_prepass; /* K6a: -1 or 1 on wherever it applies (trees with internal nodes,
                           beams of >= 7 subrays), 0 off                                  */
  int32_t builder;      /* helios_build_accel hierarchy: 0 PLOC (default), 1 Karras LBVH     */
  int32_t lane_order;   /* K6 lanes <-> subrays: 1 Hilbert patches (default), 0 ring order R4 */
  int32_t pad_lanes;    /* pad a pulse's lanes to whole warps: -1 auto (<= 6 % waste), 0, 1  */
  int32_t serialize;    /* 1: every kernel on the caller's stream, no overlap (exclusive
                           per-kernel device times in helios_stats); 0 default             */
  int32_t trace_spans;  /* 1: print per-stream device spans of every call to stderr         */
  uint64_t chunk_pulses;/* 0 auto, else pulses per pipeline chunk (>= 1024)                 */
  uint64_t fault_alloc_bytes; /* fault injection (SURVEY s.5): 0 off, else every library
                                 device allocation larger than this fails as out of memory  */
} helios_tuning;
helios_status helios_get_tuning(helios_tuning* out);
helios_status helios_set_tuning(const helios_tuning* tuning); /* INVALID_ARGUMENT if out of range */

/* ------------------------------------------------------------------------
 * On-device pulse generation (P:155 platforms, P:177 scan deflectors;
 * reading R30 of DESIGN.md s.3).  Pulse g of a survey is emitted at
 * t = t0_s + g / pulse_freq_hz.  Deflector angle with u = frac(f t),
 * A = scan_angle_rad:
 *   POLYGON      theta = -A + 2 A u                       (parallel lines)
 *   FIBRE        theta = -A + 2 A (k + 1/2) / n_fibres, k = floor(u n_fibres)
 *   OSCILLATING  theta = A sin(2 pi f t)                  (zig-zag)
 *   PALMER       cone of half-angle A around nadir, azimuth 2 pi u
 * Scanner-frame beam (0, -sin theta, -cos theta) (theta > 0 to starboard;
 * Palmer (sin A cos phi, sin A sin phi, -cos A)), rotated by the head
 * (Rz(head_rotation_rad_s t)), by the mount matrix, and by the platform yaw:
 * Static (one waypoint, yaw 0) or LinearPath (constant speed along the
 * waypoints, "orientation ... always towards the next waypoint"; at
 * the last waypoint it stays).  Origin = platform position + rotated
 * mount_offset.  All in fp64, stored as fp32 origin/direction + fp64 time.
 * ---------------------------------------------------------------------- */
typedef enum {
  HELIOS_DEFLECTOR_POLYGON = 0,
  HELIOS_DEFLECTOR_FIBRE = 1,
  HELIOS_DEFLECTOR_OSCILLATING = 2,
  HELIOS_DEFLECTOR_PALMER = 3
} helios_deflector;

typedef struct {
  const double* h_waypoints;  /* [n_waypoints][3] (m), host memory, copied per call   */
  uint32_t n_waypoints;       /* >= 1; 1 = Static platform                           */
  uint32_t deflector;         /* helios_deflector                                    */
  double speed_m_s;           /* LinearPath speed, > 0 when n_waypoints > 1          */
  double mount[9];            /* scanner -> platform rotation, row-major (identity:
                                 scan plane across track, nadir at theta = 0)        */
  double mount_offset[3];     /* scanner position in the platform frame (m)          */
  double head_rotation_rad_s; /* rotation of the scanner head about platform z       */
  double pulse_freq_hz;       /* PRF, > 0                                            */
  double t0_s;                /* emission time of survey pulse 0                     */
  double scan_freq_hz;        /* sweeps (lines / cone turns / periods) per s, > 0    */
  double scan_angle_rad;      /* A: half-amplitude in [0, pi) (a 330-degree line
                                 scanner has A = 165 deg), Palmer cone angle in
                                 [0, pi/2)                                          */
  uint32_t n_fibres;          /* FIBRE: lines per sweep, >= 1                        */
  uint32_t reserved_;         /* must be 0                                           */
} helios_survey;

/* Simulate survey pulses first_pulse .. first_pulse + n_pulses - 1, generated
 * on the device (no pulse arrays cross the boundary); pulse_index_base is the
 * global id of the first one (Philox counter, output pulse id).  Outputs and
 * errors as helios_simulate, plus INVALID_ARGUMENT for an invalid survey
 * (NULL, no waypoint, non-finite values, speed <= 0 with > 1 waypoint,
 * PRF / scan frequency <= 0, angle outside its range, n_fibres == 0 with
 * FIBRE, unknown deflector).  p_beam_* receive the generated pulses. */
helios_status helios_simulate_survey(helios_scene scene, const helios_scanner_params* params,
                                     const helios_survey* survey, uint64_t first_pulse,
                                     uint64_t n_pulses, uint64_t pulse_index_base,
                                     const helios_outputs* outputs, helios_stream stream,
                                     helios_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* HELIOS_H_ */
