"""Thin ctypes binding over libhelios.so (include/helios.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  torch is used for device memory and streams.
There is no CPU fallback: if libhelios.so is missing or no CUDA device is
present, the calls raise.

The C names are exposed as-is (``helios_scene_create`` ...) together with a
small object layer (``Scene``, ``simulate``) that allocates outputs.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HELIOS_LIB") or os.path.join(_HERE, "libhelios.so")

HELIOS_OK = 0
HELIOS_ERR_INVALID_ARGUMENT = 1
HELIOS_ERR_OUT_OF_MEMORY = 2
HELIOS_ERR_CUDA = 3
HELIOS_ERR_NOT_BUILT = 4
HELIOS_ERR_EMPTY_SCENE = 5
HELIOS_ERR_CAPACITY = 6
_STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "OUT_OF_MEMORY", 3: "CUDA", 4: "NOT_BUILT",
           5: "EMPTY_SCENE", 6: "CAPACITY"}

EXPORTED = ("helios_last_error", "helios_version", "helios_scene_create", "helios_build_accel",
            "helios_scene_destroy", "helios_scene_get_info", "helios_waveform_bins",
            "helios_accel_export", "helios_accel_import",
            "helios_pulse_taps", "helios_simulate", "helios_simulate_batches",
            "helios_simulate_batches_async", "helios_call_wait", "helios_simulate_survey",
            "helios_get_tuning", "helios_set_tuning",
            "helios_util_sort_pairs_u64", "helios_util_scan_u64",
            "helios_util_fp64_fma_tflops")


class HeliosError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"helios {_STATUS.get(status, status)}: {msg}")
        self.status = status


_d, _u32, _u64, _vp, _f = ctypes.c_double, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_float


class helios_scene_desc(ctypes.Structure):
    _fields_ = [("p_tri_xyz", _vp), ("p_tri_reflectance", _vp), ("n_tris", _u32),
                ("p_voxel_pad", _vp), ("nx", _u32), ("ny", _u32), ("nz", _u32),
                ("grid_origin", _d * 3), ("voxel_size", _d), ("h_g_lut", _vp), ("n_lut", _u32),
                ("voxel_mode", _u32), ("voxel_reflectance", _f), ("pad_max", _d),
                ("scale_alpha", _d), ("scale_shift", _u32), ("reserved_", _u32)]


VOXEL_MODES = {"transmissive": 0, "opaque": 1, "scaled": 2}


class helios_scanner_params(ctypes.Structure):
    _fields_ = [("divergence_rad", _d), ("subray_count", _u32), ("pulse_length_ns", _d),
                ("bin_width_ns", _d), ("max_fullwave_range_ns", _d),
                ("detection_threshold", _f), ("max_returns", _u32), ("peak_power_w", _d),
                ("efficiency", _d), ("receiver_diameter_m", _d), ("wavelength_nm", _d),
                ("beam_waist_m", _d), ("focus_range_m", _d), ("seed", _u64),
                ("fit_echo_width", _u32), ("reserved_", _u32), ("range_noise_sd_m", _d)]


class helios_pulses(ctypes.Structure):
    _fields_ = [("p_origin", _vp), ("p_direction", _vp), ("p_time_s", _vp),
                ("n_pulses", _u64), ("pulse_index_base", _u64)]


class helios_outputs(ctypes.Structure):
    _fields_ = [("p_n_returns", _vp), ("p_returns", _vp), ("p_wf_first_bin", _vp),
                ("p_waveform", _vp), ("p_subray_hits", _vp), ("p_wf_compact", _vp),
                ("p_wf_offset", _vp), ("wf_compact_capacity", _u64), ("p_beam_origin", _vp),
                ("p_beam_direction", _vp), ("p_beam_time", _vp), ("p_returns_packed", _vp),
                ("p_return_offset", _vp), ("returns_capacity", _u64)]


DEFLECTORS = {"polygon": 0, "fibre": 1, "oscillating": 2, "palmer": 3}


class helios_survey(ctypes.Structure):
    _fields_ = [("h_waypoints", _vp), ("n_waypoints", _u32), ("deflector", _u32),
                ("speed_m_s", _d), ("mount", _d * 9), ("mount_offset", _d * 3),
                ("head_rotation_rad_s", _d), ("pulse_freq_hz", _d), ("t0_s", _d),
                ("scan_freq_hz", _d), ("scan_angle_rad", _d), ("n_fibres", _u32),
                ("reserved_", _u32)]


class helios_stats(ctypes.Structure):
    _fields_ = ([("collect_counters", _u32), ("kernel_launches", _u32), ("node_bytes", _u32),
                 ("trace_launches", _u32)] +
                [(n, _u64) for n in ("pulses", "subrays", "subray_hits", "voxel_returns",
                                     "returns", "nodes_visited", "tris_tested", "voxel_steps",
                                     "fp64_tests")] +
                [("trace_ms", _d), ("waveform_ms", _d), ("beam_nodes", _u64), ("beam_ms", _d),
                 ("batches", _u32), ("chunks", _u32), ("warp_entries", _u64),
                 ("warp_entries_walked", _u64), ("warp_steps", _u64), ("warp_leaf_tris", _u64),
                 ("warp_fp64_in_walk", _u64), ("second_definite_hits", _u64)])


class helios_tuning(ctypes.Structure):
    _fields_ = [("beam_prepass", ctypes.c_int32), ("builder", ctypes.c_int32),
                ("lane_order", ctypes.c_int32), ("pad_lanes", ctypes.c_int32),
                ("serialize", ctypes.c_int32), ("trace_spans", ctypes.c_int32),
                ("chunk_pulses", _u64), ("fault_alloc_bytes", _u64)]


class helios_scene_info(ctypes.Structure):
    _fields_ = [("n_tris", _u32), ("n_nodes", _u32), ("max_depth", _u32), ("leaf_max", _u32),
                ("node_bytes", _u64), ("tri_bytes", _u64), ("grid_bytes", _u64),
                ("build_ms", _d)]


RETURN_DTYPE = np.dtype([("range_m", "<f8"), ("gps_time_s", "<f8"), ("intensity", "<f4"),
                         ("prim_id", "<u4"), ("return_number", "u1"), ("n_returns", "u1"),
                         ("pad", "u1", 2), ("echo_width_ns", "<f4")])
SUBRAY_DTYPE = np.dtype([("range_m", "<f8"), ("amplitude", "<f4"), ("prim_id", "<u4")])
assert RETURN_DTYPE.itemsize == 32 and SUBRAY_DTYPE.itemsize == 16

_lib = None


def lib() -> ctypes.CDLL:
    """Load libhelios.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2101_09154_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.helios_last_error.restype = ctypes.c_char_p
        L.helios_version.restype = ctypes.c_char_p
        L.helios_scene_create.restype = ctypes.c_int
        L.helios_scene_create.argtypes = [ctypes.POINTER(helios_scene_desc), _vp,
                                          ctypes.POINTER(_vp)]
        L.helios_build_accel.restype = ctypes.c_int
        L.helios_build_accel.argtypes = [_vp, _vp]
        L.helios_accel_export.restype = ctypes.c_int
        L.helios_accel_export.argtypes = [_vp, _vp, ctypes.POINTER(_u64), _vp]
        L.helios_accel_import.restype = ctypes.c_int
        L.helios_accel_import.argtypes = [_vp, _vp, _u64, _vp]
        L.helios_scene_destroy.restype = ctypes.c_int
        L.helios_scene_destroy.argtypes = [_vp]
        L.helios_scene_get_info.restype = ctypes.c_int
        L.helios_scene_get_info.argtypes = [_vp, ctypes.POINTER(helios_scene_info)]
        L.helios_waveform_bins.restype = _u32
        L.helios_waveform_bins.argtypes = [ctypes.POINTER(helios_scanner_params)]
        L.helios_pulse_taps.restype = _u32
        L.helios_pulse_taps.argtypes = [ctypes.POINTER(helios_scanner_params)]
        L.helios_simulate_survey.restype = ctypes.c_int
        L.helios_simulate_survey.argtypes = [_vp, ctypes.POINTER(helios_scanner_params),
                                             ctypes.POINTER(helios_survey), _u64, _u64, _u64,
                                             ctypes.POINTER(helios_outputs), _vp,
                                             ctypes.POINTER(helios_stats)]
        L.helios_simulate.restype = ctypes.c_int
        L.helios_simulate.argtypes = [_vp, ctypes.POINTER(helios_scanner_params),
                                      ctypes.POINTER(helios_pulses),
                                      ctypes.POINTER(helios_outputs), _vp,
                                      ctypes.POINTER(helios_stats)]
        L.helios_simulate_batches.restype = ctypes.c_int
        L.helios_simulate_batches.argtypes = [_vp, ctypes.POINTER(helios_scanner_params),
                                              ctypes.POINTER(helios_pulses),
                                              ctypes.POINTER(helios_outputs), _u32, _vp,
                                              ctypes.POINTER(helios_stats)]
        L.helios_simulate_batches_async.restype = ctypes.c_int
        L.helios_simulate_batches_async.argtypes = [_vp, ctypes.POINTER(helios_scanner_params),
                                                    ctypes.POINTER(helios_pulses),
                                                    ctypes.POINTER(helios_outputs), _u32, _vp,
                                                    ctypes.POINTER(helios_stats),
                                                    ctypes.POINTER(_vp)]
        L.helios_call_wait.restype = ctypes.c_int
        L.helios_call_wait.argtypes = [_vp, ctypes.POINTER(helios_stats)]
        L.helios_get_tuning.restype = ctypes.c_int
        L.helios_get_tuning.argtypes = [ctypes.POINTER(helios_tuning)]
        L.helios_set_tuning.restype = ctypes.c_int
        L.helios_set_tuning.argtypes = [ctypes.POINTER(helios_tuning)]
        L.helios_util_sort_pairs_u64.restype = ctypes.c_int
        L.helios_util_sort_pairs_u64.argtypes = [_vp, _vp, _u64, ctypes.c_int, _vp]
        L.helios_util_fp64_fma_tflops.restype = ctypes.c_int
        L.helios_util_fp64_fma_tflops.argtypes = [ctypes.POINTER(_d), _vp]
        L.helios_util_scan_u64.restype = ctypes.c_int
        L.helios_util_scan_u64.argtypes = [_vp, _vp, _u64, ctypes.c_int, _vp]
        _lib = L
    return _lib


def _check(status: int):
    if status != HELIOS_OK:
        raise HeliosError(status, lib().helios_last_error().decode())


def _ptr(x):
    """Pointer of a torch tensor (device or host) or numpy array; None -> NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ raw C names
def helios_version() -> str:
    return lib().helios_version().decode()


def helios_last_error() -> str:
    return lib().helios_last_error().decode()


def helios_scene_create(desc: helios_scene_desc, stream=None) -> int:
    h = _vp()
    _check(lib().helios_scene_create(ctypes.byref(desc), _stream(stream), ctypes.byref(h)))
    return h.value


def helios_build_accel(scene: int, stream=None) -> None:
    _check(lib().helios_build_accel(scene, _stream(stream)))


def helios_accel_export(scene: int, stream=None) -> bytes:
    """The built tree and triangle records as one blob."""
    n = _u64(0)
    _check(lib().helios_accel_export(scene, None, ctypes.byref(n), _stream(stream)))
    buf = ctypes.create_string_buffer(n.value)
    _check(lib().helios_accel_export(scene, buf, ctypes.byref(n), _stream(stream)))
    return buf.raw[:n.value]


def helios_accel_import(scene: int, blob: bytes, stream=None) -> None:
    _check(lib().helios_accel_import(scene, blob, len(blob), _stream(stream)))


def helios_scene_destroy(scene: int) -> None:
    _check(lib().helios_scene_destroy(scene))


def helios_scene_get_info(scene: int) -> helios_scene_info:
    info = helios_scene_info()
    _check(lib().helios_scene_get_info(scene, ctypes.byref(info)))
    return info


def helios_waveform_bins(params: helios_scanner_params) -> int:
    return int(lib().helios_waveform_bins(ctypes.byref(params)))


def helios_pulse_taps(params: helios_scanner_params) -> int:
    return int(lib().helios_pulse_taps(ctypes.byref(params)))


def helios_simulate(scene: int, params: helios_scanner_params, pulses: helios_pulses,
                    outputs: helios_outputs, stream=None, stats: helios_stats | None = None):
    _check(lib().helios_simulate(scene, ctypes.byref(params), ctypes.byref(pulses),
                                 ctypes.byref(outputs), _stream(stream),
                                 None if stats is None else ctypes.byref(stats)))


def helios_simulate_batches(scene: int, params: helios_scanner_params, pulses, outputs,
                            stream=None, stats: helios_stats | None = None):
    """pulses / outputs: sequences of helios_pulses / helios_outputs (one per batch)."""
    n = len(pulses)
    assert len(outputs) == n
    P = (helios_pulses * n)(*pulses)
    O = (helios_outputs * n)(*outputs)
    _check(lib().helios_simulate_batches(scene, ctypes.byref(params), P, O, n, _stream(stream),
                                         None if stats is None else ctypes.byref(stats)))


def helios_simulate_batches_async(scene: int, params: helios_scanner_params, pulses, outputs,
                                  stream=None, stats: helios_stats | None = None) -> int:
    """Submit; returns the helios_call handle (an int).  The descriptor arrays
    are copied by the library; the arrays they point to must outlive the wait."""
    n = len(pulses)
    assert len(outputs) == n
    P = (helios_pulses * n)(*pulses)
    O = (helios_outputs * n)(*outputs)
    h = _vp()
    _check(lib().helios_simulate_batches_async(scene, ctypes.byref(params), P, O, n,
                                               _stream(stream),
                                               None if stats is None else ctypes.byref(stats),
                                               ctypes.byref(h)))
    return h.value


def helios_call_wait(call: int, stats: helios_stats | None = None) -> None:
    _check(lib().helios_call_wait(call, None if stats is None else ctypes.byref(stats)))


def helios_get_tuning() -> helios_tuning:
    t = helios_tuning()
    _check(lib().helios_get_tuning(ctypes.byref(t)))
    return t


def helios_set_tuning(t: helios_tuning) -> None:
    _check(lib().helios_set_tuning(ctypes.byref(t)))


class tuning:
    """Context manager: tuning switches for the calls inside, e.g.
    ``with tuning(beam_prepass=0): ...`` (restored on exit)."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = None

    def __enter__(self):
        self.old = helios_get_tuning()
        t = helios_get_tuning()
        for k, v in self.kw.items():
            setattr(t, k, v)
        helios_set_tuning(t)
        return t

    def __exit__(self, *exc):
        helios_set_tuning(self.old)
        return False


def util_sort_pairs_u64(keys, vals, key_bits: int = 64, stream=None) -> None:
    """In-place stable radix sort of CUDA tensors keys (int64/uint64) and vals (int32/uint32)."""
    rc = lib().helios_util_sort_pairs_u64(_ptr(keys), _ptr(vals), int(keys.numel()), key_bits,
                                          _stream(stream))
    if rc:
        raise HeliosError(HELIOS_ERR_CUDA if rc == 3 else HELIOS_ERR_INVALID_ARGUMENT,
                          f"helios_util_sort_pairs_u64 returned {rc}")


def util_scan_u64(src, dst, inclusive: bool = True, stream=None) -> None:
    rc = lib().helios_util_scan_u64(_ptr(src), _ptr(dst), int(src.numel()), int(inclusive),
                                    _stream(stream))
    if rc:
        raise HeliosError(HELIOS_ERR_CUDA if rc == 3 else HELIOS_ERR_INVALID_ARGUMENT,
                          f"helios_util_scan_u64 returned {rc}")


def util_fp64_fma_tflops(stream=None) -> float:
    """Measured device fp64 FMA throughput (TFLOP/s)."""
    v = _d()
    rc = lib().helios_util_fp64_fma_tflops(ctypes.byref(v), _stream(stream))
    if rc:
        raise HeliosError(HELIOS_ERR_CUDA, f"helios_util_fp64_fma_tflops returned {rc}")
    return v.value


def helios_simulate_survey(scene: int, params: helios_scanner_params, survey: helios_survey,
                           first_pulse: int, n_pulses: int, pulse_index_base: int,
                           outputs: helios_outputs, stream=None,
                           stats: helios_stats | None = None):
    _check(lib().helios_simulate_survey(scene, ctypes.byref(params), ctypes.byref(survey),
                                        first_pulse, n_pulses, pulse_index_base,
                                        ctypes.byref(outputs), _stream(stream),
                                        None if stats is None else ctypes.byref(stats)))


# ------------------------------------------------------------------ object layer
def make_params(p) -> helios_scanner_params:
    """helios_scanner_params from any object with the same field names."""
    out = helios_scanner_params()
    for name, _ in helios_scanner_params._fields_:
        setattr(out, name, getattr(p, name, 0))
    return out


class Scene:
    """A built scene.  Arrays may be torch tensors (CUDA or CPU) or numpy."""

    def __init__(self, tri_xyz, tri_reflectance=None, voxel_pad=None, grid_origin=(0, 0, 0),
                 voxel_size=1.0, g_lut=None, stream=None, build=True, voxel_mode="transmissive",
                 voxel_reflectance=0.5, pad_max=1.0, scale_alpha=1.0, scale_shift=0):
        keep = []

        def arr(x, dtype):
            if x is None:
                return None
            if isinstance(x, np.ndarray):
                x = np.ascontiguousarray(x, dtype)
            else:
                x = x.contiguous()
            keep.append(x)
            return x

        tri = arr(tri_xyz, np.float32)
        refl = arr(tri_reflectance, np.float32)
        pad = arr(voxel_pad, np.float32)
        lut = None if g_lut is None else np.ascontiguousarray(
            g_lut.cpu().numpy() if hasattr(g_lut, "cpu") else g_lut, np.float32)
        d = helios_scene_desc()
        d.p_tri_xyz = _ptr(tri)
        d.p_tri_reflectance = _ptr(refl)
        d.n_tris = 0 if tri is None else int(tri.shape[0])
        d.p_voxel_pad = _ptr(pad)
        if pad is not None:
            nz, ny, nx = (int(s) for s in pad.shape)
            d.nx, d.ny, d.nz = nx, ny, nz
            d.grid_origin[:] = tuple(float(v) for v in grid_origin)
            d.voxel_size = float(voxel_size)
        d.h_g_lut = _ptr(lut)
        d.n_lut = 0 if lut is None else int(lut.size)
        d.voxel_mode = VOXEL_MODES[voxel_mode] if isinstance(voxel_mode, str) else int(voxel_mode)
        d.voxel_reflectance = float(voxel_reflectance)
        d.pad_max = float(pad_max)
        d.scale_alpha = float(scale_alpha)
        d.scale_shift = int(scale_shift)
        self.n_tris = d.n_tris
        self.handle = helios_scene_create(d, stream)
        if build:
            helios_build_accel(self.handle, stream)

    @classmethod
    def from_workload_scene(cls, sc, device="cuda", stream=None):
        import torch
        t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(device)
        return cls(t(sc.tri_xyz), t(sc.tri_reflectance), t(sc.voxel_pad), sc.grid_origin,
                   sc.voxel_size, sc.g_lut, stream=stream,
                   voxel_mode=getattr(sc, "voxel_mode", "transmissive"),
                   voxel_reflectance=getattr(sc, "voxel_reflectance", 0.5),
                   pad_max=getattr(sc, "pad_max", 1.0), scale_alpha=getattr(sc, "scale_alpha", 1.0),
                   scale_shift=getattr(sc, "scale_shift", 0))

    def info(self) -> helios_scene_info:
        return helios_scene_get_info(self.handle)

    def export_accel(self, stream=None) -> bytes:
        """helios_accel_export: the built tree (save it; skip the build later)."""
        return helios_accel_export(self.handle, stream)

    def import_accel(self, blob: bytes, stream=None) -> None:
        """helios_accel_import: install a saved tree (scene created with build=False)."""
        helios_accel_import(self.handle, blob, stream)

    def destroy(self):
        if getattr(self, "handle", None):
            helios_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


@dataclass
class Outputs:
    n_returns: object      # uint8 [n]
    returns: object        # uint8 [n, R, 32] (RETURN_DTYPE records)
    wf_first_bin: object   # int64 [n]
    waveform: object       # float32 [n, n_bins] or None
    subray_hits: object    # uint8 [n, N, 16] (SUBRAY_DTYPE records) or None
    wf_compact: object = None  # float32 [capacity] packed support rows, or None
    wf_offset: object = None   # uint64 [n + 1] row offsets into wf_compact, or None
    beam_origin: object = None     # float32 [n, 3] generated pulses (survey mode), or None
    beam_direction: object = None  # float32 [n, 3]
    beam_time: object = None       # float64 [n]
    returns_packed: object = None  # uint8 [capacity, 32] used return slots, pulse after pulse
    return_offset: object = None   # uint64 [n + 1] offsets into returns_packed

    def compact_row(self, p: int):
        """Support row p as a host numpy array: W[0 .. len_p) of the dense row."""
        host = lambda x: x if isinstance(x, np.ndarray) else x.cpu().numpy()
        off = host(self.wf_offset)
        return host(self.wf_compact[int(off[p]):int(off[p + 1])])

    def numpy(self) -> dict:
        """Host copies; records decoded to numpy structured arrays."""
        def host(x):
            if x is None:
                return None
            return x if isinstance(x, np.ndarray) else x.cpu().numpy()
        out = {"n_returns": host(self.n_returns), "wf_first_bin": host(self.wf_first_bin),
               "waveform": host(self.waveform)}
        r = host(self.returns)
        out["returns"] = None if r is None else np.ascontiguousarray(r).view(RETURN_DTYPE)[..., 0]
        h = host(self.subray_hits)
        out["subray_hits"] = None if h is None else np.ascontiguousarray(h).view(
            SUBRAY_DTYPE)[..., 0]
        out["wf_offset"] = host(self.wf_offset)
        out["beam_origin"] = host(self.beam_origin)
        out["beam_direction"] = host(self.beam_direction)
        out["beam_time"] = host(self.beam_time)
        rp = host(self.returns_packed)
        out["returns_packed"] = None if rp is None else np.ascontiguousarray(rp).view(
            RETURN_DTYPE)[..., 0]
        out["return_offset"] = host(self.return_offset)
        out["wf_compact"] = host(self.wf_compact)
        return out


def alloc_outputs(n: int, params, device="cuda", waveform=True, subray_hits=False,
                  pin_memory=False, compact: bool = False,
                  compact_capacity: int | None = None, beams: bool = False,
                  packed_returns: bool = False, returns_capacity: int | None = None,
                  slots: bool = True) -> Outputs:
    """Caller-owned outputs.  compact=True adds the packed support rows
    (default capacity n * (L_p + 64) floats; helios_simulate reports
    HELIOS_ERR_CAPACITY with the exact need if that is too small)."""
    import torch
    hp = params if isinstance(params, helios_scanner_params) else make_params(params)
    nb = helios_waveform_bins(hp)
    if nb == 0:
        raise HeliosError(HELIOS_ERR_INVALID_ARGUMENT, helios_last_error())
    kw = dict(device=device)
    if device == "cpu" and pin_memory:
        kw["pin_memory"] = True
    R, N = int(hp.max_returns), int(hp.subray_count)
    return Outputs(
        n_returns=torch.empty(n, dtype=torch.uint8, **kw),
        returns=torch.empty((n, R, 32), dtype=torch.uint8, **kw) if slots else None,
        wf_first_bin=torch.empty(n, dtype=torch.int64, **kw),
        waveform=torch.empty((n, nb), dtype=torch.float32, **kw) if waveform else None,
        subray_hits=torch.empty((n, N, 16), dtype=torch.uint8, **kw) if subray_hits else None,
        wf_compact=torch.empty(int(compact_capacity if compact_capacity is not None else
                                   n * (helios_pulse_taps(hp) + 64)), dtype=torch.float32, **kw)
        if compact else None,
        wf_offset=torch.empty(n + 1, dtype=torch.int64, **kw) if compact else None,
        beam_origin=torch.empty((n, 3), dtype=torch.float32, **kw) if beams else None,
        beam_direction=torch.empty((n, 3), dtype=torch.float32, **kw) if beams else None,
        beam_time=torch.empty(n, dtype=torch.float64, **kw) if beams else None,
        returns_packed=torch.empty((int(returns_capacity if returns_capacity is not None
                                        else 2 * n), 32), dtype=torch.uint8, **kw)
        if packed_returns else None,
        return_offset=torch.empty(n + 1, dtype=torch.int64, **kw) if packed_returns else None,
    )


def simulate(scene: Scene, params, origin, direction, time_s=None, pulse_index_base: int = 0,
             outputs: Outputs | None = None, waveform: bool = True, subray_hits: bool = False,
             stream=None, stats: bool = False, counters: bool = False, compact: bool = False,
             packed_returns: bool = False):
    """Run helios_simulate.  origin/direction: [n,3] float32 (CUDA tensors, or
    host tensors / numpy arrays -- staged by the library).  Returns
    (Outputs, helios_stats | None).  stats=True: per-kernel device times;
    counters=True: also the instrumented traversal counters."""
    hp = params if isinstance(params, helios_scanner_params) else make_params(params)
    def host(x, dt):
        if x is None:
            return None
        if isinstance(x, np.ndarray):
            return np.ascontiguousarray(x, dt)
        return x if x.is_contiguous() else x.contiguous()
    origin, direction = host(origin, np.float32), host(direction, np.float32)
    time_s = host(time_s, np.float64)
    n = int(origin.shape[0])
    if outputs is None:
        dev = "cuda" if (not isinstance(origin, np.ndarray) and origin.is_cuda) else "cpu"
        outputs = alloc_outputs(n, hp, dev, waveform, subray_hits, compact=compact,
                                packed_returns=packed_returns)
    p = helios_pulses()
    p.p_origin = _ptr(origin)
    p.p_direction = _ptr(direction)
    p.p_time_s = _ptr(time_s)
    p.n_pulses = n
    p.pulse_index_base = int(pulse_index_base)
    o = _marshal_outputs(outputs)
    st = helios_stats() if (stats or counters) else None
    if st is not None:
        st.collect_counters = 1 if counters else 0
    _run_with_capacity_retry(lambda: helios_simulate(scene.handle, hp, p, o, stream, st),
                             outputs, o)
    return outputs, st


def simulate_batches(scene: Scene, params, batches, outputs, stream=None, stats: bool = False,
                     counters: bool = False):
    """helios_simulate_batches: `batches` = [(origin, direction, time_s, pulse_index_base)],
    `outputs` = [Outputs] (one per batch, non-overlapping).  One call, one
    chunk pipeline over all batches.  Returns helios_stats | None."""
    hp = params if isinstance(params, helios_scanner_params) else make_params(params)
    ps, keep = [], []
    for (o, d, t, base) in batches:
        p = helios_pulses()
        p.p_origin, p.p_direction, p.p_time_s = _ptr(o), _ptr(d), _ptr(t)
        p.n_pulses = int(o.shape[0])
        p.pulse_index_base = int(base)
        ps.append(p)
        keep.append((o, d, t))
    os_ = [_marshal_outputs(x) for x in outputs]
    st = helios_stats() if (stats or counters) else None
    if st is not None:
        st.collect_counters = 1 if counters else 0
    try:
        helios_simulate_batches(scene.handle, hp, ps, os_, stream, st)
    except HeliosError as err:
        if err.status != HELIOS_ERR_CAPACITY:
            raise
        # grow every batch's packed buffer that was too small, run again
        for out, o in zip(outputs, os_):
            _grow_packed(out, o)
        helios_simulate_batches(scene.handle, hp, ps, os_, stream, st)
    del keep
    return st


class Call:
    """A submitted helios_simulate_batches_async call; wait() returns its
    helios_stats (or None) and raises HeliosError on failure.  Keeps the pulse
    and output arrays alive until the wait."""

    def __init__(self, handle, keep, stats):
        self._h, self._keep, self._stats = handle, keep, stats

    def wait(self):
        if self._h is None:
            raise RuntimeError("helios call already waited for")
        h, self._h = self._h, None
        try:
            helios_call_wait(h, self._stats)
        finally:
            self._keep = None
        return self._stats


def simulate_batches_async(scene: Scene, params, batches, outputs, stream=None,
                           stats: bool = False, counters: bool = False) -> Call:
    """helios_simulate_batches_async: the same arguments as simulate_batches;
    returns at once with a Call (wait() for the results; no capacity retry)."""
    hp = params if isinstance(params, helios_scanner_params) else make_params(params)
    ps, keep = [], [hp, batches, outputs]
    for (o, d, t, base) in batches:
        p = helios_pulses()
        p.p_origin, p.p_direction, p.p_time_s = _ptr(o), _ptr(d), _ptr(t)
        p.n_pulses = int(o.shape[0])
        p.pulse_index_base = int(base)
        ps.append(p)
    os_ = [_marshal_outputs(x) for x in outputs]
    st = helios_stats() if (stats or counters) else None
    if st is not None:
        st.collect_counters = 1 if counters else 0
    h = helios_simulate_batches_async(scene.handle, hp, ps, os_, stream, st)
    return Call(h, keep, st)


def make_survey(sv) -> tuple:
    """helios_survey from a workloads.Survey-like object; returns (struct, keep-alive)."""
    wp = np.ascontiguousarray(np.asarray(sv.waypoints, np.float64).reshape(-1, 3))
    c = helios_survey()
    c.h_waypoints = wp.ctypes.data
    c.n_waypoints = wp.shape[0]
    c.deflector = DEFLECTORS[sv.deflector] if isinstance(sv.deflector, str) else int(sv.deflector)
    c.speed_m_s = float(sv.speed_m_s)
    c.mount[:] = tuple(float(x) for x in np.asarray(sv.mount, np.float64).reshape(9))
    c.mount_offset[:] = tuple(float(x) for x in np.asarray(sv.mount_offset, np.float64).reshape(3))
    c.head_rotation_rad_s = float(sv.head_rotation_rad_s)
    c.pulse_freq_hz = float(sv.pulse_freq_hz)
    c.t0_s = float(sv.t0_s)
    c.scan_freq_hz = float(sv.scan_freq_hz)
    c.scan_angle_rad = float(sv.scan_angle_rad)
    c.n_fibres = int(sv.n_fibres)
    return c, wp


def simulate_survey(scene: Scene, params, survey, first_pulse: int, n_pulses: int,
                    pulse_index_base: int | None = None, outputs: Outputs | None = None,
                    device="cuda", waveform: bool = True, subray_hits: bool = False,
                    beams: bool = False, compact: bool = False, stream=None,
                    stats: bool = False, counters: bool = False):
    """helios_simulate_survey: pulses first_pulse .. +n_pulses of `survey`
    generated on the device.  Returns (Outputs, helios_stats | None)."""
    hp = params if isinstance(params, helios_scanner_params) else make_params(params)
    if outputs is None:
        outputs = alloc_outputs(n_pulses, hp, device, waveform, subray_hits, compact=compact,
                                beams=beams)
    sv, keep = make_survey(survey)
    o = _marshal_outputs(outputs)
    st = helios_stats() if (stats or counters) else None
    if st is not None:
        st.collect_counters = 1 if counters else 0
    base = first_pulse if pulse_index_base is None else pulse_index_base
    _run_with_capacity_retry(
        lambda: helios_simulate_survey(scene.handle, hp, sv, first_pulse, n_pulses, base, o,
                                       stream, st), outputs, o)
    del keep
    return outputs, st


def _run_with_capacity_retry(call, outputs, o):
    """Run; on HELIOS_ERR_CAPACITY grow the packed buffer(s) to the exact need
    reported in the offsets and run again."""
    try:
        call()
    except HeliosError as err:
        if err.status != HELIOS_ERR_CAPACITY:
            raise
        _grow_packed(outputs, o)
        call()


def _grow_packed(outputs, o):
    """Grow the packed buffers of `outputs` whose offsets report more than
    their capacity (after a HELIOS_ERR_CAPACITY call)."""
    import torch
    pin = lambda t: bool(getattr(t, "is_pinned", lambda: False)())
    if outputs.wf_compact is not None and int(outputs.wf_offset[-1]) > o.wf_compact_capacity:
        need = int(outputs.wf_offset[-1])
        old = outputs.wf_compact
        outputs.wf_compact = torch.empty(need, dtype=torch.float32, device=old.device,
                                         pin_memory=pin(old))
        o.p_wf_compact = _ptr(outputs.wf_compact)
        o.wf_compact_capacity = need
    if (outputs.returns_packed is not None and
            int(outputs.return_offset[-1]) > o.returns_capacity):
        need = int(outputs.return_offset[-1])
        old = outputs.returns_packed
        outputs.returns_packed = torch.empty((need, 32), dtype=torch.uint8, device=old.device,
                                             pin_memory=pin(old))
        o.p_returns_packed = _ptr(outputs.returns_packed)
        o.returns_capacity = need


def _marshal_outputs(outputs: Outputs) -> helios_outputs:
    o = helios_outputs()
    o.p_n_returns = _ptr(outputs.n_returns)
    o.p_returns = _ptr(outputs.returns)
    o.p_wf_first_bin = _ptr(outputs.wf_first_bin)
    o.p_waveform = _ptr(outputs.waveform)
    o.p_subray_hits = _ptr(outputs.subray_hits)
    o.p_wf_compact = _ptr(outputs.wf_compact)
    o.p_wf_offset = _ptr(outputs.wf_offset)
    wc = outputs.wf_compact
    o.wf_compact_capacity = 0 if wc is None else int(wc.numel() if hasattr(wc, "numel")
                                                     else wc.size)
    o.p_beam_origin = _ptr(outputs.beam_origin)
    o.p_beam_direction = _ptr(outputs.beam_direction)
    o.p_beam_time = _ptr(outputs.beam_time)
    o.p_returns_packed = _ptr(outputs.returns_packed)
    o.p_return_offset = _ptr(outputs.return_offset)
    rp = outputs.returns_packed
    o.returns_capacity = 0 if rp is None else int(rp.shape[0])
    return o
