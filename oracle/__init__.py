"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding to ``oracle/liboracle.so`` (built from ``oracle/oracle.cpp``):
the plain fp64 CPU implementation of the HELIOS++ hot path that the CUDA
library is checked against.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product package ``paper_2101_09154_b200`` never imports
it, and the two share no code (DESIGN.md s.4).

Every function cites the PAPER.md passage it follows (``P:n``) and the
DESIGN.md reading (``R<k>``) where the paper is silent or garbled.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "oracle.cpp")

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (plain g++, -O2, no fast-math)."""
    if force or not os.path.exists(LIB_PATH) or (
        os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH)
    ):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
             "-ffp-contract=off", SRC_PATH, "-o", tmp]
        )
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_d = ctypes.c_double
_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


class OracleParams(ctypes.Structure):
    _fields_ = [
        ("divergence_rad", _d), ("pulse_length_ns", _d), ("bin_width_ns", _d),
        ("max_fullwave_range_ns", _d), ("detection_threshold", _d),
        ("peak_power_w", _d), ("efficiency", _d), ("receiver_diameter_m", _d),
        ("wavelength_nm", _d), ("beam_waist_m", _d), ("focus_range_m", _d),
        ("seed", _u64), ("subray_count", _u32), ("max_returns", _u32),
        ("fit_echo_width", _u32), ("pad_", _u32), ("range_noise_sd_m", _d),
    ]


class OracleScene(ctypes.Structure):
    _fields_ = [
        ("tris", _vp), ("refl", _vp), ("n_tris", _u32), ("pad", _vp),
        ("n", _u32 * 3), ("origin", _d * 3), ("voxel_size", _d),
        ("g_lut", _vp), ("n_lut", _u32), ("voxel_mode", _u32), ("voxel_reflectance", _d),
        ("pad_max", _d), ("scale_alpha", _d), ("scale_shift", _u32), ("pad2_", _u32),
    ]


class OracleOutputs(ctypes.Structure):
    _fields_ = [(n, _vp) for n in (
        "n_returns", "k0", "waveform", "ret_range", "ret_time", "ret_intensity",
        "ret_prim", "ret_number", "ret_width", "peak_margin", "attr_margin", "sub_range",
        "sub_amp", "sub_prim", "sub_k", "sub_ncand", "sub_gap", "sub_kmargin",
        "sub_umargin", "sub_cand", "ret_cand")]

MAX_CAND = 8   # kMaxCand: triangle candidates per subray (C-4)
MAX_ATTR = 4   # kMaxAttr: attribution candidates per return (C-4)
DECISION_EPS = 2.5e-7  # kDecisionEps: margins below this may flip on the CUDA path


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_resolve_subrays.restype = ctypes.c_int
        L.oracle_resolve_subrays.argtypes = [_u32, ctypes.POINTER(ctypes.c_int)]
        L.oracle_subray_pattern.restype = ctypes.c_int
        L.oracle_subray_pattern.argtypes = [_u32, _d, _vp, _vp, _vp, _vp, _vp]
        L.oracle_subray_direction.restype = None
        L.oracle_subray_direction.argtypes = [_vp, _d, _d, _vp]
        for name, n in (("oracle_eq1_intensity", 3), ("oracle_eq2_beam_width", 4),
                        ("oracle_subray_intensity", 7), ("oracle_eq3_pulse", 3),
                        ("oracle_eq7_intensity", 6)):
            f = getattr(L, name)
            f.restype = _d
            f.argtypes = [_d] * n
        L.oracle_ray_triangle.restype = _d
        L.oracle_ray_triangle.argtypes = [_vp, _vp, _vp, _vp]
        L.oracle_nearest_triangle.restype = _i64
        L.oracle_nearest_triangle.argtypes = [_vp, _vp, _vp, _u32, _vp, _vp, _vp, _vp]
        L.oracle_nearest_candidates.restype = _i64
        L.oracle_nearest_candidates.argtypes = [_vp, _vp, _vp, _u32, _vp, _vp, _vp, _vp, _vp,
                                                ctypes.c_int32]
        L.oracle_cone_may_hit.restype = ctypes.c_int
        L.oracle_cone_may_hit.argtypes = [_vp, _vp, _d, _vp]
        L.oracle_bin_of.restype = _i64
        L.oracle_bin_of.argtypes = [_d, _d, _vp]
        L.oracle_transmits.restype = ctypes.c_int
        L.oracle_transmits.argtypes = [_d, _d, _d, _vp]
        L.oracle_waveform_peaks.restype = ctypes.c_int
        L.oracle_waveform_peaks.argtypes = [ctypes.POINTER(OracleParams), _vp, _vp, _vp, _d, _u64,
                                            _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                            _vp, _vp]
        L.oracle_philox4x32_10.restype = None
        L.oracle_philox4x32_10.argtypes = [_vp, _vp, _vp]
        L.oracle_transmission_u.restype = _d
        L.oracle_transmission_u.argtypes = [_u64, _u64, _u32, _u32]
        L.oracle_g_function.restype = _d
        L.oracle_g_function.argtypes = [_vp, _u32, _d]
        L.oracle_voxel_segments.restype = _i64
        L.oracle_voxel_segments.argtypes = [_vp, _vp, _vp, _vp, _d, _d, _vp, _vp, _vp, _i64]
        L.oracle_generate_pulses.restype = None
        L.oracle_generate_pulses.argtypes = [_vp, _u64, _i64, _vp, _vp, _vp]
        L.oracle_voxel_cube.restype = None
        L.oracle_voxel_cube.argtypes = [_vp, _vp, _d, _u32, _d, _u32, _d, _d, _u32, _u64, _vp,
                                        _vp]
        L.oracle_range_noise.restype = _d
        L.oracle_range_noise.argtypes = [_u64, _u64, _u32]
        L.oracle_fit_echo_width.restype = _d
        L.oracle_fit_echo_width.argtypes = [_vp, _i64, _i64, _d, _d, _vp, _vp]
        L.oracle_waveform_bins.restype = _u32
        L.oracle_waveform_bins.argtypes = [_d, _d]
        L.oracle_simulate.restype = ctypes.c_int
        L.oracle_simulate.argtypes = [ctypes.POINTER(OracleScene),
                                      ctypes.POINTER(OracleParams), _vp, _vp, _vp,
                                      _vp, _i64, ctypes.c_int,
                                      ctypes.POINTER(OracleOutputs)]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_vp)


# ---------------------------------------------------------------- primitives
def resolve_subrays(count: int):
    """(q, rule) for a subray count (R1); q = -1 if unreachable."""
    r = ctypes.c_int(-1)
    q = lib().oracle_resolve_subrays(count, ctypes.byref(r))
    return q, r.value


def subray_pattern(count: int, beta: float):
    """ring, slot, ring_n, theta, phi arrays for every subray (R2, R4)."""
    ring = np.zeros(count, np.int32)
    slot = np.zeros(count, np.int32)
    rn = np.zeros(count, np.int32)
    th = np.zeros(count, np.float64)
    ph = np.zeros(count, np.float64)
    if lib().oracle_subray_pattern(count, beta, _p(ring), _p(slot), _p(rn), _p(th), _p(ph)):
        raise ValueError(f"subray count {count} reachable by neither rule (R1)")
    return ring, slot, rn, th, ph


def subray_direction(d, theta: float, phi: float) -> np.ndarray:
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(3, np.float64)
    lib().oracle_subray_direction(_p(d), theta, phi, _p(out))
    return out


def eq1_intensity(I0, r, w):
    return lib().oracle_eq1_intensity(I0, r, w)


def eq2_beam_width(w0, lambda_nm, R, R0):
    return lib().oracle_eq2_beam_width(w0, lambda_nm, R, R0)


def subray_intensity(I0, theta, beta, R, w0=0.0, lambda_nm=1064.0, R0=0.0):
    return lib().oracle_subray_intensity(I0, theta, beta, R, w0, lambda_nm, R0)


def eq3_pulse(I, t, tau):
    return lib().oracle_eq3_pulse(I, t, tau)


def eq7_intensity(lambda_eff, sigma, P, alpha, d, beta):
    return lib().oracle_eq7_intensity(lambda_eff, sigma, P, alpha, d, beta)


def ray_triangle(o, d, tri9):
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    tri = np.ascontiguousarray(tri9, np.float32).reshape(9)
    c = ctypes.c_double(0.0)
    t = lib().oracle_ray_triangle(_p(o), _p(d), _p(tri), ctypes.byref(c))
    return t, c.value


def nearest_triangle(o, d, tris):
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
    t = ctypes.c_double()
    c = ctypes.c_double()
    nc = ctypes.c_int32()
    g = ctypes.c_double()
    i = lib().oracle_nearest_triangle(_p(o), _p(d), _p(tris), tris.shape[0],
                                      ctypes.byref(t), ctypes.byref(c),
                                      ctypes.byref(nc), ctypes.byref(g))
    return int(i), t.value, c.value, nc.value, g.value


def nearest_candidates(o, d, tris):
    """(id, t, n_cand, candidate ids by (t, id)) of the nearest hit (C-4:
    every triangle within 1e-6 m of the nearest)."""
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    tris = np.ascontiguousarray(tris, np.float32).reshape(-1, 9)
    t = ctypes.c_double()
    c = ctypes.c_double()
    nc = ctypes.c_int32()
    g = ctypes.c_double()
    cand = np.zeros(MAX_CAND, np.uint32)
    i = lib().oracle_nearest_candidates(_p(o), _p(d), _p(tris), tris.shape[0], ctypes.byref(t),
                                        ctypes.byref(c), ctypes.byref(nc), ctypes.byref(g),
                                        _p(cand), MAX_CAND)
    return int(i), t.value, nc.value, cand[:min(nc.value, MAX_CAND)].copy()


def cone_may_hit(o, d, theta: float, tri9) -> bool:
    """False only if no ray from o within angle theta of unit d can hit the
    triangle (its bounding sphere lies outside the cone): the per-pulse skip
    of oracle_simulate's brute force."""
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    tri = np.ascontiguousarray(tri9, np.float32).reshape(9)
    return bool(lib().oracle_cone_may_hit(_p(o), _p(d), theta, _p(tri)))


def bin_of(R: float, delta_ns: float):
    """(k, margin): k = floor(2R / c / Delta) (R8, R9), margin = distance of
    2R / c / Delta from the nearest integer."""
    m = ctypes.c_double()
    k = lib().oracle_bin_of(R, delta_ns, ctypes.byref(m))
    return int(k), m.value


def transmits(u: float, sigma: float, L: float):
    """(passes, margin): u < exp(-sigma L) (R17), margin |u - exp(-sigma L)|."""
    m = ctypes.c_double()
    r = lib().oracle_transmits(u, sigma, L, ctypes.byref(m))
    return bool(r), m.value


def philox4x32_10(ctr, key) -> np.ndarray:
    ctr = np.ascontiguousarray(ctr, np.uint32)
    key = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_p(ctr), _p(key), _p(out))
    return out


def transmission_u(seed: int, pulse: int, subray: int, voxel: int) -> float:
    return lib().oracle_transmission_u(seed, pulse, subray, voxel)


def g_function(lut, abs_dz: float) -> float:
    if lut is None:
        return lib().oracle_g_function(None, 0, abs_dz)
    lut = np.ascontiguousarray(lut, np.float32)
    return lib().oracle_g_function(_p(lut), lut.size, abs_dz)


def voxel_segments(o, d, n, origin, vs, t_max=float("inf")):
    o = np.ascontiguousarray(o, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    n = np.ascontiguousarray(n, np.uint32)
    origin = np.ascontiguousarray(origin, np.float64)
    cap = int(n.sum()) + 2
    ta = np.zeros(cap)
    tb = np.zeros(cap)
    vid = np.zeros(cap, np.uint32)
    k = lib().oracle_voxel_segments(_p(o), _p(d), _p(n), _p(origin), vs, t_max,
                                    _p(ta), _p(tb), _p(vid), cap)
    k = abs(int(k))
    return ta[:k].copy(), tb[:k].copy(), vid[:k].copy()


class OracleSurvey(ctypes.Structure):
    _fields_ = [("waypoints", _vp), ("n_waypoints", _u32), ("deflector", _u32),
                ("speed_m_s", _d), ("mount", _d * 9), ("mount_offset", _d * 3),
                ("head_rotation_rad_s", _d), ("pulse_freq_hz", _d), ("t0_s", _d),
                ("scan_freq_hz", _d), ("scan_angle_rad", _d), ("n_fibres", _u32),
                ("pad_", _u32)]


DEFLECTORS = {"polygon": 0, "fibre": 1, "oscillating": 2, "palmer": 3}
VOXEL_MODES = {"transmissive": 0, "opaque": 1, "scaled": 2}


def generate_pulses(survey, first: int, n: int):
    """(origin f32 [n,3], direction f32 [n,3], time f64 [n]) of pulses
    first .. first+n-1 of a survey (P:155 platforms, P:177 deflectors; R30).
    `survey`: workloads.Survey (or any object with its fields)."""
    wp = np.ascontiguousarray(survey.waypoints, np.float64).reshape(-1, 3)
    sv = OracleSurvey()
    sv.waypoints = _p(wp)
    sv.n_waypoints = wp.shape[0]
    sv.deflector = DEFLECTORS[survey.deflector] if isinstance(survey.deflector, str) \
        else int(survey.deflector)
    sv.speed_m_s = survey.speed_m_s
    sv.mount[:] = tuple(np.asarray(survey.mount, np.float64).reshape(9))
    sv.mount_offset[:] = tuple(np.asarray(survey.mount_offset, np.float64).reshape(3))
    sv.head_rotation_rad_s = survey.head_rotation_rad_s
    sv.pulse_freq_hz = survey.pulse_freq_hz
    sv.t0_s = survey.t0_s
    sv.scan_freq_hz = survey.scan_freq_hz
    sv.scan_angle_rad = survey.scan_angle_rad
    sv.n_fibres = survey.n_fibres
    o = np.zeros((n, 3), np.float32)
    d = np.zeros((n, 3), np.float32)
    t = np.zeros(n, np.float64)
    lib().oracle_generate_pulses(ctypes.byref(sv), first, n, _p(o), _p(d), _p(t))
    return o, d, t


def voxel_cube(n, origin, voxel_size, vid, pad, mode, pad_max=1.0, alpha=1.0, shift=0,
               seed=0):
    """(lo[3], side) of the opaque / scaled cube of voxel `vid` (P:231-239,
    Eq. 5; R31)."""
    nn = (_u32 * 3)(*n)
    org = (_d * 3)(*origin)
    lo = (_d * 3)()
    side = _d()
    lib().oracle_voxel_cube(nn, org, voxel_size, vid, pad,
                            VOXEL_MODES[mode] if isinstance(mode, str) else mode, pad_max,
                            alpha, shift, seed, lo, ctypes.byref(side))
    return np.array(lo[:]), side.value


def range_noise(seed: int, pulse: int, return_number: int) -> float:
    """Standard-normal ranging error of a return (R29, Box-Muller on
    Philox stream tag 1)."""
    return float(lib().oracle_range_noise(seed, pulse, return_number))


def fit_echo_width(W, k: int, delta_ns: float, pulse_length_ns: float):
    """(sigma, A, m) of the Gaussian fitted around bin k (R28)."""
    W = np.ascontiguousarray(W, np.float64)
    A = ctypes.c_double()
    m = ctypes.c_double()
    s = lib().oracle_fit_echo_width(_p(W), W.size, int(k), delta_ns, pulse_length_ns,
                                    ctypes.byref(A), ctypes.byref(m))
    return s, A.value, m.value


def waveform_bins(window_ns: float, bin_ns: float) -> int:
    return int(lib().oracle_waveform_bins(window_ns, bin_ns))


# ---------------------------------------------------------------- simulate
def _oracle_params(params) -> OracleParams:
    pr = OracleParams()
    for f, _ in OracleParams._fields_:
        if f != "pad_":
            setattr(pr, f, getattr(params, f, 0))
    # the threshold crosses the C ABI as a float (helios_scanner_params): the
    # oracle thresholds with that same value
    pr.detection_threshold = float(np.float32(params.detection_threshold))
    return pr


def waveform_peaks(params, A, k, prim, time_s: float = 0.0, pulse_id: int = 0):
    """Steps O6-O8 for ONE pulse from per-subray amplitudes A[s], bins k[s]
    (-1 = no event) and prims (R9-R13).  Returns a dict with
    n_returns, k0, waveform, ret_range/time/intensity/prim/number/width,
    ret_cand and the decision margins peak_margin / attr_margin."""
    pr = _oracle_params(params)
    N = int(params.subray_count)
    R = int(params.max_returns)
    A = np.ascontiguousarray(A, np.float64).reshape(N)
    k = np.ascontiguousarray(k, np.int64).reshape(N)
    prim = np.ascontiguousarray(prim, np.uint32).reshape(N)
    nb = waveform_bins(params.max_fullwave_range_ns, params.bin_width_ns)
    out = dict(waveform=np.zeros(nb), ret_range=np.zeros(R), ret_time=np.zeros(R),
               ret_intensity=np.zeros(R), ret_prim=np.zeros(R, np.uint32),
               ret_number=np.zeros(R, np.int32), ret_width=np.full(R, np.nan),
               ret_cand=np.full((R, MAX_ATTR), 0xFFFFFFFF, np.uint32))
    nr = ctypes.c_int32()
    k0 = ctypes.c_int64()
    pm = ctypes.c_double()
    am = ctypes.c_double()
    rc = lib().oracle_waveform_peaks(
        ctypes.byref(pr), _p(A), _p(k), _p(prim), time_s, pulse_id, ctypes.byref(nr),
        ctypes.byref(k0), _p(out["waveform"]), _p(out["ret_range"]), _p(out["ret_time"]),
        _p(out["ret_intensity"]), _p(out["ret_prim"]), _p(out["ret_number"]),
        _p(out["ret_width"]), _p(out["ret_cand"]), ctypes.byref(pm), ctypes.byref(am))
    if rc != 0:
        raise ValueError("oracle_waveform_peaks: invalid parameters")
    out.update(n_returns=nr.value, k0=k0.value, peak_margin=pm.value, attr_margin=am.value)
    return out


@dataclass
class OracleResult:
    n_returns: np.ndarray
    k0: np.ndarray
    waveform: np.ndarray | None
    ret_range: np.ndarray
    ret_time: np.ndarray
    ret_intensity: np.ndarray
    ret_prim: np.ndarray
    ret_number: np.ndarray
    ret_width: np.ndarray
    peak_margin: np.ndarray
    attr_margin: np.ndarray
    sub_range: np.ndarray
    sub_amp: np.ndarray
    sub_prim: np.ndarray
    sub_k: np.ndarray
    sub_ncand: np.ndarray
    sub_gap: np.ndarray
    sub_kmargin: np.ndarray
    sub_umargin: np.ndarray
    sub_cand: np.ndarray   # [n, N, MAX_CAND] triangle candidates (C-4), UINT32_MAX-padded
    ret_cand: np.ndarray   # [n, R, MAX_ATTR] attribution candidates (C-4), UINT32_MAX-padded


def simulate(scene, params, origins, directions, times, pulse_ids,
             n_threads: int | None = None, want_waveform: bool = True) -> OracleResult:
    """Run the oracle on the listed pulses.

    ``scene``: workloads.Scene; ``params``: workloads.ScannerParams;
    ``pulse_ids``: GLOBAL pulse ids (Philox counters, output ids).
    """
    L = lib()
    n = int(len(pulse_ids))
    N = int(params.subray_count)
    R = int(params.max_returns)
    nb = waveform_bins(params.max_fullwave_range_ns, params.bin_width_ns)
    if nb == 0:
        raise ValueError("bad bin width / window")
    tris = np.ascontiguousarray(scene.tri_xyz, np.float32).reshape(-1, 9)
    refl = None if scene.tri_reflectance is None else np.ascontiguousarray(
        scene.tri_reflectance, np.float32)
    pad = None if scene.voxel_pad is None else np.ascontiguousarray(scene.voxel_pad, np.float32)
    lut = None if scene.g_lut is None else np.ascontiguousarray(scene.g_lut, np.float32)
    sc = OracleScene()
    sc.tris = _p(tris)
    sc.refl = _p(refl)
    sc.n_tris = tris.shape[0]
    sc.pad = _p(pad)
    if pad is not None:
        nz, ny, nx = pad.shape
        sc.n[:] = (nx, ny, nz)
        sc.origin[:] = tuple(float(x) for x in scene.grid_origin)
        sc.voxel_size = float(scene.voxel_size)
    sc.g_lut = _p(lut)
    sc.n_lut = 0 if lut is None else lut.size
    sc.voxel_mode = VOXEL_MODES[getattr(scene, "voxel_mode", "transmissive")]
    sc.voxel_reflectance = float(getattr(scene, "voxel_reflectance", 0.5))
    sc.pad_max = float(getattr(scene, "pad_max", 1.0))
    sc.scale_alpha = float(getattr(scene, "scale_alpha", 1.0))
    sc.scale_shift = int(getattr(scene, "scale_shift", 0))
    pr = _oracle_params(params)
    o = np.ascontiguousarray(origins, np.float32).reshape(n, 3)
    d = np.ascontiguousarray(directions, np.float32).reshape(n, 3)
    t = np.ascontiguousarray(times, np.float64).reshape(n)
    ids = np.ascontiguousarray(pulse_ids, np.uint64).reshape(n)
    res = OracleResult(
        n_returns=np.zeros(n, np.int32), k0=np.zeros(n, np.int64),
        waveform=np.zeros((n, nb), np.float64) if want_waveform else None,
        ret_range=np.zeros((n, R)), ret_time=np.zeros((n, R)),
        ret_intensity=np.zeros((n, R)), ret_prim=np.zeros((n, R), np.uint32),
        ret_number=np.zeros((n, R), np.int32), ret_width=np.zeros((n, R)),
        peak_margin=np.zeros(n),
        attr_margin=np.zeros(n), sub_range=np.zeros((n, N)), sub_amp=np.zeros((n, N)),
        sub_prim=np.zeros((n, N), np.uint32), sub_k=np.zeros((n, N), np.int64),
        sub_ncand=np.zeros((n, N), np.int32), sub_gap=np.zeros((n, N)),
        sub_kmargin=np.zeros((n, N)), sub_umargin=np.zeros((n, N)),
        sub_cand=np.zeros((n, N, MAX_CAND), np.uint32),
        ret_cand=np.zeros((n, R, MAX_ATTR), np.uint32))
    out = OracleOutputs()
    for f, _ in OracleOutputs._fields_:
        setattr(out, f, _p(getattr(res, f)))
    if n_threads is None:
        n_threads = os.cpu_count() or 1
    rc = L.oracle_simulate(ctypes.byref(sc), ctypes.byref(pr), _p(o), _p(d), _p(t),
                           _p(ids), n, int(n_threads), ctypes.byref(out))
    if rc != 0:
        raise ValueError("oracle_simulate: invalid parameters")
    return res
