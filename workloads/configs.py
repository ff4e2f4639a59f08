"""Seeded synthetic workloads C1..C5 (BASELINE.json ``configs``).

The recipes follow SURVEY.md s.8(d) D-2 and are restated in DESIGN.md s.5.
Randomness: numpy ``default_rng(SeedSequence([seed, config_id, stream]))``
with one stream per quantity, so every array is reproducible on any machine.
Triangle ids follow generation order.  Pulses are generated on demand for any
contiguous index range (``Workload.pulses(start, count)``), so a 100 M-pulse
config never has to exist in host memory at once.

Nothing here implements any step of the method (no subrays, intersection,
radiometry, waveforms or peaks): these are inputs only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable

import numpy as np

C_LIGHT = 299792458.0  # m/s, only to express "a 200 m window" in ns (config input)


def window_ns_for_range(metres: float) -> float:
    """Two-way time of flight over ``metres`` of range, in ns (config input)."""
    return 2.0 * metres / C_LIGHT * 1e9


@dataclass
class Scene:
    tri_xyz: np.ndarray                 # [n][3][3] float32
    tri_reflectance: np.ndarray | None  # [n] float32
    voxel_pad: np.ndarray | None = None  # [nz][ny][nx] float32
    grid_origin: tuple = (0.0, 0.0, 0.0)
    voxel_size: float = 1.0
    g_lut: np.ndarray | None = None
    # voxel interpretation (Eq. 5; R31)
    voxel_mode: str = "transmissive"   # transmissive | opaque | scaled
    voxel_reflectance: float = 0.5     # rho of opaque / scaled cubes
    pad_max: float = 1.0               # PAD_max of Eq. 5
    scale_alpha: float = 1.0           # alpha of Eq. 5
    scale_shift: int = 0               # 1: reproducible random shift of scaled cubes

    @property
    def n_tris(self) -> int:
        return int(self.tri_xyz.shape[0])


@dataclass
class ScannerParams:
    divergence_rad: float = 0.3e-3
    subray_count: int = 19
    pulse_length_ns: float = 4.0
    bin_width_ns: float = 1.0
    max_fullwave_range_ns: float = field(default_factory=lambda: window_ns_for_range(200.0))
    detection_threshold: float = 0.05
    max_returns: int = 7
    peak_power_w: float = 1.0
    efficiency: float = 1.0
    receiver_diameter_m: float = 1.0
    wavelength_nm: float = 1064.0
    beam_waist_m: float = 0.0
    focus_range_m: float = 0.0
    seed: int = 0
    fit_echo_width: int = 0  # optional Gaussian echo-width fit
    reserved_: int = 0
    range_noise_sd_m: float = 0.0  # ranging error sigma, 0 -> none


@dataclass
class Survey:
    """A platform + scanner description for on-device pulse generation
    (NEXT f2; P:155 platforms, P:177 deflectors; R30).  Plain data:
    the generators live in the oracle and in the CUDA library."""
    waypoints: np.ndarray            # [n][3] m; one point = Static platform
    pulse_freq_hz: float
    deflector: str = "polygon"       # polygon | fibre | oscillating | palmer
    scan_freq_hz: float = 100.0
    scan_angle_rad: float = 0.5      # half-amplitude, or Palmer cone angle
    speed_m_s: float = 0.0           # LinearPath speed (> 0 with >= 2 waypoints)
    t0_s: float = 0.0
    n_fibres: int = 0                # fibre deflector: lines per sweep
    head_rotation_rad_s: float = 0.0
    mount: np.ndarray = field(default_factory=lambda: np.eye(3))
    mount_offset: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class Workload:
    name: str
    scene: Scene
    params: ScannerParams
    n_pulses: int
    _pulse_fn: Callable[[np.ndarray], tuple] = field(repr=False, default=None)
    # the same pulses as surveys (NEXT f2): [(Survey, first global id, count)],
    # survey pulse g <-> global id first + g; None if not survey-expressible
    surveys: list | None = None
    # generator facts for test stratification (C5: building circles, tree
    # positions, heightfield, pulses per flight line); inputs only
    meta: dict | None = None

    def pulses(self, start: int = 0, count: int | None = None):
        """(origins f32 [n,3], directions f32 [n,3], times f64 [n]) for the
        global pulse ids start .. start+count-1."""
        if count is None:
            count = self.n_pulses - start
        idx = np.arange(start, start + count, dtype=np.int64)
        return self.pulses_at(idx)

    def pulses_at(self, ids: np.ndarray):
        o, d, t = self._pulse_fn(np.asarray(ids, np.int64))
        return (np.ascontiguousarray(o, np.float32), np.ascontiguousarray(d, np.float32),
                np.ascontiguousarray(t, np.float64))


def _rng(seed: int, cfg: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, cfg, stream]))


# ---------------------------------------------------------------- geometry kit
def _square(half: float, z: float) -> np.ndarray:
    v = np.array([[-half, -half, z], [half, -half, z], [half, half, z], [-half, half, z]],
                 np.float64)
    return np.stack([v[[0, 1, 2]], v[[0, 2, 3]]]).astype(np.float32)


def fbm_heightfield(n: int, base_period: float, amp: float, rng: np.random.Generator,
                    octaves: int = 6) -> np.ndarray:
    """h[iy, ix] at 1 m spacing: amp * sum_o 0.5^o V_o / sum_o 0.5^o, V_o value
    noise (lattice values 2u-1, smoothstep bilinear) at 2^o / base_period m^-1."""
    x = np.arange(n, dtype=np.float64)
    total = np.zeros((n, n))
    wsum = 0.0
    for o in range(octaves):
        f = (2.0 ** o) / base_period
        m = int(math.ceil((n - 1) * f)) + 2
        lat = 2.0 * rng.random((m, m)) - 1.0
        g = x * f
        i0 = np.floor(g).astype(np.int64)
        t = g - i0
        s = t * t * (3.0 - 2.0 * t)
        # rows = y, cols = x
        a = lat[np.ix_(i0, i0)]
        b = lat[np.ix_(i0, i0 + 1)]
        c = lat[np.ix_(i0 + 1, i0)]
        d = lat[np.ix_(i0 + 1, i0 + 1)]
        sx = s[None, :]
        sy = s[:, None]
        v = (a * (1 - sx) + b * sx) * (1 - sy) + (c * (1 - sx) + d * sx) * sy
        total += (0.5 ** o) * v
        wsum += 0.5 ** o
    return amp * total / wsum


def heightfield_triangles(h: np.ndarray) -> np.ndarray:
    """Each cell -> (v00, v10, v11), (v00, v11, v01): lower-left to upper-right
    diagonal.  Returns [2 (n-1)^2][3][3] float32, cell-major (y, x)."""
    n = h.shape[0]
    iy, ix = np.meshgrid(np.arange(n - 1), np.arange(n - 1), indexing="ij")
    iy = iy.ravel()
    ix = ix.ravel()

    def v(dx, dy):
        return np.stack([(ix + dx).astype(np.float64), (iy + dy).astype(np.float64),
                         h[iy + dy, ix + dx]], axis=-1)

    v00, v10, v11, v01 = v(0, 0), v(1, 0), v(1, 1), v(0, 1)
    t0 = np.stack([v00, v10, v11], axis=1)
    t1 = np.stack([v00, v11, v01], axis=1)
    out = np.empty((ix.size * 2, 3, 3), np.float32)
    out[0::2] = t0
    out[1::2] = t1
    return out


def _orthonormal(nrm: np.ndarray):
    helper = np.where(np.abs(nrm[:, 2:3]) > 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 0, 1.0]]))
    e1 = np.cross(nrm, helper)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(nrm, e1)
    return e1, e2


def trees(rng_tree: np.random.Generator, rng_leaf: np.random.Generator, xy: np.ndarray,
          base_z: np.ndarray, leaves_lo: int, leaves_hi: int):
    """Trees of SURVEY D-2 C3: 16-gon trunk prism (32 side triangles, rho 0.25)
    + leaves (equilateral, side 5 cm, random orientation, uniform in an
    ellipsoidal crown, rho 0.45).  Returns (tris f32 [n,3,3], refl f32 [n])."""
    nt = xy.shape[0]
    r_trunk = rng_tree.uniform(0.1, 0.4, nt)
    H = rng_tree.uniform(10.0, 25.0, nt)
    ax = rng_tree.uniform(2.0, 5.0, nt)
    ay = rng_tree.uniform(2.0, 5.0, nt)
    n_leaves = rng_leaf.integers(leaves_lo, leaves_hi + 1, nt)
    out_t, out_r = [], []
    ang = 2 * np.pi * np.arange(17) / 16.0
    for k in range(nt):
        x, y, z0 = xy[k, 0], xy[k, 1], base_z[k]
        ring = np.stack([x + r_trunk[k] * np.cos(ang), y + r_trunk[k] * np.sin(ang)], -1)
        b = np.concatenate([ring, np.full((17, 1), z0)], 1)
        t = np.concatenate([ring, np.full((17, 1), z0 + H[k])], 1)
        side = np.empty((32, 3, 3))
        side[0::2] = np.stack([b[:-1], b[1:], t[1:]], 1)
        side[1::2] = np.stack([b[:-1], t[1:], t[:-1]], 1)
        out_t.append(side.astype(np.float32))
        out_r.append(np.full(32, 0.25, np.float32))
        # leaves
        m = int(n_leaves[k])
        cen = np.empty((0, 3))
        while cen.shape[0] < m:
            p = rng_leaf.uniform(-1.0, 1.0, (2 * (m - cen.shape[0]) + 16, 3))
            p = p[(p * p).sum(1) <= 1.0]
            cen = np.concatenate([cen, p])
        cen = cen[:m] * np.array([ax[k], ay[k], 0.35 * H[k]]) + np.array(
            [x, y, z0 + 0.65 * H[k]])
        nrm = rng_leaf.normal(size=(m, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        alpha = rng_leaf.uniform(0.0, 2 * np.pi, m)
        e1, e2 = _orthonormal(nrm)
        rad = 0.05 / math.sqrt(3.0)
        verts = []
        for j in range(3):
            a = alpha + 2 * np.pi * j / 3.0
            verts.append(cen + rad * (np.cos(a)[:, None] * e1 + np.sin(a)[:, None] * e2))
        out_t.append(np.stack(verts, 1).astype(np.float32))
        out_r.append(np.full(m, 0.45, np.float32))
    return np.concatenate(out_t), np.concatenate(out_r)


def boxes(rng: np.random.Generator, n: int, h: np.ndarray, lo: float, hi: float):
    """Extruded yawed boxes (C5 buildings): 4 walls x 2 + roof x 2 triangles."""
    cx = rng.uniform(lo, hi, n)
    cy = rng.uniform(lo, hi, n)
    sx = rng.uniform(4.0, 12.0, n)
    sy = rng.uniform(4.0, 12.0, n)
    yaw = np.radians(rng.uniform(0.0, 90.0, n))
    height = rng.uniform(5.0, 80.0, n)
    refl = rng.uniform(0.1, 0.6, n)
    lx = np.array([-0.5, 0.5, 0.5, -0.5])
    ly = np.array([-0.5, -0.5, 0.5, 0.5])
    c, s = np.cos(yaw)[:, None], np.sin(yaw)[:, None]
    px = cx[:, None] + c * (lx * sx[:, None]) - s * (ly * sy[:, None])
    py = cy[:, None] + s * (lx * sx[:, None]) + c * (ly * sy[:, None])
    nmax = h.shape[0] - 1
    hx = np.clip(np.rint(px).astype(np.int64), 0, nmax)
    hy = np.clip(np.rint(py).astype(np.int64), 0, nmax)
    base = h[hy, hx].min(1) - 0.5
    top = base + height
    bot = np.stack([px, py, np.repeat(base[:, None], 4, 1)], -1)  # [n,4,3]
    tp = np.stack([px, py, np.repeat(top[:, None], 4, 1)], -1)
    tris = np.empty((n, 10, 3, 3))
    for k in range(4):
        k1 = (k + 1) % 4
        tris[:, 2 * k] = np.stack([bot[:, k], bot[:, k1], tp[:, k1]], 1)
        tris[:, 2 * k + 1] = np.stack([bot[:, k], tp[:, k1], tp[:, k]], 1)
    tris[:, 8] = np.stack([tp[:, 0], tp[:, 1], tp[:, 2]], 1)
    tris[:, 9] = np.stack([tp[:, 0], tp[:, 2], tp[:, 3]], 1)
    radius = 0.5 * np.hypot(sx, sy)
    return (tris.reshape(-1, 3, 3).astype(np.float32),
            np.repeat(refl, 10).astype(np.float32), np.stack([cx, cy, radius], 1))


def _scaled_flight(alt: float, fov_deg: float, width: float, scale: float):
    """Full size: (alt, fov) as stated.  Reduced parity scenes: fly lower and
    narrow the swath so it stays on the smaller scene (most subrays hit)."""
    if scale >= 1.0:
        return alt, fov_deg
    a = max(alt * scale, 120.0)
    return a, min(fov_deg, float(np.degrees(np.arctan(0.42 * width / a))))


def _dir_sawtooth(theta: np.ndarray) -> np.ndarray:
    """Across-track (x) deflection, nadir-looking: (sin th, 0, -cos th)."""
    return np.stack([np.sin(theta), np.zeros_like(theta), -np.cos(theta)], -1)


# ---------------------------------------------------------------- configs
def _c1(scale: float, seed: int):
    tri = _square(50.0, 0.0)
    scene = Scene(tri, np.full(2, 0.5, np.float32))
    params = ScannerParams(divergence_rad=0.3e-3, subray_count=19, bin_width_ns=1.0, seed=seed)
    side = 100

    def fn(idx):
        i = idx // side
        j = idx % side
        zen = np.radians(100.0 + 70.0 * i / 99.0)
        az = np.radians(3.6 * j)
        d = np.stack([np.sin(zen) * np.cos(az), np.sin(zen) * np.sin(az), np.cos(zen)], -1)
        o = np.broadcast_to(np.array([0.0, 0.0, 10.0]), d.shape)
        return (o.astype(np.float32), d.astype(np.float32), idx.astype(np.float64) * 1e-5)

    return scene, params, side * side, fn, None


def _c2(scale: float, seed: int):
    n = max(8, int(round(512 * scale)))
    h = fbm_heightfield(n, 128.0 * n / 512.0, 40.0, _rng(seed, 2, 1))
    tri = heightfield_triangles(h)
    refl = _rng(seed, 2, 2).uniform(0.1, 0.6, tri.shape[0]).astype(np.float32)
    scene = Scene(tri, refl)
    params = ScannerParams(divergence_rad=0.25e-3, subray_count=19, bin_width_ns=1.0, seed=seed)
    n_pulses = max(1000, int(round(1_000_000 * scale * scale)))
    dur = (n - 1) / 60.0
    prf = n_pulses / dur
    xc = (n - 1) / 2.0
    # reduced scenes keep the swath on the (smaller) DTM
    alt, fov = _scaled_flight(500.0, 30.0, n, scale)

    def fn(idx):
        t = idx.astype(np.float64) / prf
        th = np.radians(-fov + 2 * fov * np.mod(100.0 * t, 1.0))
        d = _dir_sawtooth(th)
        o = np.stack([np.full_like(t, xc), 60.0 * t, np.full_like(t, alt)], -1)
        return o.astype(np.float32), d.astype(np.float32), t

    sv = Survey(waypoints=np.array([[xc, 0.0, alt], [xc, n - 1.0, alt]]), pulse_freq_hz=prf,
                deflector="polygon", scan_freq_hz=100.0, scan_angle_rad=math.radians(fov),
                speed_m_s=60.0)
    return scene, params, n_pulses, fn, [(sv, 0, n_pulses)]


def _c3(scale: float, seed: int, n_trees: int | None = None, leaves=(8000, 20000)):
    ground = _square(100.0, 0.0)
    if n_trees is None:
        n_trees = max(1, int(round(300 * scale)))
    rt = _rng(seed, 3, 3)
    xy = np.empty((0, 2))
    while xy.shape[0] < n_trees:
        p = rt.uniform(-95.0, 95.0, (2 * n_trees, 2))
        p = p[np.hypot(p[:, 0], p[:, 1]) >= 3.0]
        xy = np.concatenate([xy, p])
    xy = xy[:n_trees]
    lo, hi = leaves
    if scale < 1.0:
        lo, hi = max(10, int(lo * scale)), max(20, int(hi * scale))
    tt, tr = trees(rt, _rng(seed, 3, 4), xy, np.zeros(n_trees), lo, hi)
    tri = np.concatenate([ground, tt])
    refl = np.concatenate([np.full(2, 0.3, np.float32), tr])
    scene = Scene(tri, refl)
    params = ScannerParams(divergence_rad=0.3e-3, subray_count=37, bin_width_ns=1.0,
                           detection_threshold=0.05, seed=seed)
    n_az = max(2, int(round(7200 * scale)))
    n_el = max(2, int(round(2400 * scale)))
    step_az = 360.0 / n_az
    step_el = 120.0 / n_el

    def fn(idx):
        j = idx // n_el
        i = idx % n_el
        az = np.radians(step_az * j)
        zen = np.radians(30.0 + step_el * i)
        d = np.stack([np.sin(zen) * np.cos(az), np.sin(zen) * np.sin(az), np.cos(zen)], -1)
        o = np.broadcast_to(np.array([0.0, 0.0, 1.5]), d.shape)
        return o.astype(np.float32), d.astype(np.float32), idx.astype(np.float64) * 1e-6

    return scene, params, n_az * n_el, fn, None


def _c4(scale: float, seed: int):
    nxy = max(8, int(round(400 * scale)))
    nz = 40
    vs = 0.5
    half = nxy * vs / 2.0
    org = (-half, -half, 0.0)
    rc = _rng(seed, 4, 5)
    n_crowns = max(1, int(round(200 * scale * scale)))
    cx = rc.uniform(-half + 5.0, half - 5.0, n_crowns) if half > 6 else np.zeros(n_crowns)
    cy = rc.uniform(-half + 5.0, half - 5.0, n_crowns) if half > 6 else np.zeros(n_crowns)
    cz = rc.uniform(8.0, 14.0, n_crowns)
    ah = rc.uniform(2.0, 6.0, n_crowns)
    av = rc.uniform(2.0, 5.0, n_crowns)
    inside = np.zeros((nz, nxy, nxy), bool)
    cxs = org[0] + (np.arange(nxy) + 0.5) * vs
    czs = org[2] + (np.arange(nz) + 0.5) * vs
    for k in range(n_crowns):
        # only the crown's bounding box of voxels can be inside it
        x0, x1 = np.searchsorted(cxs, [cx[k] - ah[k], cx[k] + ah[k]])
        y0, y1 = np.searchsorted(cxs, [cy[k] - ah[k], cy[k] + ah[k]])
        z0, z1 = np.searchsorted(czs, [cz[k] - av[k], cz[k] + av[k]])
        dz = ((czs[z0:z1] - cz[k]) / av[k]) ** 2
        dx = ((cxs[x0:x1] - cx[k]) / ah[k]) ** 2
        dy = ((cxs[y0:y1] - cy[k]) / ah[k]) ** 2
        inside[z0:z1, y0:y1, x0:x1] |= (
            dz[:, None, None] + dy[None, :, None] + dx[None, None, :]) <= 1.0
    pad = np.zeros((nz, nxy, nxy), np.float32)
    pad[inside] = _rng(seed, 4, 6).beta(2.0, 5.0, int(inside.sum())).astype(np.float32)
    scene = Scene(_square(half, 0.0), np.full(2, 0.3, np.float32), pad, org, vs, None)
    params = ScannerParams(divergence_rad=0.3e-3, subray_count=19, bin_width_ns=0.5, seed=seed)
    n_pulses = max(1000, int(round(5_000_000 * scale * scale)))
    speed = 5.0
    dur = 2 * half / speed
    prf = n_pulses / dur
    fov = 45.0 if scale >= 1.0 else min(45.0, float(np.degrees(np.arctan(0.42 * 2 * half / 60.0))))

    def fn(idx):
        t = idx.astype(np.float64) / prf
        th = np.radians(-fov + 2 * fov * np.mod(50.0 * t, 1.0))
        d = _dir_sawtooth(th)
        o = np.stack([np.zeros_like(t), -half + speed * t, np.full_like(t, 80.0)], -1)
        return o.astype(np.float32), d.astype(np.float32), t

    sv = Survey(waypoints=np.array([[0.0, -half, 80.0], [0.0, half, 80.0]]), pulse_freq_hz=prf,
                deflector="polygon", scan_freq_hz=50.0, scan_angle_rad=math.radians(fov),
                speed_m_s=speed)
    return scene, params, n_pulses, fn, [(sv, 0, n_pulses)]


def _c5(scale: float, seed: int):
    n = max(16, int(round(2048 * scale)))
    h = fbm_heightfield(n, 256.0 * n / 2048.0, 40.0, _rng(seed, 5, 1))
    dtm = heightfield_triangles(h)
    dtm_refl = _rng(seed, 5, 2).uniform(0.1, 0.6, dtm.shape[0]).astype(np.float32)
    n_boxes = max(1, int(round(40_000 * scale * scale)))
    bt, br, circ = boxes(_rng(seed, 5, 7), n_boxes, h, 10.0, n - 11.0)
    # trees: uniform, outside building bounding circles, based on the terrain
    n_trees = max(1, int(round(2000 * scale * scale)))
    mask = np.zeros((n, n), bool)
    gy, gx = np.mgrid[-9:10, -9:10]
    for cx, cy, r in circ:
        ix = int(round(cx)) + gx
        iy = int(round(cy)) + gy
        ok = (np.hypot(ix - cx, iy - cy) <= r) & (ix >= 0) & (ix < n) & (iy >= 0) & (iy < n)
        mask[iy[ok], ix[ok]] = True
    rt = _rng(seed, 5, 3)
    xy = np.empty((0, 2))
    while xy.shape[0] < n_trees:
        p = rt.uniform(10.0, n - 11.0, (2 * n_trees, 2))
        keep = ~mask[np.rint(p[:, 1]).astype(int), np.rint(p[:, 0]).astype(int)]
        xy = np.concatenate([xy, p[keep]])
    xy = xy[:n_trees]
    base = h[np.rint(xy[:, 1]).astype(int), np.rint(xy[:, 0]).astype(int)] - 0.2
    lo, hi = (18000, 23000) if scale >= 1.0 else (max(10, int(18000 * scale)),
                                                  max(20, int(23000 * scale)))
    tt, tr = trees(rt, _rng(seed, 5, 4), xy, base, lo, hi)
    tri = np.concatenate([dtm, bt, tt])
    refl = np.concatenate([dtm_refl, br, tr])
    scene = Scene(tri, refl)
    params = ScannerParams(divergence_rad=0.5e-3, subray_count=91, bin_width_ns=1.0, seed=seed)
    n_pulses = max(2000, int(round(100_000_000 * scale * scale)))
    per_line = n_pulses // 2
    n_pulses = 2 * per_line
    line_dur = (n - 1) / 60.0
    prf = per_line / line_dur
    xs = (600.0 * (n / 2048.0), 1448.0 * (n / 2048.0))
    alt, fov = _scaled_flight(1000.0, 35.0, 0.8 * n, scale)

    def fn(idx):
        line = idx // per_line
        m = idx % per_line
        tl = m.astype(np.float64) / prf
        t = line * line_dur + tl
        th = np.radians(-fov + 2 * fov * np.mod(200.0 * t, 1.0))
        d = _dir_sawtooth(th)
        x = np.where(line == 0, xs[0], xs[1])
        o = np.stack([x, 60.0 * tl, np.full_like(tl, alt)], -1)
        return o.astype(np.float32), d.astype(np.float32), t

    svs = [(Survey(waypoints=np.array([[x, 0.0, alt], [x, n - 1.0, alt]]), pulse_freq_hz=prf,
                   deflector="polygon", scan_freq_hz=200.0, scan_angle_rad=math.radians(fov),
                   speed_m_s=60.0, t0_s=k * line_dur), k * per_line, per_line)
           for k, x in enumerate(xs)]
    meta = {"buildings": circ, "trees": xy, "heights": h, "per_line": per_line, "fov_deg": fov}
    return scene, params, n_pulses, fn, svs, meta


def _prism(cx, cy, z0, h, r, sides, yaw, cap=True):
    """Vertical prism over a regular `sides`-gon of circumradius r (walls, and
    the roof as a triangle fan when cap)."""
    a = yaw + 2 * np.pi * np.arange(sides) / sides
    ring = np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], -1)
    out = []
    for k in range(sides):
        p0, p1 = ring[k], ring[(k + 1) % sides]
        b0, b1 = [*p0, z0], [*p1, z0]
        t0, t1 = [*p0, z0 + h], [*p1, z0 + h]
        out += [[b0, b1, t1], [b0, t1, t0]]
        if cap:
            out.append([[cx, cy, z0 + h], t0, t1])
    return np.array(out)


def _pyramid(cx, cy, z0, h, half, yaw):
    a = yaw + np.pi / 4 + np.pi / 2 * np.arange(4)
    r = half * np.sqrt(2.0)
    base = np.stack([cx + r * np.cos(a), cy + r * np.sin(a), np.full(4, z0)], -1)
    apex = [cx, cy, z0 + h]
    return np.array([[base[k], base[(k + 1) % 4], apex] for k in range(4)])


def _c6(scale: float, seed: int):
    """MLS stand-in for Table 3 Scene 2: a car driving 208 m at
    20 m/s between downtown buildings modelled as prisms, cylinders and
    pyramids; oblique-mounted 330-degree line scanner (VUX-1UAV-like: 550 kHz,
    200 lines/s, 0.5 mrad); paper waveform defaults beamSampleQuality 3
    (37 subrays), bin 0.25 ns, 100 bins."""
    rng = _rng(seed, 6, 1)
    length = 208.0
    objs, refl = [], []
    n_slots = max(2, int(round(15 * scale)))
    for side in (-1.0, 1.0):
        for row, (ylo, yhi) in enumerate(((12.0, 24.0), (28.0, 42.0))):
            for k in range(n_slots):
                cx = (k + 0.5) * length / n_slots + rng.uniform(-1.5, 1.5)
                cy = side * rng.uniform(ylo + 5.0, yhi - 5.0)
                kind = rng.integers(0, 3)
                yaw = rng.uniform(0, np.pi / 2)
                if kind == 0:    # box prism
                    t = _prism(cx, cy, 0.0, rng.uniform(6.0, 40.0), rng.uniform(3.5, 6.5), 4, yaw)
                elif kind == 1:  # cylinder (24-gon)
                    t = _prism(cx, cy, 0.0, rng.uniform(5.0, 30.0), rng.uniform(3.0, 5.5), 24, yaw)
                else:            # pyramid
                    t = _pyramid(cx, cy, 0.0, rng.uniform(5.0, 20.0), rng.uniform(3.0, 6.0), yaw)
                objs.append(t)
                refl.append(np.full(len(t), rng.uniform(0.1, 0.6)))
    ground = np.array([[[-50, -60, 0.0], [260, -60, 0.0], [260, 60, 0.0]],
                       [[-50, -60, 0.0], [260, 60, 0.0], [-50, 60, 0.0]]])
    tri = np.concatenate([ground] + objs).astype(np.float32)
    rf = np.concatenate([np.full(2, 0.3)] + refl).astype(np.float32)
    scene = Scene(tri, rf)
    params = ScannerParams(divergence_rad=0.5e-3, subray_count=37, bin_width_ns=0.25,
                           max_fullwave_range_ns=25.0, seed=seed)
    speed, prf, f = 20.0, 550_000.0, 200.0
    A = math.radians(165.0)                      # 330-degree field of view
    yaw_m = math.radians(45.0)                   # oblique mount: scan plane turned 45 deg
    mount = np.array([[math.cos(yaw_m), -math.sin(yaw_m), 0.0],
                      [math.sin(yaw_m), math.cos(yaw_m), 0.0], [0.0, 0.0, 1.0]])
    n_pulses = max(2000, int(round(length / speed * prf * scale)))
    dur = n_pulses / prf

    def fn(idx):
        t = idx.astype(np.float64) / prf
        u = np.mod(f * t, 1.0)
        th = -A + 2.0 * A * u
        s = np.stack([np.zeros_like(th), -np.sin(th), -np.cos(th)], -1)
        d = s @ mount.T
        o = np.stack([speed * t, np.zeros_like(t), np.full_like(t, 2.0)], -1)
        return o.astype(np.float32), d.astype(np.float32), t

    sv = Survey(waypoints=np.array([[0.0, 0.0, 2.0], [speed * dur, 0.0, 2.0]]), pulse_freq_hz=prf,
                deflector="polygon", scan_freq_hz=f, scan_angle_rad=A, speed_m_s=speed,
                mount=mount)
    return scene, params, n_pulses, fn, [(sv, 0, n_pulses)]


CONFIGS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5": _c5, "C6": _c6}

DESCRIPTIONS = {
    "C1": "tiny TLS plane: 2 tris, 10k pulses, 19 subrays, 0.3 mrad, 1 ns bins",
    "C2": "ALS over 512^2 fBm DTM (522,242 tris), 1M pulses, 19 subrays, 0.25 mrad",
    "C3": "TLS forest mesh (~4.2M tris), 17.28M pulses, 37 subrays, thr 0.05",
    "C4": "transmissive voxel canopy 400x400x40 (6.4M voxels) + ground, 5M pulses, "
          "19 subrays, 0.5 ns bins",
    "C5": "ALS city+terrain (~49.8M tris), 100M pulses, 91 subrays (hex q=5), 0.5 mrad",
    "C6": "MLS street of prisms / cylinders / pyramids (Table 3 Scene 2 stand-in), 5.72M "
          "pulses, 37 subrays, 0.25 ns bins x 100, oblique 330-degree line scanner",
}


def make_workload(name: str, scale: float = 1.0, seed: int = 0, **overrides) -> Workload:
    """Build config ``name`` (C1..C5).  ``scale`` < 1 shrinks the scene and the
    pulse grid for parity tests (the oracle is brute force); ``overrides``
    replace ScannerParams fields (e.g. subray_count=93 for the C5 variant)."""
    name = name.upper()
    built = CONFIGS[name](scale, seed)
    scene, params, n_pulses, fn, surveys = built[:5]
    meta = built[5] if len(built) > 5 else None
    if overrides:
        params = replace(params, **overrides)
    return Workload(name if scale == 1.0 else f"{name}@{scale:g}", scene, params, n_pulses, fn,
                    surveys, meta)
