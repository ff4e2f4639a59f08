"""Pins of the oracle's parity metadata: the candidate
sets and decision margins that decide which subrays / pulses the comparator
may exempt.  Each flag is built to fire on a constructed near-tie and checked
NOT to fire a little away from it, so a too-generous (or too-strict) margin
shows up here rather than as silently widened exemptions."""
import math

import numpy as np
import pytest

import oracle
from workloads import ScannerParams

C = 299792458.0


def _quad(z, half=5.0):
    """Two triangles of the square [-half, half]^2 at height z (shared diagonal)."""
    v = np.array([[-half, -half, z], [half, -half, z], [half, half, z], [-half, half, z]],
                 np.float32)
    return np.stack([v[[0, 1, 2]], v[[0, 2, 3]]])


# ---------------------------------------------------------------- candidates
@pytest.mark.parametrize("dz,expect", [(0.0, 4), (4.0e-7, 4), (9.0e-7, 4), (1.2e-6, 2),
                                       (2.0e-6, 2), (1e-3, 2)])
def test_candidate_set_of_two_parallel_planes(dz, expect):
    # ray from (0.3, 0.1, 1) straight down: hits the plane at z = dz (t = 1 - dz)
    # and the plane at z = 0 (t = 1); each plane is two triangles, the ray is
    # off the diagonal, so one triangle per plane is hit.  Candidates within
    # 1e-6 m: both planes' triangles iff dz <= 1e-6 (fp32 z: dz as rounded)
    tris = np.concatenate([_quad(0.0), _quad(np.float32(dz))]).reshape(-1, 9)
    o = np.array([0.3, 0.1, 1.0])
    d = np.array([0.0, 0.0, -1.0])
    idx, t, nc, cand = oracle.nearest_candidates(o, d, tris)
    zf = float(np.float32(dz))
    near = 2 if zf > 0 else 0  # the upper plane's triangle (ids 2, 3) is nearer
    assert t == pytest.approx(1.0 - zf, abs=1e-12)
    if expect == 4:  # both planes within 1e-6: two hit triangles listed by (t, id)
        assert nc == 2
        assert list(cand) == ([0, 2] if zf == 0 else [2, 0])
        assert idx == cand[0]
    else:
        assert nc == 1 and list(cand) == [near] and idx == near


def test_candidate_set_on_a_shared_edge_and_overflow():
    # ray exactly along the shared diagonal of a quad: both triangles at the
    # same t; the lower id wins (R22) and both are candidates
    tris = _quad(0.0).reshape(-1, 9)
    idx, t, nc, cand = oracle.nearest_candidates([1.0, 1.0, 2.0], [0, 0, -1.0], tris)
    assert (idx, nc, list(cand)) == (0, 2, [0, 1]) and t == 2.0
    # ten stacked planes 1e-7 m apart: ten candidates, the nearest eight listed
    stack = np.concatenate([_quad(np.float32(k * 1e-7))[:1] for k in range(10)]).reshape(-1, 9)
    idx, t, nc, cand = oracle.nearest_candidates([0.3, -0.2, 1.0], [0, 0, -1.0], stack)
    zs = np.float32(np.arange(10) * 1e-7)
    order = np.argsort(-zs, kind="stable")  # nearest = highest plane
    assert nc == 10 and idx == order[0]
    assert list(cand) == list(order[:oracle.MAX_CAND])


def test_simulate_exports_the_candidate_sets():
    # one subray through the diagonal of the quad and one off it
    from workloads.configs import Scene
    sc = Scene(tri_xyz=_quad(0.0), tri_reflectance=np.full(2, 0.5, np.float32))
    p = ScannerParams(subray_count=1, divergence_rad=1e-4)
    o = np.array([[1.0, 1.0, 3.0], [2.0, -1.0, 3.0]], np.float32)
    d = np.array([[0, 0, -1], [0, 0, -1]], np.float32)
    r = oracle.simulate(sc, p, o, d, np.zeros(2), np.arange(2, dtype=np.uint64))
    assert list(r.sub_ncand[:, 0]) == [2, 1]
    assert list(r.sub_cand[0, 0, :3]) == [0, 1, 0xFFFFFFFF]
    assert list(r.sub_cand[1, 0, :2]) == [r.sub_prim[1, 0], 0xFFFFFFFF]


# ---------------------------------------------------------------- k margin
@pytest.mark.parametrize("delta", [1.0, 0.5, 0.25])
def test_bin_margin_fires_only_at_bin_edges(delta):
    half = 0.5 * C * delta * 1e-9
    for k in (3, 667, 6671):
        kk, m = oracle.bin_of(k * half, delta)  # on a bin edge: margin at rounding level
        assert m <= 1e-9 and kk in (k - 1, k)
        kk, m = oracle.bin_of((k + 1e-6) * half, delta)  # 1e-6 bins inside: no flag
        assert kk == k and m == pytest.approx(1e-6, rel=1e-3) and m > 1e-9
        kk, m = oracle.bin_of((k + 0.5) * half, delta)
        assert kk == k and m == pytest.approx(0.5, abs=1e-9)
        kk, m = oracle.bin_of((k - 0.3) * half, delta)
        assert kk == k - 1 and m == pytest.approx(0.3, abs=1e-9)


def test_simulate_records_the_bin_margin_of_its_range():
    from workloads.configs import Scene
    sc = Scene(tri_xyz=_quad(0.0, 50.0), tri_reflectance=np.full(2, 0.5, np.float32))
    p = ScannerParams(subray_count=7, divergence_rad=2e-3)
    n = 40
    o = np.stack([np.linspace(-3, 3, n), np.zeros(n), np.linspace(5.0, 9.0, n)], 1).astype(np.float32)
    d = np.tile(np.float32([0.05, 0.0, -1.0]), (n, 1))
    r = oracle.simulate(sc, p, o, d, np.zeros(n), np.arange(n, dtype=np.uint64))
    for i in range(n):
        for s in range(7):
            k, m = oracle.bin_of(r.sub_range[i, s], p.bin_width_ns)
            assert r.sub_k[i, s] == k and r.sub_kmargin[i, s] == m


# ---------------------------------------------------------------- u margin
def test_transmission_margin_fires_only_at_the_decision_boundary():
    for u in (0.5, 0.123456789, 0.98):
        L = 0.5
        sigma = -math.log(u) / L  # exp(-sigma L) == u up to rounding
        passes, m = oracle.transmits(u, sigma, L)
        assert m <= 1e-15
        passes, m = oracle.transmits(u, sigma * (1 + 1e-6), L)  # u above exp(-sigma L): echo
        assert not passes and m == pytest.approx(u * -math.log(u) * 1e-6, rel=1e-3)
        passes, m = oracle.transmits(u, sigma * (1 - 1e-6), L)
        assert passes and m > 1e-12


def test_simulate_records_the_transmission_margin():
    # rays along +x through the centres of a 1 m voxel row: every chord is
    # exactly 1 m, so each decision's margin is |u - exp(-PAD G * 1)| with u
    # the counter-based draw of (pulse, subray, voxel)
    from workloads.configs import Scene
    nx = 6
    pad = np.zeros((1, 1, nx), np.float32)
    pad[0, 0, :] = np.float32([0.2, 0.0, 0.7, 0.05, 1.3, 0.4])
    sc = Scene(tri_xyz=np.zeros((0, 3, 3), np.float32), tri_reflectance=None, voxel_pad=pad,
               grid_origin=(0.0, 0.0, 0.0), voxel_size=1.0)
    p = ScannerParams(subray_count=1, divergence_rad=1e-4, seed=3)
    n = 64
    o = np.tile(np.float32([-1.0, 0.5, 0.5]), (n, 1))
    d = np.tile(np.float32([1.0, 0.0, 0.0]), (n, 1))
    ids = np.arange(1000, 1000 + n, dtype=np.uint64)
    r = oracle.simulate(sc, p, o, d, np.zeros(n), ids)
    for i in range(n):
        expect = math.inf
        for v in range(nx):
            if pad[0, 0, v] <= 0:
                continue
            u = oracle.transmission_u(p.seed, int(ids[i]), 0, v)
            e = math.exp(-float(pad[0, 0, v]) * 0.5 * 1.0)
            expect = min(expect, abs(u - e))
            if u >= e:  # the echo: the march stops here
                break
        assert r.sub_umargin[i, 0] == pytest.approx(expect, rel=1e-12, abs=0)


# ---------------------------------------------------------------- peaks / attribution
def _wp(A, k, prim, **kw):
    p = ScannerParams(subray_count=len(A) if len(A) in (1, 7, 19, 37) else 7, **kw)
    N = p.subray_count
    A = np.concatenate([A, np.zeros(N - len(A))])
    k = np.concatenate([k, -np.ones(N - len(k), np.int64)])
    prim = np.concatenate([prim, np.full(N - len(prim), 0xFFFFFFFF, np.uint32)])
    return p, oracle.waveform_peaks(p, A, k, prim)


def _kernel(p):
    tau = p.pulse_length_ns / 1.75
    taps = math.ceil(20 * tau / p.bin_width_ns)
    return np.array([oracle.eq3_pulse(1.0, (j + 0.5) * p.bin_width_ns, tau) for j in range(taps)])


def test_isolated_echo_has_a_wide_margin_and_one_attribution():
    p, r = _wp([1e-3], [500], [42])
    assert r["n_returns"] == 1 and r["ret_prim"][0] == 42
    assert r["peak_margin"] > 1e-3 and math.isinf(r["attr_margin"])
    assert list(r["ret_cand"][0]) == [42, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF]


def test_attribution_sets():
    # equal contributions from two prims: both listed, lowest s first (R13)
    p, r = _wp([2e-3, 2e-3], [500, 500], [9, 5])
    assert r["ret_prim"][0] == 9 and list(r["ret_cand"][0][:3]) == [9, 5, 0xFFFFFFFF]
    assert r["attr_margin"] == 0.0
    # the same prim twice: one candidate, nothing to exempt
    p, r = _wp([2e-3, 2e-3], [500, 500], [7, 7])
    assert list(r["ret_cand"][0][:2]) == [7, 0xFFFFFFFF] and math.isinf(r["attr_margin"])
    # 1e-8 apart: tied within DECISION_EPS; 1e-6 apart: decided
    for rel, tied in ((1e-8, True), (1e-6, False)):
        p, r = _wp([2e-3, 2e-3 * (1 - rel)], [500, 500], [9, 5])
        assert (r["ret_cand"][0][1] == 5) == tied
        assert r["attr_margin"] == pytest.approx(rel, rel=1e-6)


def test_peak_margin_fires_on_a_plateau_and_at_the_threshold():
    p = ScannerParams(subray_count=7)
    ker = _kernel(p)
    js = int(np.argmax(ker))
    # two subrays one bin apart whose sum has W[j] == W[j+1] at the top (a
    # plateau: no strict local maximum there):
    # a p[j] + b p[j-1] = a p[j+1] + b p[j]
    j = js
    a = 1e-3
    b = a * (ker[j] - ker[j + 1]) / (ker[j] - ker[j - 1])
    p, r = _wp([a, b], [500, 501], [1, 2])
    assert r["peak_margin"] <= oracle.DECISION_EPS
    p, r = _wp([a, b * (1 + 1e-3)], [500, 501], [1, 2])
    assert r["peak_margin"] > 1e-6
    # a weak second echo whose peak bin equals the threshold x max
    thr = float(np.float32(p.detection_threshold))
    M = a * ker[js]
    c = thr * M / ker[js]
    p, r = _wp([a, c], [500, 900], [1, 2])
    assert r["peak_margin"] <= oracle.DECISION_EPS
    p, r = _wp([a, c * 1.01], [500, 900], [1, 2])
    assert r["peak_margin"] > 1e-4 and r["n_returns"] == 2
    p, r = _wp([a, c * 0.99], [500, 900], [1, 2])
    assert r["peak_margin"] > 1e-4 and r["n_returns"] == 1


def test_peak_margin_rarely_fires_on_random_footprints():
    # no constructed coincidence: random amplitudes / offsets of a footprint
    rng = np.random.default_rng(4)
    fired = 0
    for _ in range(300):
        m = 19
        A = rng.uniform(1e-4, 1e-3, m)
        k = 700 + rng.integers(0, 6, m)
        p = ScannerParams(subray_count=19)
        r = oracle.waveform_peaks(p, A, k, rng.integers(0, 3, m).astype(np.uint32))
        fired += r["peak_margin"] <= oracle.DECISION_EPS
    assert fired <= 3


def test_threshold_is_taken_as_the_float_the_abi_carries():
    # 0.05 is not a float: the oracle thresholds with float32(0.05) like the ABI
    p = ScannerParams(subray_count=7)
    ker = _kernel(p)
    js = int(np.argmax(ker))
    a = 1e-3
    M = a * ker[js]
    t32 = float(np.float32(0.05))
    assert t32 != 0.05
    mid = 0.5 * (t32 + 0.05)  # between the double and the float threshold
    c = mid * M / ker[js]
    p, r = _wp([a, c], [500, 900], [1, 2])
    assert r["n_returns"] == (2 if mid >= t32 else 1)


# ---------------------------------------------------------------- the brute force's pulse skip
def test_cone_skip_never_rejects_a_reachable_triangle():
    # rays drawn inside the cone (incl. on its mantle): whenever one hits a
    # triangle, the per-pulse cone test must keep that triangle
    rng = np.random.default_rng(11)
    kept = rejected = 0
    for _ in range(3000):
        o = rng.uniform(-1, 1, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        theta = rng.choice([1e-4, 1e-2, 0.3])
        c = o + d * rng.uniform(-2, 20) + rng.normal(size=3) * rng.uniform(0, 3)
        tri = (c + rng.normal(size=(3, 3)) * rng.uniform(0.01, 2)).astype(np.float32)
        may = oracle.cone_may_hit(o, d, theta, tri)
        kept += may
        rejected += not may
        # rays at angle <= theta around d
        u = np.cross(d, [1.0, 0, 0] if abs(d[0]) < 0.9 else [0, 1.0, 0])
        u /= np.linalg.norm(u)
        v = np.cross(d, u)
        for a in rng.uniform(0, theta, 6).tolist() + [theta]:
            ph = rng.uniform(0, 2 * np.pi)
            ds = np.cos(a) * d + np.sin(a) * (np.cos(ph) * u + np.sin(ph) * v)
            t, _ = oracle.ray_triangle(o, ds, tri)
            if t > 0:
                assert may, (o, d, theta, tri, ds)
    assert kept > 100 and rejected > 100


def test_simulate_nearest_equals_single_ray_brute_force():
    # oracle_simulate (triangle blocks x all subrays, cone skip) == the plain
    # per-ray brute force of nearest_candidates, on a wide beam over a soup
    from workloads.configs import Scene
    rng = np.random.default_rng(2)
    n_tris = 3000
    c = rng.uniform(-10, 10, (n_tris, 1, 3))
    tris = (c + rng.uniform(-0.8, 0.8, (n_tris, 3, 3))).astype(np.float32)
    sc = Scene(tri_xyz=tris, tri_reflectance=np.full(n_tris, 0.5, np.float32))
    p = ScannerParams(subray_count=37, divergence_rad=0.05)
    n = 30
    o = rng.uniform(-12, 12, (n, 3)).astype(np.float32)
    d = (rng.uniform(-6, 6, (n, 3)) - o).astype(np.float32)
    r = oracle.simulate(sc, p, o, d, np.zeros(n), np.arange(n, dtype=np.uint64))
    ring, slot, rn, th, ph = oracle.subray_pattern(37, 0.05)
    hits = 0
    for i in range(n):
        for s in range(37):
            ds = oracle.subray_direction(d[i].astype(np.float64), th[s], ph[s])
            idx, t, nc, cand = oracle.nearest_candidates(o[i].astype(np.float64), ds, tris)
            if idx < 0:
                assert r.sub_prim[i, s] == 0xFFFFFFFF
                continue
            hits += 1
            assert r.sub_prim[i, s] == idx and r.sub_range[i, s] == t
            assert r.sub_ncand[i, s] == nc
            assert list(r.sub_cand[i, s][:min(nc, oracle.MAX_CAND)]) == list(cand)
    assert hits > 100
