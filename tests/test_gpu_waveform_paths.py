"""K7's less common evaluation paths, forced by constructed geometry and
checked against the oracle (DESIGN.md s.7, waveform.cu):

  * offsets within 64 bins, <= 16 groups   -> chunked group sums (every config)
  * offsets within 64 bins, > 16 groups    -> match_any group sums per 32-subray chunk
  * offsets spread over >= 64 bins         -> match_any groups added into W one by one
  * many such groups (61)                  -> the same path, no group cap
  * support S > 512 bins                   -> deferred to the wide pass (global scratch row),
                                              alone and mixed with ordinary pulses

A "staircase" puts one tiny triangle on each subray's own direction at its
own distance (placed with the oracle's subray_direction, pinned against the
paper's pattern), so every subray gets the bin offset the test chooses; a
near/far pair splits a footprint between two surfaces 140 m apart."""
import numpy as np
import pytest

import oracle
from gpu_util import torch_cuda
from parity import compare, gpu_invariants
from workloads import ScannerParams
from workloads.configs import Scene, Workload

pytestmark = pytest.mark.gpu


def _tri_facing(c, d, size):
    """Small equilateral triangle centred at c, perpendicular to d."""
    a = np.cross(d, [1.0, 0.0, 0.0] if abs(d[0]) < 0.9 else [0.0, 1.0, 0.0])
    a /= np.linalg.norm(a)
    b = np.cross(d, a)
    ang = 2 * np.pi * np.arange(3) / 3
    return np.stack([c + size * (np.cos(t) * a + np.sin(t) * b) for t in ang])


def _run(scene, params, o, d, n):
    import paper_2101_09154_b200 as h
    torch = torch_cuda()
    orig = np.tile(np.asarray(o, np.float32), (n, 1))
    dirs = np.tile(np.asarray(d, np.float32), (n, 1))
    # a tiny per-pulse jitter of the origin along the axis keeps the geometry
    # but gives distinct inputs (the offsets stay the same)
    orig[:, 2] += np.float32(1e-3) * np.arange(n, dtype=np.float32) / n
    tim = np.arange(n) * 1e-6
    sc = h.Scene.from_workload_scene(scene)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out, _ = h.simulate(sc, params, dev(orig), dev(dirs), dev(tim), pulse_index_base=0,
                        subray_hits=True)
    torch.cuda.synchronize()
    g = out.numpy()
    sc.destroy()
    r = oracle.simulate(scene, params, orig, dirs, tim, np.arange(n, dtype=np.uint64))
    errs = gpu_invariants(g, params.max_returns, params.detection_threshold, params)
    assert not errs, errs
    rep = compare(g, r, scene.n_tris, params.bin_width_ns)
    assert rep.ok(), rep.summary()
    assert rep.budget_ok(), rep.summary()
    return g, r


def _staircase(N, beta, dist_of_s, n=64):
    d = np.array([0.0, 0.0, -1.0])
    o = np.array([0.0, 0.0, 50.0])
    ring, slot, rn, th, ph = oracle.subray_pattern(N, beta)
    tris = []
    for s in range(N):
        dist = dist_of_s(s)
        if dist is None:
            continue
        ds = oracle.subray_direction(d, th[s], ph[s])
        tris.append(_tri_facing(o + dist * ds, ds, 2e-3))
    scene = Scene(tri_xyz=np.array(tris, np.float32),
                  tri_reflectance=np.linspace(0.2, 0.8, len(tris)).astype(np.float32))
    p = ScannerParams(subray_count=N, divergence_rad=beta, max_returns=7,
                      detection_threshold=0.01)
    return _run(scene, p, o, d, n)


def _offsets(g):
    k = np.floor(2 * g["subray_hits"]["range_m"][0] / 299792458.0 / 1e-9)
    k = k[np.isfinite(k)]
    return np.unique(k - k.min()).astype(int)


def test_many_groups_within_64_bins_match_any_sums():
    # 37 subrays, distinct offsets 0..36 bins (0.15 m apart): G = 37 > 16, maxoff < 64
    g, _ = _staircase(37, 0.05, lambda s: 10.0 + 0.15 * s + 0.05)
    off = _offsets(g)
    assert 16 < len(off) and off.max() < 64


def test_spread_offsets_match_any_groups():
    # 30 subrays 0.5 m apart (~3.3 bins), 7 miss: G = 30 <= 42, maxoff >= 64
    g, _ = _staircase(37, 0.05, lambda s: 10.0 + 0.5 * s if s < 30 else None)
    off = _offsets(g)
    assert 16 < len(off) <= 42 and off.max() >= 64


def test_many_spread_groups_no_cap():
    # 61 distinct offsets (0.3 m apart): G = 61 (the old kernel capped groups at 42)
    g, _ = _staircase(61, 0.05, lambda s: 10.0 + 0.3 * s)
    off = _offsets(g)
    assert len(off) > 42 and off.max() >= 64


def test_wide_support_in_global_scratch():
    # half of the footprint on a triangle 10 m away, the rest on a plane 150 m
    # away: offsets spread over ~934 bins, support > 512 bins (global scratch)
    d = np.array([0.0, 0.0, -1.0])
    o = np.array([0.0, 0.0, 0.0])
    near = np.array([[0.0, -5.0, -10.0], [5.0, -5.0, -10.0], [0.0, 5.0, -10.0]])
    far = np.array([[-500, -500, -150.0], [500, -500, -150.0], [500, 500, -150.0],
                    [-500, -500, -150.0], [500, 500, -150.0], [-500, 500, -150.0]])
    tris = np.concatenate([near[None], far.reshape(2, 3, 3)]).astype(np.float32)
    scene = Scene(tri_xyz=tris, tri_reflectance=np.float32([0.3, 0.6, 0.6]))
    # the far echo is (150/10)^4 = 5e4 times weaker (Eq. 7, R^-4): a low threshold
    p = ScannerParams(subray_count=19, divergence_rad=0.05, max_returns=7,
                      detection_threshold=1e-6)
    g, r = _run(scene, p, o, d, 128)
    off = _offsets(g)
    assert off.max() + 46 > 512
    assert (g["n_returns"] == 2).all()  # the near and the far echo


@pytest.mark.parametrize("bin_ns,n", [(1.0, 257), (0.05, 33)])
def test_wide_pass_mixed_with_ordinary_pulses(bin_ns, n):
    # alternate pulses see the near triangle over the far plane (support > 512
    # bins: deferred to the wide pass) or the far plane alone (main pass): the
    # deferral list must leave every other pulse to the main pass untouched.
    # 1 ns bins: 1335-bin rows, the wide pass keeps them in shared memory;
    # 0.05 ns bins over 2000 ns: 40000-bin rows (320 KB) -> global scratch rows
    import paper_2101_09154_b200 as h
    torch = torch_cuda()
    near = np.array([[0.0, -5.0, -10.0], [5.0, -5.0, -10.0], [0.0, 5.0, -10.0]])
    far = np.array([[-500, -500, -150.0], [500, -500, -150.0], [500, 500, -150.0],
                    [-500, -500, -150.0], [500, 500, -150.0], [-500, 500, -150.0]])
    tris = np.concatenate([near[None], far.reshape(2, 3, 3)]).astype(np.float32)
    scene = Scene(tri_xyz=tris, tri_reflectance=np.float32([0.3, 0.6, 0.6]))
    p = ScannerParams(subray_count=19, divergence_rad=0.05, max_returns=7,
                      detection_threshold=1e-6, bin_width_ns=bin_ns,
                      **({} if bin_ns == 1.0 else {"max_fullwave_range_ns": 2000.0}))
    orig = np.zeros((n, 3), np.float32)
    orig[1::2, 0] = 200.0  # odd pulses: beside the near triangle
    orig[:, 2] = np.float32(1e-3) * np.arange(n, dtype=np.float32) / n
    dirs = np.tile(np.float32([0.0, 0.0, -1.0]), (n, 1))
    tim = np.arange(n) * 1e-6
    sc = h.Scene.from_workload_scene(scene)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out, _ = h.simulate(sc, p, dev(orig), dev(dirs), dev(tim), pulse_index_base=0,
                        subray_hits=True)
    torch.cuda.synchronize()
    g = out.numpy()
    sc.destroy()
    r = oracle.simulate(scene, p, orig, dirs, tim, np.arange(n, dtype=np.uint64))
    errs = gpu_invariants(g, p.max_returns, p.detection_threshold, p)
    assert not errs, errs
    rep = compare(g, r, scene.n_tris, p.bin_width_ns)
    assert rep.ok(), rep.summary()
    assert (g["n_returns"][0::2] == 2).all() and (g["n_returns"][1::2] == 1).all()
