"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (1 M-pulse batches through helios_simulate, default chunking and
packet traversal): the GPU runs the whole batch, the oracle recomputes a
seeded sample of its pulses one by one (brute force over every triangle),
and the invariants that hold at any size are checked on every pulse.

C5 (the headline: km ranges, tree depth 44, 91 -> 96-lane padding, both
flight lines) is sampled in strata chosen from the GENERATOR's geometry, not
from any GPU output: swath edges, roofs, building walls, tree crowns and
plain terrain, on both flight lines."""
import numpy as np
import pytest

from parity import Report, compare, gpu_invariants, record
from gpu_util import oracle_run, take, torch_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BATCH = 1_000_000  # bench.py's default pulses per step


def _gpu_batch(w, sc, start, B):
    import paper_2101_09154_b200 as h
    torch = torch_cuda()
    o, d, t = w.pulses(start, B)
    dev = lambda a: torch.from_numpy(a).cuda()
    out, st = h.simulate(sc, w.params, dev(o), dev(d), dev(t), pulse_index_base=start,
                         subray_hits=True, stats=True)
    torch.cuda.synchronize()
    return out.numpy(), st


def _check(name, w, g, start, idx, rep=None):
    orc = oracle_run(w, start + idx)
    rep = compare(take(g, idx), orc, w.scene.n_tris, w.params.bin_width_ns, report=rep)
    return rep


def _full(name, start, sample, seed=0):
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(name)
    sc = h.Scene.from_workload_scene(w.scene)
    B = min(BATCH, w.n_pulses - start)
    g, st = _gpu_batch(w, sc, start, B)
    sc.destroy()
    errs = gpu_invariants(g, w.params.max_returns, w.params.detection_threshold, w.params)
    assert not errs, errs
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.choice(B, sample, replace=False), [0, B - 1]]))
    rep = _check(name, w, g, start, idx)
    print(name, rep.summary(), f"trace {st.trace_ms:.1f} ms waveform {st.waveform_ms:.1f} ms")
    record(f"{name} full size, batch [{start}, +{B}), {len(idx)} sampled pulses", rep)
    assert rep.ok(), rep.summary()
    assert rep.budget_ok(), rep.summary()
    return g, rep


def test_c1_full():
    _full("C1", 0, 2000)


def test_c2_full_als_dtm():
    g, rep = _full("C2", 0, 300)
    assert (g["wf_first_bin"] >= 0).mean() > 0.8  # +-30 deg at 500 m overhangs the 511 m DTM


def test_c3_full_tls_forest():
    _full("C3", 7_000_000, 150)


def test_c4_full_voxel_canopy():
    g, rep = _full("C4", 2_000_000, 400)
    vox = g["subray_hits"]["prim_id"]
    assert ((vox != 0xFFFFFFFF) & (vox >= 2)).mean() > 0.05  # voxel returns occur


def c5_strata(w, start, B, per_stratum, rng):
    """Pulse indices (relative to start) of the C5 batch, by stratum, from the
    generator's geometry: the central ray's ground point (one terrain-height
    refinement) against the building circles and tree positions."""
    o, d, _ = w.pulses(start, B)
    o = o.astype(np.float64)
    d = d.astype(np.float64)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    hf = w.meta["heights"]
    n = hf.shape[0]
    z = np.full(B, hf.mean())
    for _ in range(2):
        t = (o[:, 2] - z) / -d[:, 2]
        x, y = o[:, 0] + t * d[:, 0], o[:, 1] + t * d[:, 1]
        ix = np.clip(np.rint(x).astype(np.int64), 0, n - 1)
        iy = np.clip(np.rint(y).astype(np.int64), 0, n - 1)
        z = hf[iy, ix]
    theta = np.degrees(np.arcsin(np.abs(d[:, 0])))
    b = w.meta["buildings"]  # (cx, cy, bounding radius)
    from scipy.spatial import cKDTree
    kb = cKDTree(b[:, :2])
    db, jb = kb.query(np.stack([x, y], 1))
    rb = b[jb, 2]
    kt = cKDTree(w.meta["trees"])
    dt, _ = kt.query(np.stack([x, y], 1))
    edge = theta > w.meta["fov_deg"] - 3.0
    roof = db < 0.5 * rb
    wall = (db > 0.6 * rb) & (db < rb + 15.0) & (theta > 15.0) & ~roof
    crown = dt < 4.0
    ground = ~edge & ~roof & ~wall & ~crown & (db > rb + 20.0)
    out = {}
    for k, m in (("swath_edge", edge), ("roof", roof), ("wall", wall), ("crown", crown),
                 ("terrain", ground)):
        cand = np.nonzero(m)[0]
        out[k] = np.sort(rng.choice(cand, min(per_stratum, len(cand)), replace=False))
    return out


def test_c5_full_city_terrain_stratified():
    """>= 200 stratified full-size C5 pulses over both flight lines (the two
    1 M-pulse batches are the middle of line 0 and of line 1)."""
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload("C5")
    sc = h.Scene.from_workload_scene(w.scene)
    per_line = w.meta["per_line"]
    rng = np.random.default_rng(5)
    rep = Report()
    counts = {}
    for line in (0, 1):
        start = line * per_line + per_line // 2
        g, st = _gpu_batch(w, sc, start, BATCH)
        errs = gpu_invariants(g, w.params.max_returns, w.params.detection_threshold, w.params)
        assert not errs, (line, errs)
        strata = c5_strata(w, start, BATCH, 25, rng)
        idx = np.unique(np.concatenate(list(strata.values()) + [[0, BATCH - 1]]))
        for k, v in strata.items():
            counts[f"line{line}_{k}"] = len(v)
        rep = _check("C5", w, g, start, idx, rep)
        del g
    sc.destroy()
    print("C5 strata", counts)
    print("C5", rep.summary())
    record(f"C5 full size, 2 x {BATCH} pulses (both lines), stratified "
           f"{'/'.join(str(v) for v in counts.values())}", rep)
    assert rep.pulses >= 200, counts
    assert all(v > 0 for v in counts.values()), counts
    assert rep.ok(), rep.summary()
    assert rep.budget_ok(), rep.summary()


def test_c6_full_mls_street():
    g, rep = _full("C6", 2_500_000, 2000)
    assert (g["wf_first_bin"] >= 0).mean() > 0.5
