"""GPU edge cases, API contract, determinism and BVH == brute force."""
from dataclasses import replace

import numpy as np
import pytest

import oracle
from parity import compare, gpu_invariants
from gpu_util import gpu_run, oracle_run, take, torch_cuda, workload
from workloads import Scene, ScannerParams

pytestmark = pytest.mark.gpu


def _h():
    import paper_2101_09154_b200 as h
    return h


def _dev(a):
    torch = torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _soup(n, seed, extent=10.0, size=1.0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-extent, extent, (n, 1, 3))
    return (c + rng.uniform(-size, size, (n, 3, 3))).astype(np.float32)


@pytest.mark.parametrize("builder", ["lbvh", "ploc"])
@pytest.mark.parametrize("n_tris", [1, 2, 3, 4, 5, 17, 1000, 10000])
def test_bvh_equals_brute_force_random_soup(n_tris, builder):
    # S:87/S:725 shape: random rays vs random triangles; ids exact, t within 1e-9
    # (both hierarchies: Karras LBVH and PLOC, helios_tuning.builder)
    h = _h()
    tris = _soup(n_tris, n_tris, size=2.0 if n_tris < 100 else 0.7)
    refl = np.random.default_rng(1).uniform(0.1, 0.9, n_tris).astype(np.float32)
    with h.tuning(builder=1 if builder == "lbvh" else 0):
        sc = h.Scene(_dev(tris), _dev(refl))
    rng = np.random.default_rng(7)
    m = 1000
    o = rng.uniform(-14, 14, (m, 3)).astype(np.float32)
    tgt = rng.uniform(-8, 8, (m, 3))
    d = (tgt - o).astype(np.float32)
    p = ScannerParams(subray_count=1, divergence_rad=1e-3)
    out, _ = h.simulate(sc, p, _dev(o), _dev(d), subray_hits=True)
    g = out.numpy()["subray_hits"][:, 0]
    for i in range(m):
        dd = d[i].astype(np.float64)
        dd /= np.linalg.norm(dd)
        idx, t, _, nc, _ = oracle.nearest_triangle(o[i].astype(np.float64), dd, tris)
        if idx < 0:
            assert g["prim_id"][i] == 0xFFFFFFFF
        else:
            assert abs(g["range_m"][i] - t) <= 1e-9 * max(1.0, t), (i, g["range_m"][i], t)
            if nc == 1:
                assert g["prim_id"][i] == idx
    sc.destroy()


def test_zero_pulses_and_ragged_batches():
    h = _h()
    w = workload("C2", 0.125)
    sc_empty = np.zeros((0, 3), np.float32)
    from gpu_util import scene_for
    sc = scene_for(w)
    out, _ = h.simulate(sc, w.params, _dev(sc_empty), _dev(sc_empty))
    assert out.n_returns.numel() == 0
    for n in (1, 31, 33, 127, 1025 + 7):
        rep_g = gpu_run(w, 777, n)
        o = oracle_run(w, 777 + np.arange(n))
        rep = compare(rep_g, o, w.scene.n_tris, w.params.bin_width_ns)
        assert rep.ok(), rep.summary()


def test_batch_split_and_repeat_are_bitwise_identical():
    w = workload("C4", 0.1)
    a = gpu_run(w, 1000, 5000)
    b = gpu_run(w, 1000, 5000)
    c1 = gpu_run(w, 1000, 1234)
    c2 = gpu_run(w, 2234, 5000 - 1234)
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
        cat = np.concatenate([c1[k], c2[k]])
        assert np.array_equal(a[k].view(np.uint8), cat.view(np.uint8)), k


def test_beam_scene_chunking_and_batch_split_are_bitwise_identical():
    """Beam pre-pass scene (C5 reduced): the chunk schedule (library rule, or
    forced 1024- and 3000-pulse chunks) and a split into two calls must not
    change a bit of the output (Philox counters, lane order, entry lists and
    deferred hits are all per pulse / per subray)."""
    w = workload("C5", 0.03)
    h = _h()
    a = gpu_run(w, 300, 7000)
    runs = []
    for chunk in (1024, 3000):
        with h.tuning(chunk_pulses=chunk):
            runs.append(gpu_run(w, 300, 7000))
    c1 = gpu_run(w, 300, 2500)
    c2 = gpu_run(w, 2800, 4500)
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
        for b in runs:
            assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
        cat = np.concatenate([c1[k], c2[k]])
        assert np.array_equal(a[k].view(np.uint8), cat.view(np.uint8)), k


@pytest.mark.parametrize("subrays,n", [(37, 3000), (279, 25000)])
def test_host_buffers_match_device_buffers(subrays, n):
    # host (pageable numpy / pinned torch) buffers go through the library's
    # chunked, double-buffered staging pipeline; 279 subrays x 25000 pulses
    # spans three chunks
    import torch
    h = _h()
    w = workload("C3", 0.03)
    from gpu_util import scene_for
    sc = scene_for(w)
    p = replace(w.params, subray_count=subrays)
    o, d, t = w.pulses(100, n)
    dev_out, _ = h.simulate(sc, p, _dev(o), _dev(d), _dev(t), pulse_index_base=100,
                            subray_hits=True)
    a = dev_out.numpy()
    host_out = h.alloc_outputs(n, h.make_params(p), device="cpu", subray_hits=True)
    h.simulate(sc, p, o, d, t, pulse_index_base=100, outputs=host_out)
    pin_out = h.alloc_outputs(n, h.make_params(p), device="cpu", subray_hits=True,
                              pin_memory=True)
    h.simulate(sc, p, *(torch.from_numpy(x).pin_memory() for x in (o, d, t)),
               pulse_index_base=100, outputs=pin_out)
    for b in (host_out.numpy(), pin_out.numpy()):
        for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
            assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_waveform_output_optional_binning_still_runs():
    w = workload("C3", 0.03)
    a = gpu_run(w, 500, 2000, waveform=True)
    b = gpu_run(w, 500, 2000, waveform=False)
    assert b["waveform"] is None
    for k in ("n_returns", "wf_first_bin", "returns"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_zero_direction_is_reported_and_zeroed():
    h = _h()
    w = workload("C1")
    from gpu_util import scene_for
    sc = scene_for(w)
    o, d, t = w.pulses(0, 64)
    d = d.copy()
    d[5] = 0.0
    out = h.alloc_outputs(64, h.make_params(w.params), subray_hits=True)
    with pytest.raises(h.HeliosError) as e:
        h.simulate(sc, w.params, _dev(o), _dev(d), _dev(t), outputs=out)
    assert e.value.status == 1 and "zero length" in str(e.value)
    g = out.numpy()
    assert g["wf_first_bin"][5] == -1 and g["n_returns"][5] == 0
    assert not g["waveform"][5].any()
    assert np.all(g["subray_hits"]["prim_id"][5] == 0xFFFFFFFF)


def test_status_codes():
    h = _h()
    p = ScannerParams()
    tri = _soup(8, 3)
    # NOT_BUILT
    sc = h.Scene(_dev(tri), build=False)
    o = _dev(np.zeros((4, 3), np.float32))
    d = _dev(np.tile([0, 0, -1.0], (4, 1)).astype(np.float32))
    with pytest.raises(h.HeliosError) as e:
        h.simulate(sc, p, o, d)
    assert e.value.status == h.helios.HELIOS_ERR_NOT_BUILT
    h.helios_build_accel(sc.handle)
    h.simulate(sc, p, o, d)
    # INVALID_ARGUMENT: bad subray count, threshold
    with pytest.raises(h.HeliosError) as e:
        h.simulate(sc, replace(p, subray_count=20), o, d)
    assert e.value.status == 1 and "subray_count" in str(e.value)
    sc.destroy()
    # EMPTY_SCENE
    with pytest.raises(h.HeliosError) as e:
        h.Scene(_dev(np.zeros((0, 3, 3), np.float32)))
    assert e.value.status == h.helios.HELIOS_ERR_EMPTY_SCENE
    # non-finite vertex, reflectance out of range, negative PAD
    bad = tri.copy()
    bad[2, 1, 0] = np.nan
    with pytest.raises(h.HeliosError) as e:
        h.Scene(_dev(bad))
    assert "non-finite" in str(e.value)
    with pytest.raises(h.HeliosError):
        h.Scene(_dev(tri), _dev(np.full(8, 1.5, np.float32)))
    with pytest.raises(h.HeliosError):
        h.Scene(None, None, _dev(np.full((2, 2, 2), -1.0, np.float32)), (0, 0, 0), 1.0)
    h.helios_scene_destroy(None)  # NULL is a no-op


def test_voxel_only_scene_and_origin_inside_grid():
    # no triangles, one grid; scanner inside the grid (t_in = 0)
    pad = np.zeros((10, 10, 10), np.float32)
    pad[2:8, 2:8, 2:8] = 0.4
    sc = Scene(np.zeros((0, 3, 3), np.float32), None, pad, (-5.0, -5.0, -5.0), 1.0)
    p = ScannerParams(subray_count=19, seed=5)
    from workloads.configs import Workload
    rng = np.random.default_rng(3)
    n = 3000
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    orig = rng.uniform(-4, 4, (n, 3)).astype(np.float32)
    orig[:100] = 0.0  # exactly on voxel planes
    dirs[100:200] = [0, 0, -1]  # axis-aligned directions (zero components)
    fn = lambda idx: (orig[idx], dirs[idx], idx * 1e-6)
    w = Workload("vox", sc, p, n, fn)
    g = gpu_run(w, 0, n)
    o = oracle_run(w, np.arange(n))
    rep = compare(g, o, 0, p.bin_width_ns)
    assert rep.ok(), rep.summary()
    assert (o.sub_prim != 0xFFFFFFFF).mean() > 0.2


def test_degenerate_rays_on_edges_and_planes():
    # rays through shared triangle edges and vertices of a DTM: tie-exempt or exact
    w = workload("C2", 0.03)
    from workloads.configs import Workload
    n = 2000
    rng = np.random.default_rng(9)
    xy = rng.integers(1, 14, (n, 2)).astype(np.float32)  # lattice points (vertices)
    xy[n // 2:] += 0.5  # cell diagonals
    orig = np.concatenate([xy, np.full((n, 1), 300.0, np.float32)], 1)
    dirs = np.tile(np.float32([0, 0, -1]), (n, 1))
    fn = lambda idx: (orig[idx], dirs[idx], idx * 1e-6)
    w2 = Workload("edges", w.scene, replace(w.params, subray_count=1), n, fn)
    g = gpu_run(w2, 0, n)
    o = oracle_run(w2, np.arange(n))
    rep = compare(g, o, w.scene.n_tris, w.params.bin_width_ns)
    assert rep.ok(), rep.summary()
    # the case is really exercised: subrays with several candidates within 1e-6 m
    # (the GPU's exact-replica fp64 test takes the oracle's own choice)
    assert rep.checked.get("tie_subrays_same_id", 0) + rep.exempt_subrays.get("tie_taken", 0) > 0
    assert rep.budget_ok(), rep.summary()


def test_stats_counters():
    w = workload("C4", 0.1)
    g, st = gpu_run(w, 0, 4000, stats=True)
    assert st.pulses == 4000 and st.subrays == 4000 * 19
    assert st.subray_hits == int((g["subray_hits"]["prim_id"] != 0xFFFFFFFF).sum())
    assert st.returns == int(g["n_returns"].sum())
    vox = (g["subray_hits"]["prim_id"] != 0xFFFFFFFF) & (g["subray_hits"]["prim_id"] >= 2)
    assert st.voxel_returns == int(vox.sum())
    assert st.voxel_steps > 0 and st.nodes_visited == 0 and st.tris_tested > 0
    assert st.trace_ms > 0 and st.waveform_ms > 0 and st.kernel_launches >= 2


def test_invariants_on_a_full_reduced_run():
    w = workload("C5", 0.03)
    g = gpu_run(w, 0, w.n_pulses, subray_hits=False)
    errs = gpu_invariants(g, w.params.max_returns, w.params.detection_threshold, w.params)
    assert not errs, errs
    assert (g["wf_first_bin"] >= 0).mean() > 0.9


@pytest.mark.parametrize("N,beta", [(19, 1e-3), (91, 5e-4), (37, 1e-7), (37, 0.05), (7, 0.099)])
def test_beam_prepass_axis_aligned_and_grazing(N, beta):
    """K6a's interval cone test on its hard cases: pulse axes exactly along
    +-x, +-y, +-z (direction intervals straddling 0 on two axes), axis-plane
    triangles (flat, zero-thickness boxes), origins inside the scene, and a
    cone far narrower than the boxes.  With the pre-pass forced on, every
    subray must match the brute-force oracle (and the run without it, bitwise)."""
    h = _h()
    rng = np.random.default_rng(N)
    soup = _soup(3000, N, extent=12.0, size=0.8)
    # axis-plane quads: z = const floors, x = const and y = const walls
    flat = []
    for k in range(200):
        c = rng.uniform(-10, 10, 3)
        a, b = rng.uniform(0.2, 2.0, 2)
        ax = k % 3
        u, v = [(1, 2), (0, 2), (0, 1)][ax]
        q = np.zeros((4, 3))
        q[:, ax] = c[ax]
        for i, (du, dv) in enumerate([(-a, -b), (a, -b), (a, b), (-a, b)]):
            q[i, u], q[i, v] = c[u] + du, c[v] + dv
        flat += [q[[0, 1, 2]], q[[0, 2, 3]]]
    tris = np.concatenate([soup, np.array(flat, np.float32)]).astype(np.float32)
    scene = Scene(tri_xyz=tris, tri_reflectance=np.full(len(tris), 0.4, np.float32))
    axes = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], float)
    dirs = np.concatenate([np.repeat(axes, 20, 0), rng.normal(size=(120, 3))]).astype(np.float32)
    n = len(dirs)
    org = rng.uniform(-11, 11, (n, 3)).astype(np.float32)
    tim = np.zeros(n)
    p = ScannerParams(subray_count=N, divergence_rad=beta, max_fullwave_range_ns=2000.0)
    sc = h.Scene.from_workload_scene(scene)
    outs = {}
    for beam in ("0", "1"):
        with h.tuning(beam_prepass=int(beam)):
            o, st = h.simulate(sc, p, _dev(org), _dev(dirs), _dev(tim), subray_hits=True,
                               stats=True, counters=True)
        torch_cuda().cuda.synchronize()
        outs[beam] = (o.numpy(), st)
    sc.destroy()
    g0, g1 = outs["0"][0], outs["1"][0]
    assert outs["1"][1].beam_nodes > 0 and outs["0"][1].beam_nodes == 0
    for k in g0:
        if g0[k] is not None:
            assert np.array_equal(g0[k].view(np.uint8), g1[k].view(np.uint8)), k
    r = oracle.simulate(scene, p, org, dirs, tim, np.arange(n, dtype=np.uint64))
    sh = g1["subray_hits"]
    tie = r.sub_ncand > 1
    assert np.array_equal(sh["prim_id"][~tie], r.sub_prim[~tie])
    hit = r.sub_prim != 0xFFFFFFFF
    assert hit.mean() > 0.2
    dr = np.abs(sh["range_m"][hit] - r.sub_range[hit])
    assert np.all(dr <= 1e-6 * r.sub_range[hit] + 1e-5)


@pytest.mark.parametrize("name,scale,start,count", [("C5", 0.03, 100, 3000), ("C3", 0.03, 500, 6000)])
def test_lane_order_and_padding_are_bitwise_invariant(name, scale, start, count):
    """K6's lane order (R4 ring order vs the Hilbert patch order) and the lane
    padding to whole warps only change which lane computes which subray: every
    output must be bitwise identical (with the beam pre-pass on and off)."""
    w = workload(name, scale)
    h = _h()
    ref = None
    for beam in ("0", "1"):
        for order in ("0", "1"):
            for pad in ("0", "1"):
                with h.tuning(beam_prepass=int(beam), lane_order=int(order), pad_lanes=int(pad)):
                    g = gpu_run(w, start, count)
                if ref is None:
                    ref = g
                    continue
                for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
                    assert np.array_equal(ref[k].view(np.uint8), g[k].view(np.uint8)), (k, beam, order, pad)


@pytest.mark.slow
@pytest.mark.parametrize("cfg,scale", [("C2", 1.0), ("C3", 1.0), ("C5", 1.0), ("C4", 1.0)])
def test_karras_and_ploc_trees_give_bitwise_identical_results(cfg, scale):
    """The nearest hit is the minimum over every triangle, exact ties
    -> lower id (R22), so the result cannot depend on the hierarchy: the Karras
    LBVH (helios_tuning.builder = 1) and PLOC trees of the FULL BASELINE
    scenes (0.5 M / 4.2 M / 49.8 M triangles) must give bitwise equal outputs
    on a stretch of each config's own pulses."""
    import paper_2101_09154_b200 as h
    torch = torch_cuda()
    w = workload(cfg, scale)
    n = min(50_000, w.n_pulses)
    start = w.n_pulses // 2
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, n))
    res, depth = [], []
    for builder in (1, 0):
        with h.tuning(builder=builder):
            sc = h.Scene.from_workload_scene(w.scene)
        depth.append(sc.info().max_depth)
        out, _ = h.simulate(sc, w.params, o, d, t, pulse_index_base=start, subray_hits=True)
        res.append(out.numpy())
        sc.destroy()
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
        assert np.array_equal(np.ascontiguousarray(res[0][k]).view(np.uint8),
                              np.ascontiguousarray(res[1][k]).view(np.uint8)), (k, depth)
