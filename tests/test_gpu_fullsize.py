"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py
times (1 M-pulse batches through helios_simulate, default chunking and
packet traversal): the GPU runs the whole batch, the oracle recomputes a
seeded sample of its pulses one by one (brute force over every triangle),
and the invariants that hold at any size are checked on every pulse."""
import numpy as np
import pytest

from parity import compare, gpu_invariants
from gpu_util import oracle_run, take, torch_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BATCH = 1_000_000  # bench.py's default pulses per step


def _full(name, start, sample, seed=0):
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    torch = torch_cuda()
    w = make_workload(name)
    sc = h.Scene.from_workload_scene(w.scene)
    B = min(BATCH, w.n_pulses - start)
    o, d, t = w.pulses(start, B)
    dev = lambda a: torch.from_numpy(a).cuda()
    out, st = h.simulate(sc, w.params, dev(o), dev(d), dev(t), pulse_index_base=start,
                         subray_hits=True, stats=True)
    torch.cuda.synchronize()
    g = out.numpy()
    sc.destroy()
    errs = gpu_invariants(g, w.params.max_returns, w.params.detection_threshold)
    assert not errs, errs
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([rng.choice(B, sample, replace=False), [0, B - 1]]))
    orc = oracle_run(w, start + idx)
    rep = compare(take(g, idx), orc, w.scene.n_tris, w.params.bin_width_ns)
    print(name, rep.summary(), f"trace {st.trace_ms:.1f} ms waveform {st.waveform_ms:.1f} ms")
    assert rep.ok(), rep.summary()
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


def test_c5_full_city_terrain():
    _full("C5", 50_000_000 - 400_000, 10)


def test_c6_full_mls_street():
    g, rep = _full("C6", 2_500_000, 2000)
    assert (g["wf_first_bin"] >= 0).mean() > 0.5
