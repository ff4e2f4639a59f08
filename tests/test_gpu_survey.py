"""On-device pulse generation (NEXT f2; helios_simulate_survey, reading R30):
generated beams vs the oracle's generator, and the whole hot path on
generated pulses vs the oracle run on the same beams."""
import math
from dataclasses import replace

import numpy as np
import pytest

import oracle
from parity import compare, gpu_invariants
from gpu_util import scene_for, take, torch_cuda, workload
from workloads import Survey

pytestmark = pytest.mark.gpu


def _h():
    import paper_2101_09154_b200 as h
    return h


SURVEYS = {
    "static_head_polygon": Survey(waypoints=np.array([[3.0, -2.0, 1.5]]), pulse_freq_hz=50000.0,
                                  deflector="polygon", scan_freq_hz=25.0,
                                  scan_angle_rad=math.radians(60.0), head_rotation_rad_s=0.3,
                                  mount=np.array([[1, 0, 0], [0, 0, -1], [0, 1, 0]], float),
                                  mount_offset=np.array([0.1, 0.0, 0.2])),
    "linear_oscillating": Survey(waypoints=np.array([[-60.0, -60.0, 150.0], [60.0, -50.0, 150.0],
                                                     [60.0, 60.0, 140.0], [60.0, 60.0, 140.0]]),
                                 pulse_freq_hz=100000.0, deflector="oscillating",
                                 scan_freq_hz=70.0, scan_angle_rad=math.radians(25.0),
                                 speed_m_s=40.0, t0_s=2.5),
    "linear_palmer": Survey(waypoints=np.array([[0.0, -80.0, 120.0], [0.0, 80.0, 120.0]]),
                            pulse_freq_hz=200000.0, deflector="palmer", scan_freq_hz=30.0,
                            scan_angle_rad=math.radians(15.0), speed_m_s=20.0),
    "linear_fibre": Survey(waypoints=np.array([[-70.0, 0.0, 100.0], [70.0, 10.0, 100.0]]),
                           pulse_freq_hz=150000.0, deflector="fibre", n_fibres=64,
                           scan_freq_hz=500.0, scan_angle_rad=math.radians(20.0), speed_m_s=50.0),
}


@pytest.mark.parametrize("name", sorted(SURVEYS))
def test_generated_beams_match_the_oracle_generator(name):
    h = _h()
    w = workload("C3", 0.03)
    sv = SURVEYS[name]
    first, n = 12345, 20000
    out, _ = h.simulate_survey(scene_for(w), w.params, sv, first, n, beams=True)
    g = out.numpy()
    o, d, t = oracle.generate_pulses(sv, first, n)
    assert np.array_equal(g["beam_time"], t)
    for a, b in ((g["beam_origin"], o), (g["beam_direction"], d)):
        ulp = np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32).astype(np.int64))
        ulp[(a == 0) & (b == 0)] = 0  # +0 / -0
        assert ulp.max() <= 1, (name, ulp.max())
        assert (ulp > 0).mean() < 1e-3  # sin / cos differ from glibc by <= 1 ulp in fp64


@pytest.mark.parametrize("cfg,scale,surv", [("C3", 0.03, "static_head_polygon"),
                                            ("C3", 0.03, "linear_palmer"),
                                            ("C4", 0.1, "oscillating"),
                                            ("C5", 0.03, None)])
def test_hot_path_on_generated_pulses_matches_the_oracle(cfg, scale, surv):
    # the oracle simulates the beams the GPU generated (identical inputs), the
    # comparator is the same as for host-fed pulses
    h = _h()
    w = workload(cfg, scale)
    if surv is None:
        sv, g0, cnt = w.surveys[1]
        first, n, base = 100, 2000, g0 + 100
    elif surv == "oscillating":  # the workload's own flight line, swinging mirror
        sv = replace(w.surveys[0][0], deflector="oscillating", scan_freq_hz=35.0)
        first, n, base = 0, 3000, 0
    else:
        sv, first, n, base = SURVEYS[surv], 500, 3000, 7000
    out, _ = h.simulate_survey(scene_for(w), w.params, sv, first, n, base, beams=True,
                               subray_hits=True)
    g = out.numpy()
    errs = gpu_invariants(g, w.params.max_returns, w.params.detection_threshold, w.params)
    assert not errs, errs
    ids = np.arange(base, base + n, dtype=np.uint64)
    r = oracle.simulate(w.scene, w.params, g["beam_origin"], g["beam_direction"], g["beam_time"],
                        ids)
    rep = compare(g, r, w.scene.n_tris, w.params.bin_width_ns)
    print(rep.summary())
    assert rep.ok(), rep.summary()
    assert (r.sub_prim != 0xFFFFFFFF).mean() > 0.05


def test_survey_equals_host_fed_pulses_when_the_beams_are_equal():
    # C2's flight line as a survey generates exactly the workload's arrays
    # (origins/times bitwise, directions as numpy rounds them): same outputs
    torch = torch_cuda()
    h = _h()
    w = workload("C2", 0.125)
    sv, g0, cnt = w.surveys[0]
    n = 4000
    a, _ = h.simulate_survey(scene_for(w), w.params, sv, 200, n, g0 + 200, beams=True)
    a = a.numpy()
    o, d, t = w.pulses(g0 + 200, n)
    same = np.all(a["beam_direction"] == d, axis=1) & np.all(a["beam_origin"] == o, axis=1)
    assert same.mean() > 0.99 and np.array_equal(a["beam_time"], t)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    b, _ = h.simulate(scene_for(w), w.params, dev(o), dev(d), dev(t), pulse_index_base=g0 + 200)
    b = b.numpy()
    for k in ("n_returns", "wf_first_bin", "waveform", "returns"):
        assert np.array_equal(a[k][same].view(np.uint8), b[k][same].view(np.uint8)), k


def test_survey_host_outputs_multi_chunk_and_batch_split():
    # host-staged beams/returns over several chunks; two calls with split
    # pulse ranges == one call (bitwise)
    import torch
    h = _h()
    w = workload("C5", 0.03)
    sv, g0, cnt = w.surveys[0]
    p = replace(w.params, subray_count=271)
    n = 30000
    a, _ = h.simulate_survey(scene_for(w), p, sv, 0, n, 0, beams=True)
    a = a.numpy()
    out = h.alloc_outputs(n, h.make_params(p), device="cpu", pin_memory=True, beams=True)
    h.simulate_survey(scene_for(w), p, sv, 0, n, 0, outputs=out)
    b = out.numpy()
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "beam_origin",
              "beam_direction", "beam_time"):
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
    c1, _ = h.simulate_survey(scene_for(w), p, sv, 0, 12345, 0, beams=True)
    c2, _ = h.simulate_survey(scene_for(w), p, sv, 12345, n - 12345, 12345, beams=True)
    c1, c2 = c1.numpy(), c2.numpy()
    for k in ("n_returns", "waveform", "returns", "beam_direction"):
        assert np.array_equal(a[k].view(np.uint8),
                              np.concatenate([c1[k], c2[k]]).view(np.uint8)), k


def test_survey_validation():
    h = _h()
    w = workload("C3", 0.03)
    bad = [dict(pulse_freq_hz=0.0), dict(scan_freq_hz=-1.0), dict(scan_angle_rad=1.6),
           dict(deflector="fibre", n_fibres=0),
           dict(waypoints=np.array([[0, 0, 0], [1, 0, 0.0]]), speed_m_s=0.0),
           dict(waypoints=np.array([[0, 0, np.nan]]))]
    for kw in bad:
        sv = replace(SURVEYS["linear_palmer"], **kw)
        with pytest.raises(h.HeliosError) as ei:
            h.simulate_survey(scene_for(w), w.params, sv, 0, 10)
        assert ei.value.status == 1, kw
