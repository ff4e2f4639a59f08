"""Helpers shared by the -m gpu tests: run the CUDA path / the oracle on the
same seeded pulses."""
from __future__ import annotations

import functools

import numpy as np

import oracle


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "CUDA device required"
    return torch


@functools.lru_cache(maxsize=4)
def workload(name: str, scale: float = 1.0, **kw):
    from workloads import make_workload
    return make_workload(name, scale, **kw)


_scenes = {}  # id(workload scene) -> (workload scene, built Scene); the key object is kept
             # alive so its id cannot be reused by a later (different) scene


def scene_for(w):
    import paper_2101_09154_b200 as h
    key = id(w.scene)
    hit = _scenes.get(key)
    if hit is None or hit[0] is not w.scene:
        if hit is not None:
            _scenes.pop(key)[1].destroy()
        if len(_scenes) >= 3:
            _scenes.pop(next(iter(_scenes)))[1].destroy()
        _scenes[key] = (w.scene, h.Scene.from_workload_scene(w.scene))
    return _scenes[key][1]


def gpu_run(w, start: int, count: int, waveform=True, subray_hits=True, params=None,
            stats=False):
    import paper_2101_09154_b200 as h
    torch = torch_cuda()
    o, d, t = w.pulses(start, count)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out, st = h.simulate(scene_for(w), params or w.params, to(o), to(d), to(t),
                         pulse_index_base=start, waveform=waveform, subray_hits=subray_hits,
                         stats=stats, counters=stats)
    torch.cuda.synchronize()
    res = out.numpy()
    return (res, st) if stats else res


def oracle_run(w, ids, params=None, want_waveform=True):
    ids = np.asarray(ids, np.int64)
    o, d, t = w.pulses_at(ids)
    return oracle.simulate(w.scene, params or w.params, o, d, t, ids.astype(np.uint64),
                           want_waveform=want_waveform)


def take(gpu: dict, idx) -> dict:
    out = {}
    for k, v in gpu.items():
        out[k] = None if v is None else v[idx]
    return out


def beam_env(value: str):
    """Beam pre-pass K6a off ("0") or on where it applies ("1") for the calls
    inside (helios_set_tuning)."""
    import paper_2101_09154_b200 as h
    return h.tuning(beam_prepass=int(value))
