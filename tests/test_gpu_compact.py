"""Compact (sparse-support) waveform output (NEXT f4; include/helios.h
helios_outputs.p_wf_compact): lossless packed rows, exact support lengths,
host staging across chunks, and the capacity contract."""
from dataclasses import replace

import numpy as np
import pytest

from gpu_util import gpu_run, oracle_run, scene_for, torch_cuda, workload

pytestmark = pytest.mark.gpu


def _h():
    import paper_2101_09154_b200 as h
    return h


def _dev(a):
    torch = torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _support_from_oracle(r, n_bins, taps):
    """len_p = min(n_bins, max_s (k_s - k0) + L_p) over in-window subrays (R9),
    from the oracle's own per-subray bins."""
    out = np.zeros(len(r.k0), np.int64)
    for i, k0 in enumerate(r.k0):
        if k0 < 0:
            continue
        o = r.sub_k[i][r.sub_prim[i] != 0xFFFFFFFF] - k0
        o = o[o < n_bins]
        out[i] = min(n_bins, int(o.max()) + taps)
    return out


@pytest.mark.parametrize("name,scale,start,count", [("C2", 0.125, 500, 3000),
                                                    ("C3", 0.03, 1000, 2000),
                                                    ("C4", 0.1, 0, 4000)])
def test_compact_rows_are_the_dense_support(name, scale, start, count):
    h = _h()
    w = workload(name, scale)
    o, d, t = w.pulses(start, count)
    out, _ = h.simulate(scene_for(w), w.params, _dev(o), _dev(d), _dev(t),
                        pulse_index_base=start, compact=True)
    g = out.numpy()
    off = g["wf_offset"].astype(np.int64)
    lens = np.diff(off)
    hp = h.make_params(w.params)
    nb, taps = h.helios_waveform_bins(hp), h.helios_pulse_taps(hp)
    assert off[0] == 0 and np.all(lens >= 0) and np.all(lens <= nb)
    r = oracle_run(w, np.arange(start, start + count), want_waveform=False)
    assert np.array_equal(lens, _support_from_oracle(r, nb, taps))
    assert np.array_equal(lens == 0, g["wf_first_bin"] < 0)
    wf = g["waveform"]
    for i in range(count):
        row = g["wf_compact"][off[i]:off[i + 1]]
        assert np.array_equal(row.view(np.uint32), wf[i, :lens[i]].view(np.uint32)), i
        assert not wf[i, lens[i]:].any(), i


def test_compact_host_staged_across_chunks_matches_device():
    # 279 subrays x 25000 pulses = three chunks of the staging pipeline; the
    # packed rows of each chunk are copied out once its offsets are known
    import torch
    h = _h()
    w = workload("C3", 0.03)
    p = replace(w.params, subray_count=279)
    n = 25000
    o, d, t = w.pulses(100, n)
    a, _ = h.simulate(scene_for(w), p, _dev(o), _dev(d), _dev(t), pulse_index_base=100,
                      compact=True)
    a = a.numpy()
    for pin in (False, True):
        out = h.alloc_outputs(n, h.make_params(p), device="cpu", pin_memory=pin, compact=True,
                              waveform=pin)
        args = [torch.from_numpy(x).pin_memory() for x in (o, d, t)] if pin else [o, d, t]
        h.simulate(scene_for(w), p, *args, pulse_index_base=100, outputs=out)
        b = out.numpy()
        assert np.array_equal(a["wf_offset"], b["wf_offset"])
        tot = int(a["wf_offset"][-1])
        assert np.array_equal(a["wf_compact"][:tot].view(np.uint32),
                              b["wf_compact"][:tot].view(np.uint32))
        for k in ("n_returns", "wf_first_bin", "returns"):
            assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k


def test_compact_capacity_contract():
    import ctypes
    torch = torch_cuda()
    h = _h()
    w = workload("C2", 0.125)
    n = 2000
    o, d, t = (_dev(x) for x in w.pulses(0, n))
    ref, _ = h.simulate(scene_for(w), w.params, o, d, t, compact=True)
    ref = ref.numpy()
    need = int(ref["wf_offset"][-1])
    hp = h.make_params(w.params)
    for dev in ("cuda", "cpu"):
        out = h.alloc_outputs(n, hp, device=dev, compact=True, compact_capacity=need // 2)
        po = h.helios.helios_pulses(ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(d.data_ptr()),
                                    ctypes.c_void_p(t.data_ptr()), n, 0)
        oo = h.helios.helios_outputs()
        for f, x in (("p_n_returns", out.n_returns), ("p_returns", out.returns),
                     ("p_wf_first_bin", out.wf_first_bin), ("p_waveform", out.waveform),
                     ("p_wf_compact", out.wf_compact), ("p_wf_offset", out.wf_offset)):
            setattr(oo, f, x.data_ptr())
        oo.wf_compact_capacity = need // 2
        with pytest.raises(h.HeliosError) as ei:
            h.helios_simulate(scene_for(w).handle, hp, po, oo)
        assert ei.value.status == h.helios.HELIOS_ERR_CAPACITY
        torch.cuda.synchronize()
        got = out.numpy()
        assert int(got["wf_offset"][-1]) == need  # the exact need is reported
        for k in ("n_returns", "wf_first_bin", "returns", "waveform", "wf_offset"):
            assert np.array_equal(ref[k].view(np.uint8), got[k].view(np.uint8)), k
        # rows that fit entirely were written
        fit = np.nonzero(ref["wf_offset"][1:] <= need // 2)[0]
        last = int(ref["wf_offset"][fit[-1] + 1])
        assert np.array_equal(ref["wf_compact"][:last].view(np.uint32),
                              got["wf_compact"][:last].view(np.uint32))
    # the Python layer grows the buffer to the reported need and reruns
    out = h.alloc_outputs(n, hp, compact=True, compact_capacity=10)
    out, _ = h.simulate(scene_for(w), w.params, o, d, t, outputs=out)
    got = out.numpy()
    assert np.array_equal(ref["wf_compact"][:need], got["wf_compact"][:need])


def test_offsets_only_and_compact_without_dense_rows():
    h = _h()
    w = workload("C4", 0.1)
    n = 3000
    o, d, t = (_dev(x) for x in w.pulses(7, n))
    ref, _ = h.simulate(scene_for(w), w.params, o, d, t, pulse_index_base=7, compact=True)
    ref = ref.numpy()
    out = h.alloc_outputs(n, w.params, waveform=False, compact=True)
    out.wf_compact = None  # lengths only
    h.simulate(scene_for(w), w.params, o, d, t, pulse_index_base=7, outputs=out)
    assert np.array_equal(ref["wf_offset"], out.numpy()["wf_offset"])
    out = h.alloc_outputs(n, w.params, waveform=False, compact=True)
    h.simulate(scene_for(w), w.params, o, d, t, pulse_index_base=7, outputs=out)
    g = out.numpy()
    tot = int(ref["wf_offset"][-1])
    assert np.array_equal(ref["wf_compact"][:tot], g["wf_compact"][:tot])
    assert np.array_equal(ref["returns"].view(np.uint8), g["returns"].view(np.uint8))


def _check_packed(g):
    nr = g["n_returns"].astype(np.int64)
    off = g["return_offset"].astype(np.int64)
    assert off[0] == 0 and np.array_equal(np.diff(off), nr)
    if g["returns"] is not None:
        used = np.arange(g["returns"].shape[1])[None, :] < nr[:, None]
        a = g["returns"][used]
        b = g["returns_packed"][:off[-1]]
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("fit", [0, 1])
def test_packed_returns_device_and_host(fit):
    # packed returns (used slots only) == the fixed slots, on the device and
    # through the host staging pipeline over several chunks, with and without
    # the echo-width fits (which finish the returns on their own stream)
    import torch
    h = _h()
    w = workload("C3", 0.03)
    p = replace(w.params, subray_count=279, fit_echo_width=fit, range_noise_sd_m=0.02)
    n = 25000
    o, d, t = w.pulses(100, n)
    a, _ = h.simulate(scene_for(w), p, _dev(o), _dev(d), _dev(t), pulse_index_base=100,
                      packed_returns=True)
    a = a.numpy()
    _check_packed(a)
    assert a["return_offset"][-1] > 1000
    for pin in (False, True):
        out = h.alloc_outputs(n, h.make_params(p), device="cpu", pin_memory=pin,
                              packed_returns=True, slots=False, waveform=False)
        args = [torch.from_numpy(x).pin_memory() for x in (o, d, t)] if pin else [o, d, t]
        h.simulate(scene_for(w), p, *args, pulse_index_base=100, outputs=out)
        b = out.numpy()
        assert b["returns"] is None
        assert np.array_equal(a["return_offset"], b["return_offset"])
        tot = int(a["return_offset"][-1])
        assert np.array_equal(a["returns_packed"][:tot].view(np.uint8),
                              b["returns_packed"][:tot].view(np.uint8))


def test_packed_returns_capacity_and_retry():
    h = _h()
    w = workload("C2", 0.125)
    n = 3000
    o, d, t = (_dev(x) for x in w.pulses(0, n))
    ref, _ = h.simulate(scene_for(w), w.params, o, d, t, packed_returns=True)
    ref = ref.numpy()
    need = int(ref["return_offset"][-1])
    out = h.alloc_outputs(n, w.params, packed_returns=True, returns_capacity=need // 3,
                          compact=True, compact_capacity=7)
    out, _ = h.simulate(scene_for(w), w.params, o, d, t, outputs=out)  # grows both, reruns
    g = out.numpy()
    assert g["returns_packed"].shape[0] == need
    assert np.array_equal(ref["returns_packed"][:need].view(np.uint8),
                          g["returns_packed"][:need].view(np.uint8))
    _check_packed(g)
