"""Runtime primitives and call shapes of libhelios.so on the GPU:

* the hand-written radix sort and prefix sums (include/helios_util.h; the K2
  sort of helios_build_accel and the packed-output scans) against numpy's
  stable argsort / cumsum;
* helios_simulate_batches (one pipelined call over several batches) bitwise
  equal to separate helios_simulate calls, with device, host and packed
  outputs mixed;
* calls on several caller streams (the per-stream scratch cache), including
  streams destroyed before the scene.
"""
import numpy as np
import pytest

from gpu_util import gpu_run, scene_for, torch_cuda, workload

pytestmark = pytest.mark.gpu


def _h():
    import paper_2101_09154_b200 as h
    return h


@pytest.mark.parametrize("n", [0, 1, 2, 100, 2047, 2048, 2049, 65537, 1_000_003])
@pytest.mark.parametrize("bits", [63, 30, 8])
def test_radix_sort_is_numpys_stable_argsort(n, bits):
    torch = torch_cuda()
    h = _h()
    rng = np.random.default_rng(n * 7 + bits)
    # many duplicates (Morton codes of co-located centroids) plus a wide spread
    keys = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    dup = rng.random(n) < 0.3
    keys[dup] = rng.integers(0, 50, int(dup.sum()), dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint32)
    dk = torch.from_numpy(keys.view(np.int64).copy()).cuda()
    dv = torch.from_numpy(vals.view(np.int32).copy()).cuda()
    h.util_sort_pairs_u64(dk, dv, bits)
    masked = keys & np.uint64((1 << bits) - 1) if bits < 64 else keys
    order = np.argsort(masked, kind="stable")
    got_v = dv.cpu().numpy().view(np.uint32)
    got_k = dk.cpu().numpy().view(np.uint64)
    assert np.array_equal(got_v, vals[order])
    assert np.array_equal(got_k, keys[order])


@pytest.mark.parametrize("n", [1, 5, 2048, 2049, 3 * 2048 * 2048 + 17])
@pytest.mark.parametrize("inclusive", [True, False])
def test_scan_is_cumsum(n, inclusive):
    torch = torch_cuda()
    h = _h()
    rng = np.random.default_rng(n)
    x = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    d = torch.from_numpy(x.view(np.int64).copy()).cuda()
    out = torch.empty_like(d)
    h.util_scan_u64(d, out, inclusive)
    ref = np.cumsum(x, dtype=np.uint64)
    if not inclusive:
        ref = np.concatenate([[np.uint64(0)], ref[:-1]])
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref)
    h.util_scan_u64(d, d, inclusive)  # in place
    assert np.array_equal(d.cpu().numpy().view(np.uint64), ref)


def _outputs_equal(a, b, keys=("n_returns", "wf_first_bin", "waveform", "returns",
                               "subray_hits")):
    for k in keys:
        if a.get(k) is None:
            continue
        assert np.array_equal(np.ascontiguousarray(a[k]).view(np.uint8),
                              np.ascontiguousarray(b[k]).view(np.uint8)), k


def test_batches_equal_separate_calls():
    """One helios_simulate_batches call over ragged batches (device outputs,
    pinned-host outputs, packed device outputs) == separate calls, bitwise."""
    torch = torch_cuda()
    h = _h()
    w = workload("C5", 0.03)
    sc = scene_for(w)
    hp = h.make_params(w.params)
    nb = h.helios_waveform_bins(hp)
    spans = [(300, 2500), (9000, 1), (20000, 4099), (40000, 7000)]
    kinds = ["device", "host", "packed", "device"]
    batches, outs = [], []
    for (start, cnt), kind in zip(spans, kinds):
        o, d, t = w.pulses(start, cnt)
        dev = kind != "host"
        conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()) if dev else \
            (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory())
        batches.append((conv(o), conv(d), conv(t), start))
        if kind == "packed":
            outs.append(h.alloc_outputs(cnt, hp, device="cuda", waveform=False, compact=True,
                                        compact_capacity=cnt * nb, packed_returns=True,
                                        slots=False, returns_capacity=cnt * hp.max_returns,
                                        subray_hits=True))
        else:
            outs.append(h.alloc_outputs(cnt, hp, device="cuda" if dev else "cpu",
                                        pin_memory=not dev, subray_hits=True))
    st = h.simulate_batches(sc, hp, batches, outs, stats=True)
    torch.cuda.synchronize()
    assert st.batches == len(spans) and st.pulses == sum(c for _, c in spans)
    for (start, cnt), kind, out in zip(spans, kinds, outs):
        ref = gpu_run(w, start, cnt)
        got = out.numpy()
        if kind == "packed":
            off = got["wf_offset"].view(np.uint64)
            roff = got["return_offset"].view(np.uint64)
            for p in range(cnt):
                row = got["wf_compact"][off[p]:off[p + 1]]
                assert np.array_equal(row, ref["waveform"][p][:len(row)])
                assert not ref["waveform"][p][len(row):].any()
                r = got["returns_packed"][roff[p]:roff[p + 1]]
                m = int(ref["n_returns"][p])
                assert len(r) == m
                assert np.array_equal(r.view(np.uint8), ref["returns"][p][:m].view(np.uint8))
            _outputs_equal(got, ref, ("n_returns", "wf_first_bin", "subray_hits"))
        else:
            _outputs_equal(got, ref)


def test_calls_on_several_streams():
    """The per-stream scratch cache: the same batch on the default stream and
    on six other streams (more than the cache keeps idle) gives bitwise the
    same outputs; streams destroyed before the scene are never touched."""
    torch = torch_cuda()
    h = _h()
    w = workload("C2", 0.125)
    sc = h.Scene.from_workload_scene(w.scene)
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(500, 3000))
    ref, _ = h.simulate(sc, w.params, o, d, t, pulse_index_base=500)
    torch.cuda.synchronize()
    ref = ref.numpy()
    for i in range(6):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            out, _ = h.simulate(sc, w.params, o, d, t, pulse_index_base=500, stream=st)
        st.synchronize()
        _outputs_equal(out.numpy(), ref)
        del st
    torch.cuda.synchronize()
    sc.destroy()


def test_tuning_switches_are_validated():
    h = _h()
    t = h.helios_get_tuning()
    bad = h.helios_tuning()
    bad.beam_prepass, bad.builder, bad.lane_order, bad.pad_lanes = -1, 0, 1, -1
    bad.chunk_pulses = 5  # below 1024
    with pytest.raises(h.HeliosError):
        h.helios_set_tuning(bad)
    after = h.helios_get_tuning()
    assert bytes(after) == bytes(t)


def test_async_calls_equal_blocking_calls():
    """helios_simulate_batches_async: two calls in flight on two caller streams
    (device and pinned-host outputs) while the host thread is free, each
    bitwise equal to the blocking call; stats come back through the wait."""
    torch = torch_cuda()
    h = _h()
    w = workload("C5", 0.03)
    sc = scene_for(w)
    hp = h.make_params(w.params)
    specs = [((300, 2500), (9000, 3001)), ((20000, 4099), (40000, 700))]
    calls, outs_all = [], []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for ci, spans in enumerate(specs):
        batches, outs = [], []
        for start, cnt in spans:
            o, d, t = w.pulses(start, cnt)
            dev = ci == 0
            conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()) if dev else \
                (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory())
            batches.append((conv(o), conv(d), conv(t), start))
            outs.append(h.alloc_outputs(cnt, hp, device="cuda" if dev else "cpu",
                                        pin_memory=not dev, subray_hits=True))
        torch.cuda.synchronize()  # inputs in place before a worker thread reads them
        calls.append(h.simulate_batches_async(sc, hp, batches, outs, stream=streams[ci],
                                              stats=True))
        outs_all.append((spans, outs))
    for c, (spans, outs) in zip(calls, outs_all):
        st = c.wait()
        assert st.batches == len(spans) and st.pulses == sum(n for _, n in spans)
        with pytest.raises(RuntimeError):
            c.wait()  # a handle is waited for once
        for (start, cnt), out in zip(spans, outs):
            _outputs_equal(out.numpy(), gpu_run(w, start, cnt))
    torch.cuda.synchronize()


def test_async_call_reports_errors_at_the_wait():
    torch = torch_cuda()
    h = _h()
    w = workload("C2", 0.125)
    sc = scene_for(w)
    hp = h.make_params(w.params)
    hp.subray_count = 20  # in neither pattern sequence (R1)
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(0, 100))
    out = h.alloc_outputs(100, h.make_params(w.params), device="cuda")
    c = h.simulate_batches_async(sc, hp, [(o, d, t, 0)], [out])
    with pytest.raises(h.HeliosError) as e:
        c.wait()
    assert e.value.status == 1 and "subray_count" in str(e.value)
