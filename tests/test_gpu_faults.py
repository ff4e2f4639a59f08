"""Injected device-allocation failures (SURVEY s.5 failure detection:
helios_tuning.fault_alloc_bytes makes every library allocation above the
limit fail as out of memory): scene creation, the build, a simulate call and
an accel import each return HELIOS_ERR_OUT_OF_MEMORY with a message, leave no
half-built state behind, and the library works -- bitwise as before -- once
the limit is lifted."""
import numpy as np
import pytest

from gpu_util import torch_cuda, workload

pytestmark = pytest.mark.gpu
OOM = 2


def _h():
    import paper_2101_09154_b200 as h
    return h


def test_out_of_memory_paths_fail_cleanly_and_recover():
    torch = torch_cuda()
    h = _h()
    w = workload("C3", 0.03)
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ref_scene = h.Scene.from_workload_scene(w.scene)
    o, d, tm = (t(a) for a in w.pulses(100, 2000))
    ref, _ = h.simulate(ref_scene, w.params, o, d, tm, pulse_index_base=100)
    torch.cuda.synchronize()
    ref = ref.numpy()
    blob = ref_scene.export_accel()
    unbuilt = h.Scene(t(w.scene.tri_xyz), t(w.scene.tri_reflectance), build=False)
    limit = 4096  # every triangle array of the scene is larger
    with h.tuning(fault_alloc_bytes=limit):
        with pytest.raises(h.HeliosError) as e:
            h.Scene(t(w.scene.tri_xyz), t(w.scene.tri_reflectance))
        assert e.value.status == OOM and "memory" in str(e.value)
        with pytest.raises(h.HeliosError) as e:
            h.helios_build_accel(unbuilt.handle)
        assert e.value.status == OOM
        with pytest.raises(h.HeliosError) as e:
            unbuilt.import_accel(blob)
        assert e.value.status == OOM
        # a new caller stream needs new scratch (the default stream's is cached)
        st = torch.cuda.Stream()
        with pytest.raises(h.HeliosError) as e:
            h.simulate(ref_scene, w.params, o, d, tm, pulse_index_base=100, stream=st)
        assert e.value.status == OOM
        st.synchronize()
    assert h.helios_get_tuning().fault_alloc_bytes == 0
    # nothing half-built: the failed build / import left the scene unbuilt
    with pytest.raises(h.HeliosError) as e:
        unbuilt.export_accel()
    assert e.value.status == 4  # NOT_BUILT
    h.helios_build_accel(unbuilt.handle)
    for sc in (ref_scene, unbuilt):
        out, _ = h.simulate(sc, w.params, o, d, tm, pulse_index_base=100)
        torch.cuda.synchronize()
        got = out.numpy()
        for k in ("n_returns", "wf_first_bin", "waveform", "returns"):
            assert np.array_equal(np.ascontiguousarray(got[k]).view(np.uint8),
                                  np.ascontiguousarray(ref[k]).view(np.uint8)), k
    assert unbuilt.export_accel() == blob
    ref_scene.destroy()
    unbuilt.destroy()
