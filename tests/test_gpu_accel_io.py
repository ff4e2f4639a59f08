"""Saving and loading a built acceleration structure (helios_accel_export /
helios_accel_import; "Saving and loading already built scenes"): a
scene that imports the blob instead of building traces bitwise like the
exporting one; blobs from other triangles, damaged or truncated blobs are
rejected; the blob may live in host or device memory."""
import ctypes

import numpy as np
import pytest

from gpu_util import torch_cuda, workload

pytestmark = pytest.mark.gpu


def _h():
    import paper_2101_09154_b200 as h
    return h


def _run(h, torch, sc, w, start=0, n=3000):
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, n))
    out, _ = h.simulate(sc, w.params, o, d, t, pulse_index_base=start, subray_hits=True)
    torch.cuda.synchronize()
    return out.numpy()


def _same(a, b):
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
        assert np.array_equal(np.ascontiguousarray(a[k]).view(np.uint8),
                              np.ascontiguousarray(b[k]).view(np.uint8)), k


@pytest.mark.parametrize("cfg,scale", [("C2", 0.125), ("C3", 0.03), ("C5", 0.03)])
def test_imported_tree_traces_bitwise_like_the_built_one(cfg, scale):
    torch = torch_cuda()
    h = _h()
    w = workload(cfg, scale)
    a = h.Scene.from_workload_scene(w.scene)
    blob = a.export_accel()
    ref = _run(h, torch, a, w)
    t = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x)).cuda()
    b = h.Scene(t(w.scene.tri_xyz), t(w.scene.tri_reflectance), t(w.scene.voxel_pad),
                w.scene.grid_origin, w.scene.voxel_size, w.scene.g_lut, build=False)
    with pytest.raises(h.HeliosError):  # not built yet
        b.export_accel()
    b.import_accel(blob)
    ia, ib = a.info(), b.info()
    assert (ia.n_nodes, ia.max_depth) == (ib.n_nodes, ib.max_depth)
    _same(_run(h, torch, b, w), ref)
    assert b.export_accel() == blob  # the round trip is exact
    # a blob held in device memory
    dblob = torch.from_numpy(np.frombuffer(blob, np.uint8).copy()).cuda()
    c = h.Scene(t(w.scene.tri_xyz), t(w.scene.tri_reflectance), t(w.scene.voxel_pad),
                w.scene.grid_origin, w.scene.voxel_size, w.scene.g_lut, build=False)
    assert h.lib().helios_accel_import(c.handle, ctypes.c_void_p(dblob.data_ptr()),
                                       len(blob), None) == 0
    _same(_run(h, torch, c, w), ref)
    for s in (a, b, c):
        s.destroy()


def test_foreign_damaged_and_truncated_blobs_are_rejected():
    torch = torch_cuda()
    h = _h()
    w = workload("C2", 0.125)
    a = h.Scene.from_workload_scene(w.scene)
    blob = a.export_accel()
    xyz = np.array(w.scene.tri_xyz, np.float32, copy=True)
    xyz[17, 1, 2] = np.nextafter(xyz[17, 1, 2], np.float32(np.inf))  # one ulp of one vertex
    other = h.Scene(torch.from_numpy(xyz).cuda(),
                    torch.from_numpy(np.ascontiguousarray(w.scene.tri_reflectance)).cuda(),
                    build=False)
    with pytest.raises(h.HeliosError) as e:
        other.import_accel(blob)
    assert e.value.status == 1 and "other triangles" in str(e.value)
    same = h.Scene(torch.from_numpy(np.ascontiguousarray(w.scene.tri_xyz)).cuda(),
                   torch.from_numpy(np.ascontiguousarray(w.scene.tri_reflectance)).cuda(),
                   build=False)
    bad = bytearray(blob)
    bad[0] ^= 0xFF  # magic
    for damaged in (bytes(bad), blob[:100], blob[:-64]):
        with pytest.raises(h.HeliosError) as e:
            same.import_accel(damaged)
        assert e.value.status == 1
    same.import_accel(blob)  # the intact blob still loads
    for s in (a, other, same):
        s.destroy()
