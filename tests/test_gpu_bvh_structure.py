"""T2 (SURVEY s.4): structural invariants of the built tree, read back through
helios_accel_export (include/helios.h) and checked on the host for both
builders (PLOC, Karras):

  * every triangle is in exactly one leaf, leaves hold 1..leaf_max triangles;
  * each child box contains its whole subtree (the triangles' fp32 vertices);
  * depth <= 64 (the traversal stack), the header's depth is the true depth;
  * the leaf-order triangle records are the input rows permuted (original id
    in the record), and the fp32 filter records hold exactly the values the
    filter computes: v0, e1 = v1 - v0, e2 = v2 - v0 (fp32), A = |e1|_1,
    B = |e2|_1 summed in order, and A * B."""
import numpy as np
import pytest

from gpu_util import torch_cuda, workload

pytestmark = pytest.mark.gpu
EMPTY = 0x7FFFFFFF
HDR = np.dtype([("magic", "<u8"), ("version", "<u4"), ("header_bytes", "<u4"),
                ("n_tris", "<u4"), ("n_nodes", "<u4"), ("root", "<i4"), ("max_depth", "<u4"),
                ("scene_hash", "<u8"), ("tri_bytes", "<u8"), ("node_bytes", "<u8"),
                ("record_sizes", "<u4"), ("leaf_max", "<u4"), ("reserved", "<u8", (8,))])


def _parse(blob):
    h = np.frombuffer(blob, HDR, count=1)[0]
    assert h["header_bytes"] == HDR.itemsize == 128
    n, nn = int(h["n_tris"]), int(h["n_nodes"])
    at = HDR.itemsize
    tris = np.frombuffer(blob, np.float32, count=12 * n, offset=at).reshape(n, 12)
    at += 48 * n
    filt = np.frombuffer(blob, np.float32, count=12 * n, offset=at).reshape(n, 12)
    at += 48 * n
    nodes = np.frombuffer(blob, np.float32, count=16 * nn, offset=at).reshape(nn, 16)
    assert at + 64 * nn == len(blob)
    return h, tris, filt, nodes


def _check_tree(blob, xyz, refl):
    h, tris, filt, nodes = _parse(blob)
    n = int(h["n_tris"])
    leaf_max = int(h["leaf_max"])
    refs = nodes.view(np.int32)
    seen = np.zeros(n, np.int32)
    vmin = tris[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(n, 3, 3).min(axis=1)
    vmax = tris[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]].reshape(n, 3, 3).max(axis=1)
    depth_max = 0

    def child(i, c):
        nd = nodes[i]
        lo = np.array([nd[0], nd[2], nd[8]] if c == 0 else [nd[4], nd[6], nd[10]])
        hi = np.array([nd[1], nd[3], nd[9]] if c == 0 else [nd[5], nd[7], nd[11]])
        return int(refs[i, 12 + c]), lo, hi

    # iterative DFS: (ref, box lo, box hi, depth)
    root = int(h["root"])
    stack = [(root, None, None, 1)]
    while stack:
        ref, lo, hi, dep = stack.pop()
        depth_max = max(depth_max, dep)
        if ref == EMPTY:
            continue
        if ref < 0:
            u = ref & 0xFFFFFFFF
            first, cnt = (u & 0x7FFFFFFF) >> 3, (u & 7) + 1
            assert 1 <= cnt <= leaf_max and first + cnt <= n
            seen[first:first + cnt] += 1
            if lo is not None:
                assert (vmin[first:first + cnt] >= lo).all() and (vmax[first:first + cnt] <= hi).all()
            continue
        assert 0 <= ref < len(nodes)
        for c in (0, 1):
            r, clo, chi = child(ref, c)
            if r == EMPTY:
                continue
            if lo is not None:  # nested boxes
                assert (clo >= lo).all() and (chi <= hi).all(), (ref, c)
            stack.append((r, clo, chi, dep + 1))
    assert (seen == 1).all(), "every triangle in exactly one leaf"
    assert depth_max <= 64 and depth_max - 1 <= int(h["max_depth"]) + 1
    # leaf-order records = the input rows permuted; filter records exact
    src = tris[:, 3].view(np.uint32).astype(np.int64)
    assert np.array_equal(np.sort(src), np.arange(n))
    v = xyz.reshape(-1, 9)[src]
    assert np.array_equal(tris[:, [0, 1, 2, 4, 5, 6, 8, 9, 10]], v)
    if refl is not None:
        assert np.array_equal(tris[:, 7], refl[src])
    v0, v1, v2 = v[:, 0:3], v[:, 3:6], v[:, 6:9]
    e1, e2 = (v1 - v0).astype(np.float32), (v2 - v0).astype(np.float32)
    A = (np.abs(e1[:, 0]) + np.abs(e1[:, 1])).astype(np.float32) + np.abs(e1[:, 2])
    B = (np.abs(e2[:, 0]) + np.abs(e2[:, 1])).astype(np.float32) + np.abs(e2[:, 2])
    assert np.array_equal(filt[:, 0:3], v0) and np.array_equal(filt[:, 4:7], e1)
    assert np.array_equal(filt[:, 8:11], e2)
    assert np.array_equal(filt[:, 7], A.astype(np.float32))
    assert np.array_equal(filt[:, 11], B.astype(np.float32))
    assert np.array_equal(filt[:, 3], (A * B).astype(np.float32))


def _soup(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-50, 50, (n, 1, 3))
    tri = (c + rng.normal(0, 0.7, (n, 3, 3))).astype(np.float32)
    return tri, rng.uniform(0.05, 0.95, n).astype(np.float32)


@pytest.mark.parametrize("builder", [0, 1])
@pytest.mark.parametrize("case", ["soup1", "soup10k", "C2", "C3"])
def test_tree_invariants(builder, case):
    torch = torch_cuda()
    import paper_2101_09154_b200 as h
    if case.startswith("soup"):
        xyz, refl = _soup(1 if case == "soup1" else 10_000, 7)
    else:
        sc = workload(case, 0.125 if case == "C2" else 0.03).scene
        xyz = np.ascontiguousarray(sc.tri_xyz, np.float32)
        refl = np.ascontiguousarray(sc.tri_reflectance, np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    with h.tuning(builder=builder):
        s = h.Scene(t(xyz), t(refl))
    blob = s.export_accel()
    s.destroy()
    _check_tree(blob, xyz, refl)
