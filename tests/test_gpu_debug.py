"""The assert-enabled debug build (libhelios_debug.so, -DHELIOS_DEBUG: the
kernels check their invariants -- traversal stack depth, beam entry list
bound, subray table index, waveform window, a contributor for every peak --
and trap on a violation; it stands in for compute-sanitizer, which this pool
does not offer).  Every config runs under it in a separate process (the
library is loaded once per process) and must (a) not trap and (b) give
outputs bitwise equal to the release library's."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2101_09154_b200 as h
from workloads import make_workload
from dataclasses import replace
out = {{}}
for cfg, scale, n, fit in {cases!r}:
    w = make_workload(cfg, scale)
    p = replace(w.params, fit_echo_width=fit)
    sc = h.Scene.from_workload_scene(w.scene)
    n = min(n, w.n_pulses)
    start = (w.n_pulses - n) // 2
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, n))
    r, _ = h.simulate(sc, p, o, d, t, pulse_index_base=start, subray_hits=True)
    g = r.numpy()
    torch.cuda.synchronize()
    for k in ("n_returns", "wf_first_bin", "waveform", "returns", "subray_hits"):
        out[cfg + "/" + k] = np.ascontiguousarray(g[k]).view(np.uint8)
    sc.destroy()
np.savez({path!r}, **out)
from paper_2101_09154_b200 import helios as hh
print("lib", hh.LIB_PATH)
"""

CASES = [("C1", 1.0, 10_000, 0), ("C2", 0.1, 20_000, 1), ("C3", 0.05, 20_000, 0),
         ("C4", 0.1, 20_000, 1), ("C5", 0.02, 20_000, 0), ("C6", 0.2, 20_000, 0)]


def _run(lib, path):
    env = dict(os.environ, HELIOS_LIB=lib)
    code = RUN.format(root=ROOT, cases=CASES, path=path)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=1200)
    assert p.returncode == 0, p.stderr[-3000:]
    assert lib in p.stdout, p.stdout
    return np.load(path)


def test_debug_build_checks_pass_and_match_release(tmp_path):
    torch_cuda()
    from paper_2101_09154_b200 import build as b
    dbg = b.build_debug()
    rel = b.build()
    a = _run(dbg, str(tmp_path / "debug.npz"))
    r = _run(rel, str(tmp_path / "release.npz"))
    assert sorted(a.files) == sorted(r.files)
    for k in a.files:
        assert np.array_equal(a[k], r[k]), k
