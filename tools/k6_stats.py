"""Per-lane and per-warp traversal counts of K6 (instrumented variant) for a
few configs: how much of a warp's work is the union of its lanes' paths.

  python tools/k6_stats.py [C5 C3 C2 ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfgs):
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    for cfg in cfgs:
        w = make_workload(cfg)
        sc = h.Scene.from_workload_scene(w.scene)
        B = min(200_000, w.n_pulses)
        start = min(w.n_pulses - B, w.n_pulses // 3)
        o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, B))
        _, st = h.simulate(sc, w.params, o, d, t, pulse_index_base=start, counters=True,
                           waveform=False)
        N = w.params.subray_count
        lanes = 96 if N == 91 else N
        warps = B * lanes / 32
        S = B * N
        print(f"{cfg}: per subray: nodes {st.nodes_visited / S:.2f} tris {st.tris_tested / S:.2f} "
              f"fp64 {st.fp64_tests / S:.2f}; per pulse: K6a nodes {st.beam_nodes / B:.1f}; "
              f"per warp: entries {st.warp_entries / warps:.1f} walked "
              f"{st.warp_entries_walked / warps:.1f} steps {st.warp_steps / warps:.1f} "
              f"leaf tris {st.warp_leaf_tris / warps:.1f}; lane tris / warp tris "
              f"{st.tris_tested / max(1, st.warp_leaf_tris) :.2f} "
              f"(lanes per tested triangle, of {32 if N >= 32 else N}); in-walk fp64 groups "
              f"per warp {st.warp_fp64_in_walk / warps:.2f}, second definite hits per subray "
              f"{st.second_definite_hits / S:.4f}", flush=True)
        sc.destroy()
        del w


if __name__ == "__main__":
    main([a.upper() for a in sys.argv[1:]] or ["C5", "C3", "C2"])
