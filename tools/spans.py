"""Device spans of one helios_simulate_batches call (HELIOS_TRACE_SPANS=1
prints them to stderr): b/B K6a, t/T K6, w/W K7 per chunk, ms from the call's
start.  python tools/spans.py C5 [batches] [batch_pulses]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg="C5", nb=3, B=1_000_000):
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(cfg)
    sc = h.Scene.from_workload_scene(w.scene)
    hp = h.make_params(w.params)
    batches = []
    for i in range(nb):
        o, d, t = w.pulses(i * B, B)
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        batches.append((to(o), to(d), to(t), i * B))
    outs = [h.alloc_outputs(B, hp, device="cuda") for _ in range(nb)]
    h.simulate_batches(sc, hp, batches, outs)  # warm
    torch.cuda.synchronize()
    with h.tuning(trace_spans=1):
        h.simulate_batches(sc, hp, batches, outs)
    torch.cuda.synchronize()
    sc.destroy()


if __name__ == "__main__":
    main(sys.argv[1].upper() if len(sys.argv) > 1 else "C5",
         int(sys.argv[2]) if len(sys.argv) > 2 else 3,
         int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000)
