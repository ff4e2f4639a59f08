"""Device spans of one helios_simulate_batches call (HELIOS_TRACE_SPANS=1
prints them to stderr): b/B K6a, t/T K6, w/W K7 per chunk, c/C packed-row
copy-out, f/F fixed copy-out, ms from the call's start.

  python tools/spans.py C5 [batches] [batch_pulses] [--host]

--host: pinned host inputs and packed host outputs (bench.py's e2e arm)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg="C5", nb=3, B=1_000_000, host=False):
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(cfg)
    sc = h.Scene.from_workload_scene(w.scene)
    hp = h.make_params(w.params)
    batches = []
    for i in range(nb):
        o, d, t = w.pulses(i * B, B)
        if host:
            to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        else:
            to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        batches.append((to(o), to(d), to(t), i * B))
    if host:
        outs = [h.alloc_outputs(B, hp, device="cpu", waveform=False, pin_memory=True,
                                compact=True, compact_capacity=B * 192, packed_returns=True,
                                slots=False, returns_capacity=B * w.params.max_returns)
                for _ in range(nb)]
    else:
        outs = [h.alloc_outputs(B, hp, device="cuda") for _ in range(nb)]
    h.simulate_batches(sc, hp, batches, outs)  # warm (and grow capacities)
    torch.cuda.synchronize()
    with h.tuning(trace_spans=1):
        h.simulate_batches(sc, hp, batches, outs)
    torch.cuda.synchronize()
    sc.destroy()


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args[0].upper() if args else "C5", int(args[1]) if len(args) > 1 else 3,
         int(args[2]) if len(args) > 2 else 1_000_000, "--host" in sys.argv)
