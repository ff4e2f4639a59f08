"""bench.py's e2e arm in isolation: K host batches (pinned inputs, packed host
outputs) through helios_simulate_batches, timed with CUDA events; prints the
per-step time of repeated calls and the device spans of the last one.

  python tools/e2e_repro.py C3 [steps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg="C3", K=5, B=1_000_000):
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(cfg)
    sc = h.Scene.from_workload_scene(w.scene)
    hp = h.make_params(w.params)
    hb = []
    for i in range(K):
        o, d, t = w.pulses(i * B, B)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hb.append((pin(o), pin(d), pin(t), i * B))
    houts = [h.alloc_outputs(B, hp, device="cpu", waveform=False, pin_memory=True, compact=True,
                             compact_capacity=B * 192, packed_returns=True, slots=False,
                             returns_capacity=B * w.params.max_returns) for _ in range(K)]
    s = torch.cuda.current_stream()
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        if rep == 3:
            with h.tuning(trace_spans=1):
                h.simulate_batches(sc, hp, hb, houts)
        else:
            h.simulate_batches(sc, hp, hb, houts)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"rep {rep}: {e0.elapsed_time(e1) / K:.3f} ms/step (events), "
              f"{(time.perf_counter() - t0) * 1e3 / K:.3f} ms/step (host)", flush=True)
    sc.destroy()


if __name__ == "__main__":
    main(sys.argv[1].upper() if len(sys.argv) > 1 else "C3",
         int(sys.argv[2]) if len(sys.argv) > 2 else 5)
