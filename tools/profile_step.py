"""Run a few helios_simulate steps of one workload (for ncu / compute-sanitizer).

  python tools/profile_step.py --config C2 --batch 200000 --steps 2
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--batch", type=int, default=200000)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--subray-hits", action="store_true")
    ap.add_argument("--fit-echo-width", action="store_true")
    ap.add_argument("--compact", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(args.config, args.scale)
    from dataclasses import replace
    w.params = replace(w.params, fit_echo_width=int(args.fit_echo_width))
    sc = h.Scene.from_workload_scene(w.scene)
    B = min(args.batch, w.n_pulses)
    hp = h.make_params(w.params)
    out = h.alloc_outputs(B, hp, subray_hits=args.subray_hits, compact=args.compact,
                          compact_capacity=B * h.helios_waveform_bins(hp) if args.compact else None)
    for i in range(args.steps):
        start = (i * B) % max(1, w.n_pulses - B + 1)
        o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, B))
        _, st = h.simulate(sc, hp, o, d, t, pulse_index_base=start, outputs=out, stats=True)
        print(f"step {i}: trace {st.trace_ms:.3f} ms, waveform {st.waveform_ms:.3f} ms, "
              f"launches {st.kernel_launches}", flush=True)
    torch.cuda.synchronize()
    sc.destroy()


if __name__ == "__main__":
    main()
