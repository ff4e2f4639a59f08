"""Where does the end-to-end time go?  Times helios_simulate on one batch with
inputs / outputs placed on the device or in pinned host memory, one output
kind at a time (CUDA events around the calls).

  python tools/e2e_probe.py --config C5 --batch 1000000 --steps 3
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--stats", action="store_true", help="also time with stats=True")
    args = ap.parse_args()
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(args.config)
    sc = h.Scene.from_workload_scene(w.scene)
    hp = h.make_params(w.params)
    nb = h.helios_waveform_bins(hp)
    B = min(args.batch, w.n_pulses)
    o, d, t = w.pulses(args.start, B)
    dev_in = [torch.from_numpy(x).cuda() for x in (o, d, t)]
    host_in = [torch.from_numpy(x).pin_memory() for x in (o, d, t)]
    N = w.params.subray_count

    def outs(device, packed):
        pin = device == "cpu"
        return h.alloc_outputs(B, hp, device=device, pin_memory=pin, waveform=not packed,
                               compact=packed, compact_capacity=B * nb if packed else None,
                               packed_returns=packed, slots=not packed,
                               returns_capacity=B * w.params.max_returns if packed else None)

    def timed(inp, out, stats=False):
        h.simulate(sc, hp, *inp, outputs=out, stats=stats)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            h.simulate(sc, hp, *inp, outputs=out, stats=stats)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        return ms, B * N / (ms / 1e3) / 1e6

    for name, inp, dev, packed in (("dev in, dev out, dense", dev_in, "cuda", False),
                                   ("dev in, dev out, packed", dev_in, "cuda", True),
                                   ("host in, dev out, packed", host_in, "cuda", True),
                                   ("dev in, host out, packed", dev_in, "cpu", True),
                                   ("host in, host out, packed", host_in, "cpu", True)):
        ms, mr = timed(inp, outs(dev, packed))
        _, st = h.simulate(sc, hp, *inp, outputs=outs(dev, packed), stats=True)
        print(f"{args.config} {name:28s} {ms:8.2f} ms/step  {mr:8.1f} Mrays/s  "
              f"K6 {st.trace_ms:6.2f} ms  K7 {st.waveform_ms:6.2f} ms", flush=True)
        if args.stats:
            ms, mr = timed(inp, outs(dev, packed), stats=True)
            print(f"{args.config} {name + ' +stats':28s} {ms:8.2f} ms/step  {mr:8.1f} Mrays/s",
                  flush=True)
    sc.destroy()


if __name__ == "__main__":
    main()
