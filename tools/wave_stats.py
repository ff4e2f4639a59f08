"""Distribution of K7's evaluation paths on a workload, from the subray
export of one GPU run: per pulse the bin offsets o_s = k_s - k0 of its hits,
the number of distinct offsets G, max offset, and the support S.

  python tools/wave_stats.py [C5] [pulses]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(cfg="C5", n=200_000):
    import torch
    import paper_2101_09154_b200 as h
    from workloads import make_workload
    w = make_workload(cfg)
    p = w.params
    hp = h.make_params(p)
    taps = int(np.ceil(20 * p.pulse_length_ns / 1.75 / p.bin_width_ns))
    nb = h.helios_waveform_bins(hp)
    sc = h.Scene.from_workload_scene(w.scene)
    start = min(w.n_pulses - n, w.n_pulses // 3)
    o, d, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in w.pulses(start, n))
    out, _ = h.simulate(sc, p, o, d, t, pulse_index_base=start, subray_hits=True, waveform=False)
    g = out.numpy()
    sc.destroy()
    R = g["subray_hits"]["range_m"]
    k = np.floor(2 * R / 299792458.0 / (p.bin_width_ns * 1e-9))
    hit = np.isfinite(k)
    k0 = np.where(hit, k, np.inf).min(axis=1)
    has = np.isfinite(k0)
    off = np.where(hit, k - k0[:, None], np.nan)[has]
    off = np.where(off >= nb, np.nan, off)
    maxoff = np.nanmax(off, axis=1)
    G = np.array([len(np.unique(r[np.isfinite(r)])) for r in off])
    S = np.minimum(nb, maxoff + taps)
    wide = maxoff >= 64
    print(f"{cfg}: {n} pulses, {has.mean():.3f} with hits; taps {taps}, n_bins {nb}")
    print(f"  grouped (maxoff < 64): {np.mean(~wide):.3f}  [G<=16 {np.mean(~wide & (G <= 16)):.3f}]")
    print(f"  wide (maxoff >= 64): {np.mean(wide):.3f}  [G<=64 {np.mean(wide & (G <= 64)):.3f}]")
    for cap in (448, 512):
        print(f"  S > {cap}: {np.mean(S > cap):.4f}")
    print("  G quantiles (grouped):", np.percentile(G[~wide], [50, 90, 99]).tolist())
    if wide.any():
        print("  G quantiles (wide):", np.percentile(G[wide], [50, 90, 99]).tolist(),
              " S quantiles (wide):", np.percentile(S[wide], [50, 90, 99]).tolist())
        cov = [len(np.unique(np.concatenate([np.arange(int(x) // 32, min(int(s) - 1, int(x) + taps - 1) // 32 + 1)
                                              for x in np.unique(r[np.isfinite(r)])])))
               for r, s in zip(off[wide][:5000], S[wide][:5000])]
        print("  covered 32-bin blocks (wide) median/90%:", np.percentile(cov, [50, 90]).tolist(),
              " of S/32 median", float(np.median(np.ceil(S[wide] / 32))))


if __name__ == "__main__":
    main(sys.argv[1].upper() if len(sys.argv) > 1 else "C5",
         int(sys.argv[2]) if len(sys.argv) > 2 else 200_000)
