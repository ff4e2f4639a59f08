"""Per-kernel DRAM traffic, instruction counts and limiter metrics from one
`ncu --set full` capture of tools/profile_step.py, written into
profiles/traffic.json under the config's key (bench.py reads it for the
roofline 'traffic', 'ncu_limiter' and 'issue_roofline' fields).

  python tools/traffic_from_ncu.py gpurun_out/x/full.ncu-rep C5 "<source text>" [pulses]

Units: K6a + K6 per subray (pulses of the captured launch x N), K7 per pulse.
`pulses`: pulses per captured launch -- capture with HELIOS_CHUNK_PULSES=50000 (as
tools/gpu_check.sh does) so that every launch covers exactly 50000 pulses.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_OF = {"C1": 19, "C2": 19, "C3": 37, "C4": 19, "C5": 91, "C6": 37}
COLS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active")
PIPES = {"fp64_pipe_busy": COLS[8], "alu_pipe_busy": COLS[9], "fma_pipe_busy": COLS[10]}


def scale(unit, v):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3}
    return float(v.replace(",", "")) * f.get(unit, 1)


def main(rep, cfg, source, pulses=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = {c: h.index(c) for c in COLS}
    kn = h.index("Kernel Name")
    per = {}
    for r in rows[2:]:
        name = r[kn]
        wave_main = re.search(r"k_waveform<(\(bool\))?(0|false)", name)
        key = ("k_beam" if ("k_beam<0>" in name or "k_beam<false>" in name)
               else "k_trace" if ("k_trace<0," in name or "k_trace<false" in name)
               else "k_waveform" if wave_main
               else "k_waveform_wide" if "k_waveform" in name else None)
        if key is None or key in per:
            continue
        per[key] = {c: scale(units[idx[c]], r[idx[c]]) for c in COLS}
    N = N_OF[cfg]
    chunk = int(pulses) if pulses else 50000
    subrays = chunk * N
    t = per["k_trace"]
    b = per.get("k_beam", {c: 0.0 for c in COLS})
    # K7 = the main pass + the wide pass (pulses whose support exceeds the
    # shared-memory window) of the same chunk
    w = dict(per["k_waveform"])
    ww = per.get("k_waveform_wide")
    if ww:
        for c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "smsp__inst_executed.sum"):
            w[c] += ww[c]
    rec = {
        "source": source,
        "k_trace": {
            "dram_bytes": t["dram__bytes_read.sum"] + t["dram__bytes_write.sum"]
                          + b["dram__bytes_read.sum"] + b["dram__bytes_write.sum"],
            "warp_inst": t["smsp__inst_executed.sum"] + b["smsp__inst_executed.sum"],
            "units": subrays, "unit": "subray (K6a + K6)",
            "issue_slots_busy": t["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100,
            "l1_hit": t["l1tex__t_sector_hit_rate.pct"] / 100,
            "l2_hit": t["lts__t_sector_hit_rate.pct"] / 100,
            "achieved_occupancy": t["sm__warps_active.avg.pct_of_peak_sustained_active"] / 100,
            "duration_us": t["gpu__time_duration.sum"],
            "k_beam_duration_us": b["gpu__time_duration.sum"],
            "k_beam_warp_inst": b["smsp__inst_executed.sum"],
            "k_beam_occupancy": b["sm__warps_active.avg.pct_of_peak_sustained_active"] / 100,
            **{k: t[c] / 100 for k, c in PIPES.items()},
        },
        "k_waveform": {
            "dram_bytes": w["dram__bytes_read.sum"] + w["dram__bytes_write.sum"],
            "warp_inst": w["smsp__inst_executed.sum"],
            "units": chunk, "unit": "pulse",
            "issue_slots_busy": w["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100,
            "duration_us": w["gpu__time_duration.sum"],
            "wide_pass_duration_us": ww["gpu__time_duration.sum"] if ww else 0.0,
            "wide_pass_warp_inst": ww["smsp__inst_executed.sum"] if ww else 0.0,
            **{k: per["k_waveform"][c] / 100 for k, c in PIPES.items()},
        },
    }
    path = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    tj[cfg] = rec
    with open(path, "w") as f:
        json.dump(tj, f, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1],
         sys.argv[4] if len(sys.argv) > 4 else None)
