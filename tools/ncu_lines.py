"""Per-source-line stall samples / instructions of one kernel from an ncu report.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_waveform [top]
"""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass,cuda", "--kernel-name", f"regex:{kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    agg = {}
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ie = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        k = (int(r[0]), r[1][:100])
        a = agg.setdefault(k, [0, 0])
        a[0] += s
        a[1] += ie
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    print(f"total stall samples {tot}, warp instructions {toti}")
    for (ln, src), (s, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * s / tot:5.1f}% samples {100 * ie / toti:5.1f}% inst  L{ln:4d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
