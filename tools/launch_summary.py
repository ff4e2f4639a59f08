"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launches, total / average device time and share.

  python tools/launch_summary.py gpurun_out/x/launches.csv [header line]
"""
import collections
import csv
import sys


def main(path, header=""):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            name = name.split("::")[-1][:40]
            agg[name][0] += 1
            agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(t for _, t in agg.values())
    if header:
        print(header)
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} launches {n:4d}  total {t / 1e6:9.3f} ms  avg {t / n / 1e3:9.1f} us"
              f"  share {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
