"""Instructions / stall samples of one kernel by source-line region (ncu report).

  python tools/ncu_regions.py REPORT KERNEL_REGEX SOURCE_FILE N_PULSES
Regions are the source file's `// @region NAME` markers (a region runs to the next marker)."""
import csv
import io
import re
import subprocess
import sys


def main(path, kernel, src, units):
    marks = []
    for i, line in enumerate(open(src), 1):
        m = re.search(r"@region\s+(\S+)", line)
        if m:
            marks.append((i, m.group(1)))
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda",
                          "--kernel-name", f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    agg = {}
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        ln = int(r[0])
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ie = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        name = "(other)"
        for i, nm in marks:
            if ln >= i:
                name = nm
        a = agg.setdefault(name, [0, 0])
        a[0] += s
        a[1] += ie
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values())
    for nm, (s, ie) in agg.items():
        print(f"{nm:18s} {ie / units:8.1f} inst/unit {100 * s / ts:5.1f}% samples")
    print(f"total {ti / units:.1f} inst/unit")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]))
