#!/bin/bash
for cfg in C5 C3 C2 C6; do
  for f in 0 1; do
    HELIOS_FUSED_SLAB=$f timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-survey > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$f" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} fused={sys.argv[2]} {d['value']:8.1f} Mrays/s  trace avg {r['avg_launch_ms']:.3f} ms nodes/ray {r['nodes_per_ray']:6.2f} tris/ray {r['tris_per_ray']:5.2f}")
PY
  done
done
