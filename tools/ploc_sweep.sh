#!/bin/bash
# PLOC radius sweep (HELIOS_PLOC_R) on C5 and C3
for cfg in C5 C3; do
  for r in 8 16 32 64; do
    HELIOS_PLOC_R=$r timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$r" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} r={sys.argv[2]:3s} {d['value']:8.1f} Mrays/s  nodes/ray {r['nodes_per_ray']:6.2f} tris/ray {r['tris_per_ray']:6.2f} depth {d['config']['bvh_depth']} build_ms {d['config']['build_ms']}")
PY
  done
done
