#!/bin/bash
# A/B of the BVH builders on every config: Mrays/s, nodes/ray, tris/ray, build ms
for cfg in ${CFGS:-C5 C3 C2 C4}; do
  for b in lbvh ploc; do
    HELIOS_BUILDER=$b timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$b" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} {sys.argv[2]:5s} {d['value']:8.1f} Mrays/s  nodes/ray {r['nodes_per_ray']:6.2f} tris/ray {r['tris_per_ray']:6.2f} depth {d['config']['bvh_depth']} build_ms {d['config']['build_ms']}")
PY
  done
done
