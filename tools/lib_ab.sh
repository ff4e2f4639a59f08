#!/bin/bash
# A/B of library variants (HELIOS_LIB) on configs: LIBS="name=path ..." CFGS="C5 C3"
for cfg in ${CFGS:-C5 C3 C2}; do
  for pair in $LIBS; do
    name=${pair%%=*}; lib=${pair#*=}
    HELIOS_LIB=$PWD/$lib timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-survey > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} {sys.argv[2]:10s} {d['value']:8.1f} Mrays/s  trace avg {r['avg_launch_ms']:.3f} ms  nodes/ray {r['nodes_per_ray']:6.2f}")
PY
  done
done
