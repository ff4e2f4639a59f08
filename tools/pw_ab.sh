#!/bin/bash
# pulse-per-warp traversal A/B (HELIOS_TRAVERSAL=pulse) vs the default
run() {  # name env... 
  name=$1; shift
  env "$@" timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-survey > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} {sys.argv[2]:10s} {d['value']:8.1f} Mrays/s  trace avg {r['avg_launch_ms']:.3f} ms  nodes/ray {r['nodes_per_ray']:6.2f} tris/ray {r['tris_per_ray']:5.2f}")
PY
}
for cfg in ${CFGS:-C5 C3}; do
  run base HELIOS_TRAVERSAL=packet2
  run pw5 HELIOS_TRAVERSAL=pulse
  run pw4 HELIOS_TRAVERSAL=pulse HELIOS_LIB=$PWD/build_variants/libhelios_pw4.so
done
