#!/bin/bash
for cfg in C5 C3 C2; do
  for L in 1 2 3 4; do
    lib=paper_2101_09154_b200/libhelios.so
    [ $L != 2 ] && lib=build_variants/libhelios_leaf$L.so
    HELIOS_LIB=$PWD/$lib timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$L" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} leaf<={sys.argv[2]} {d['value']:8.1f} Mrays/s  nodes/ray {r['nodes_per_ray']:6.2f} tris/ray {r['tris_per_ray']:6.2f} f64/ray {r['fp64_tests_per_ray']:5.2f}")
PY
  done
done
