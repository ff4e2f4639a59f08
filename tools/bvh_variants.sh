#!/bin/bash
# Compare LBVH variants on one config (nodes/ray, tris/ray, Mrays/s).
cfg=${1:-C5}
for v in "10 1" "10 0" "21 1" "21 0"; do
  set -- $v
  echo "== bits=$1 aniso=$2"
  HELIOS_MORTON_BITS=$1 HELIOS_MORTON_ANISO=$2 timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['config']
print(round(d['value'],1), 'Mrays/s', round(d['ms_per_step'],2), 'ms/step', 'nodes/ray', round(r['nodes_per_ray'],1), 'tris/ray', round(r['tris_per_ray'],1), 'f64/ray', round(r['fp64_tests_per_ray'],2), 'depth', c['bvh_depth'], 'build_ms', c['build_ms'])"
done
