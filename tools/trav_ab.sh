#!/bin/bash
# A/B: packet vs per-ray traversal on the given configs.
for cfg in "$@"; do
  for mode in packet ray; do
    echo "== $cfg $mode"
    HELIOS_TRAVERSAL=$mode timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(round(d['value'],1), 'Mrays/s', round(d['ms_per_step'],2), 'ms/step', 'trace share', round(r['share_of_step'],3), 'nodes/ray', round(r['nodes_per_ray'],1), 'tris/ray', round(r['tris_per_ray'],1))"
  done
done
