#!/bin/bash
# A/B runs of bench.py: tools/ab.sh "C5 C2" "base:" "mb8:HELIOS_LIB=build_variants/libhelios_mb8.so"
cfgs=$1; shift
for cfg in $cfgs; do
  for v in "$@"; do
    label=${v%%:*}; envs=${v#*:}
    echo "== $cfg $label"
    env $envs timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']
  print(round(d['value'],1), 'Mrays/s', round(d['ms_per_step'],2), 'ms/step', 'trace share', round(r['share_of_step'],3), 'wave share', round(r['waveform_share_of_step'],3), 'nodes/ray', round(r['nodes_per_ray'],1), 'tris/ray', round(r['tris_per_ray'],1))
except Exception as e: print('FAILED', e)"
  done
done
