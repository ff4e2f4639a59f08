#!/bin/bash
# bench.py value through helios_simulate_batches (2 per call) vs helios_simulate_batches_async
# (one batch per call, two in flight).  Usage (one gpurun call): CFGS="C5 C3" bash tools/value_api_ab.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in ${CFGS:-C5}; do for api in batches async batches async; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --value-api $api --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 > gpurun_out/va.json 2>gpurun_out/va.err || tail -3 gpurun_out/va.err
  python -c "
import json; d=json.load(open('gpurun_out/va.json')); b=d.get('blocking_calls') or {}; k=d['roofline']['kernels_exclusive_ms_per_step']
print('$cfg $api value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'blocking', round(b.get('value',0),1), 'serial', round(k['serialized_step'],3))"
done; done
