#!/bin/bash
# Repeatability of the C5 headline: 8 bench runs (value = pipelined batches, blocking calls, serialised step).
# Usage (one gpurun call): bash tools/rep_value.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3 4 5 6 7 8; do
  timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 > gpurun_out/rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/rep.json')); b=d.get('blocking_calls') or {}; k=d['roofline']['kernels_exclusive_ms_per_step']
print('run $i value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'blocking', round(b.get('value',0),1), 'serial', round(k['serialized_step'],3))"
done
