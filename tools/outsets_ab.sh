#!/bin/bash
# bench.py value with 2 vs 5 output sets (= device batches per helios_simulate_batches call), C5.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for os in 2 5 2 5; do
  timeout 900 python bench.py --config ${CFG:-C5} --steps ${STEPS:-10} --warmup 3 --out-sets $os --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 > gpurun_out/os.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/os.json')); print('out-sets $os value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'api', d['config']['api'])"
done
