#!/bin/bash
# A/B of trace-stream modes; HELIOS_EXP_TRACE_MODE existed only in the experiment build
# recorded in profiles/r02s3_chunk_ab.txt (the shipped library ignores it).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in C5 C3 C2; do for os in 2 5; do for v in "dual:X=1" "single:HELIOS_EXP_TRACE_MODE=1" "beamst:HELIOS_EXP_TRACE_MODE=2"; do
  label=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --out-sets $os --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 > gpurun_out/st.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/st.json')); b=d.get('blocking_calls') or {}; print('$cfg out-sets $os $label value', round(d['value'],1), 'blocking', round(b.get('value',0),1))"
done; done; done
