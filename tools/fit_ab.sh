#!/bin/bash
# Echo-width fit cost (C5 --fit-echo-width) for library variants: LIBS="name=path ..."
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pair in $LIBS; do
  name=${pair%%=*}; lib=${pair#*=}
  HELIOS_LIB=$PWD/$lib timeout 900 python bench.py --config ${CFG:-C5} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 --fit-echo-width > gpurun_out/fit.json 2>gpurun_out/fit.err || tail -3 gpurun_out/fit.err
  python -c "
import json; d=json.load(open('gpurun_out/fit.json')); k=d['roofline']['kernels_exclusive_ms_per_step']
print('$name', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'serial', round(k['serialized_step'],3), 'fit ms ~', round(k['serialized_step'] - k['k_beam (K6a)'] - k['k_trace (K6)'] - k['k_waveform (K7)'], 3))"
done
