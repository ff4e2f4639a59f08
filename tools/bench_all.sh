#!/bin/bash
# Full bench lines (default flags: e2e, packed, survey, cpu baseline) for every config.
# Usage: bash tools/bench_all.sh TAG "C2 C3 C4 C5 C6"
TAG=${1:-run}; O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
for c in ${2:-C2 C3 C4 C5 C6}; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
  python -c "
import json; d=json.load(open('$O/bench_$c.json'))
e=d.get('e2e') or {}; s=d.get('device_pulse_generation') or {}
print('$c', round(d['value'],1), 'pulses/s %.1fM' % (d['pulses_per_s']/1e6), 'e2e', round(e.get('value',0),1), 'survey', round(s.get('value',0),1), round((s.get('e2e') or {}).get('value',0),1), 'frac', round(d['roofline']['frac'],3), 'R1', round(d['roofline']['step_R1'],3))"
done
