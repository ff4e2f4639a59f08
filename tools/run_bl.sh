python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bl_build.log 2>&1 || { tail -30 gpurun_out/bl_build.log; exit 1; }
for i in 1 2; do timeout 900 python bench.py --config C3 > gpurun_out/bl_c3.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bl_c3.json')); print('C3 full', round(d['value']), 'e2e', round(d['e2e']['value']))"; done
VARIANTS="pad0:HELIOS_PAD_LANES=0 def:HELIOS_BEAM=1" CFGS="C3" bash tools/env_ab.sh
