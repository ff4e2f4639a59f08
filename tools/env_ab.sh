#!/bin/bash
# A/B of tuning environments on bench.py (device value, blocking calls, packed, e2e):
#   VARS="taper1:HELIOS_TAPER=1 taper0:HELIOS_TAPER=0" CFGS="C5 C3" bash tools/env_ab.sh
for cfg in ${CFGS:-C5}; do
  for v in ${VARS}; do
    label=${v%%:*}; envs=${v#*:}
    env $envs timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline \
      --no-survey --full-config 0 > gpurun_out/envab.json 2>gpurun_out/envab.err || tail -3 gpurun_out/envab.err
    python - "$cfg" "$label" <<'PY'
import json, sys
d = json.load(open("gpurun_out/envab.json"))
e = d.get("e2e") or {}
b = d.get("blocking_calls") or {}
pk = d.get("packed_outputs") or {}
print(f"{sys.argv[1]} {sys.argv[2]:8s} value {d['value']:8.1f}  blocking {b.get('value', 0):8.1f}  "
      f"packed {pk.get('value', 0):8.1f}  e2e {e.get('value', 0):8.1f} Mrays/s", flush=True)
PY
  done
done
