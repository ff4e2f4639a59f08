#!/bin/bash
# A/B of library variants on the e2e line: LIBS="name=path ..." CFGS="C5"
for cfg in ${CFGS:-C5}; do
  for pair in $LIBS; do
    name=${pair%%=*}; lib=${pair#*=}
    HELIOS_LIB=$PWD/$lib timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-survey > gpurun_out/e2e_ab.json 2>gpurun_out/e2e_ab.err || tail -3 gpurun_out/e2e_ab.err
    python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/e2e_ab.json"))
print(f"{sys.argv[1]} {sys.argv[2]:10s} device {d['value']:8.1f}  e2e {d['e2e']['value']:8.1f}  e2e_dense {d['e2e_dense_rows']['value']:8.1f}  packed {d['packed_outputs']['value']:8.1f} Mrays/s")
PY
  done
done
