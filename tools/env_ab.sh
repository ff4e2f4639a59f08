#!/bin/bash
# A/B of runtime switches: VARIANTS="name:ENV=val[,ENV=val] ..." CFGS="C4"
for cfg in ${CFGS:-C4}; do
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    env ${envs//,/ } timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-survey --no-packed > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
print(f"{sys.argv[1]} {sys.argv[2]:10s} {d['value']:8.1f} Mrays/s  trace avg {r['avg_launch_ms']:.3f} ms  share {r['share_of_step']:.2f}/{r['waveform_share_of_step']:.2f}  vox/ray {r['voxel_steps_per_ray']:6.2f}")
PY
  done
done
