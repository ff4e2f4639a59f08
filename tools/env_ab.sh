#!/bin/bash
# A/B of environment switches on configs (one gpurun call):
#   VARIANTS="k7:HELIOS_FUSE=0 fused:HELIOS_FUSE=1" CFGS="C5 C3" bash tools/env_ab.sh
# Prints Mrays/s of the pipelined steps and the exclusive per-kernel times.
for cfg in ${CFGS:-C5 C3 C2}; do
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    env ${envs//,/ } timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 \
      --no-e2e --no-cpu-baseline --no-survey --no-packed --full-config 0 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
k = r["kernels_exclusive_ms_per_step"]
print(f"{sys.argv[1]} {sys.argv[2]:10s} {d['value']:8.1f} Mrays/s  {d['ms_per_step']:.3f} ms/step  "
      f"K6a {k['k_beam (K6a)']:.3f} K6 {k['k_trace (K6)']:.3f} K7 {k['k_waveform (K7)']:.3f} "
      f"serial {k['serialized_step']:.3f}  blocking {d['blocking_calls']['value']:.1f}", flush=True)
PY
  done
done
