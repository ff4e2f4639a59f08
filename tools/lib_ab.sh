#!/bin/bash
# A/B of library variants (HELIOS_LIB) on configs: LIBS="name=path ..." CFGS="C5 C3"
# Prints Mrays/s of the pipelined steps and the exclusive per-kernel times.
for cfg in ${CFGS:-C5 C3 C2}; do
  for pair in $LIBS; do
    name=${pair%%=*}; lib=${pair#*=}
    HELIOS_LIB=$PWD/$lib timeout 900 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 \
      --no-e2e --no-cpu-baseline --no-survey --no-packed --full-config 0 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python - "$cfg" "$name" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
r = d["roofline"]
k = r["kernels_exclusive_ms_per_step"]
print(f"{sys.argv[1]} {sys.argv[2]:10s} {d['value']:8.1f} Mrays/s  {d['ms_per_step']:.3f} ms/step  "
      f"K6a {k['k_beam (K6a)']:.3f} K6 {k['k_trace (K6)']:.3f} K7 {k['k_waveform (K7)']:.3f} "
      f"serial {k['serialized_step']:.3f}  K7 HBM frac {r['k_waveform']['frac']:.3f}", flush=True)
PY
  done
done
