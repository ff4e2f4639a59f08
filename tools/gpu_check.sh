#!/bin/bash
# One gpurun call: GPU tests, default bench, launch list, one ncu --set full capture
# of k_trace and k_waveform.  Usage: bash tools/gpu_check.sh TAG [skip_tests]
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ "$2" != "skip_tests" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -3 $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
  tail -2 $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
cat $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches.csv python bench.py --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
HELIOS_CHUNK_PULSES=50000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o $O/full python tools/profile_step.py --config C5 --batch 100000 --steps 4 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
