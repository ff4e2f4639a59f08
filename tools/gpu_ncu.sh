#!/bin/bash
# One gpurun call: launch list of a short bench run (ncu, cold-cache serialised
# per-launch times) and one `ncu --set full` capture of K6a / K6 / K7 over
# fixed 50k-pulse chunks (K7 = main + wide pass).  Usage: bash tools/gpu_ncu.sh TAG CONFIG [batch]
TAG=${1:-run}; CFG=${2:-C5}; BATCH=${3:-100000}; KPC=${4:-4}  # kernels per chunk (C4: 3, no K6a)
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_$CFG.csv python bench.py --config $CFG --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e --no-packed --no-survey --full-config 0 > $O/ncu_launches_$CFG.log 2>&1
echo "ncu launches rc=$?"
HELIOS_CHUNK_PULSES=50000 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_beam|k_trace|k_waveform' -s $KPC -c $KPC -o $O/full_$CFG \
  python tools/profile_step.py --config $CFG --batch $BATCH --steps 4 > $O/ncu_full_$CFG.log 2>&1
echo "ncu full rc=$?"
tail -3 $O/ncu_full_$CFG.log
