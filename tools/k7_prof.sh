#!/bin/bash
# ncu --set full capture of one 500k-pulse K7 main-pass launch (C5 by default).
# Usage: bash tools/k7_prof.sh TAG [CONFIG]
TAG=${1:-k7prof}; CFG=${2:-C5}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_waveform -s 2 -c 1 \
  -o $O/k7_$CFG python tools/profile_step.py --config $CFG --batch 1000000 --steps 2 > $O/ncu_$CFG.log 2>&1
echo "ncu rc=$?"; tail -2 $O/ncu_$CFG.log
