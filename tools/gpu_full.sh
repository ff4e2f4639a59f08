#!/bin/bash
# One gpurun call: build, the full-size parity tests (-s: exemption tables), then
# the ncu launch list + one --set full capture of C5 (tools/gpu_ncu.sh).
# Usage: bash tools/gpu_full.sh TAG [CONFIG]
TAG=${1:-full}; CFG=${2:-C5}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s -m gpu > $O/fullsize.log 2>&1; echo "fullsize rc=$?"
tail -20 $O/fullsize.log
bash tools/gpu_ncu.sh $TAG $CFG
