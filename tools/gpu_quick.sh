#!/bin/bash
# One gpurun call: build, GPU tests (pytest -k filter), smoke, a short default bench.
# Usage: bash tools/gpu_quick.sh TAG ["pytest -k expr"] [bench args...]
TAG=${1:-run}; K=${2:-"not fullsize"}; shift; [ $# -gt 0 ] && shift
BARGS=${@:-"--steps 5 --warmup 3 --no-cpu-baseline --no-survey"}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ "$K" != "skip" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?"
  tail -15 $O/pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
fi
timeout 900 python bench.py $BARGS > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -c 2500 $O/bench.json; tail -5 $O/bench.err
