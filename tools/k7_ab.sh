#!/bin/bash
# One gpurun call: GPU tests (pytest -k filter), then an A/B of library variants.
# Usage: LIBS="base=build_variants/libhelios_base.so new=paper_2101_09154_b200/libhelios.so" \
#        CFGS="C5 C3" bash tools/k7_ab.sh TAG ["pytest -k expr"]
TAG=${1:-ab}; K=${2:-"not fullsize"}
O=gpurun_out/$TAG; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ "$K" != "skip" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?"
  tail -15 $O/pytest.log
fi
bash tools/lib_ab.sh 2>&1 | tee $O/ab.txt
