python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bn_build.log 2>&1 || { tail -30 gpurun_out/bn_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
VARIANTS="nosplit:HELIOS_SPLIT_LAST=0 split:HELIOS_SPLIT_LAST=1" CFGS="C5 C3 C2 C4" bash tools/env_ab.sh
