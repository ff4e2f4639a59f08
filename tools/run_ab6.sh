python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab6_build.log 2>&1 || { tail -30 gpurun_out/ab6_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
VARIANTS="min4:HELIOS_STAGED_MIN_CHUNKS=4 min8:HELIOS_STAGED_MIN_CHUNKS=8 min2:HELIOS_STAGED_MIN_CHUNKS=2" CFGS="C5 C3 C2" bash tools/e2e_ab.sh
