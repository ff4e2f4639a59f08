python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab8_build.log 2>&1 || { tail -30 gpurun_out/ab8_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
VARIANTS="f0:HELIOS_TAIL_FRAC=0 f25:HELIOS_TAIL_FRAC=0.25 f15:HELIOS_TAIL_FRAC=0.15 f40:HELIOS_TAIL_FRAC=0.4" CFGS="C5 C3 C2" bash tools/e2e_ab.sh
