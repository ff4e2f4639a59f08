python -c "import __graft_entry__ as g; g.build()" > gpurun_out/as_build.log 2>&1 || { tail -30 gpurun_out/as_build.log; exit 1; }
VARIANTS="h0:HELIOS_HEAD_FRAC=0 h20:HELIOS_HEAD_FRAC=0.2 h40:HELIOS_HEAD_FRAC=0.4 h20t20:HELIOS_HEAD_FRAC=0.2,HELIOS_TAIL_FRAC=0.2" CFGS="C5 C3" bash tools/env_ab.sh
