python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bw_build.log 2>&1 || { tail -30 gpurun_out/bw_build.log; exit 1; }
VARIANTS="off:HELIOS_BEAM=0 on:HELIOS_BEAM=1" CFGS="C6" bash tools/env_ab.sh
VARIANTS="off:HELIOS_BEAM=0 on:HELIOS_BEAM=1" CFGS="C6" bash tools/env_ab.sh
