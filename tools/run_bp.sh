python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bp_build.log 2>&1 || { tail -30 gpurun_out/bp_build.log; exit 1; }
VARIANTS="serial:HELIOS_SERIAL=1 ovl1:HELIOS_SERIAL=0,HELIOS_WAVE_BLOCKS_PER_SM=1 ovl2:HELIOS_SERIAL=0,HELIOS_WAVE_BLOCKS_PER_SM=2 ovl1d0:HELIOS_SERIAL=0,HELIOS_DUAL_TRACE=0,HELIOS_WAVE_BLOCKS_PER_SM=1" CFGS="C4" bash tools/env_ab.sh
VARIANTS="def:HELIOS_BEAM=1 wb2:HELIOS_WAVE_BLOCKS_PER_SM=2 wb3:HELIOS_WAVE_BLOCKS_PER_SM=3" CFGS="C5 C2" bash tools/env_ab.sh
