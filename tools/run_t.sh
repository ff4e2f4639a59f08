python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1 || { tail -30 gpurun_out/t_build.log; exit 1; }
VARIANTS="c648k:HELIOS_CHUNK_PULSES=648000 c1m:HELIOS_CHUNK_PULSES=1000000" CFGS="C3" bash tools/env_ab.sh
VARIANTS="c276k:HELIOS_CHUNK_PULSES=276000 c552k:HELIOS_CHUNK_PULSES=552000 c1m:HELIOS_CHUNK_PULSES=1000000" CFGS="C5" bash tools/env_ab.sh
VARIANTS="c660k:HELIOS_CHUNK_PULSES=660000" CFGS="C2" bash tools/env_ab.sh
VARIANTS="c81k:HELIOS_BEAM=1 c330k:HELIOS_CHUNK_PULSES=330000" CFGS="C4 C6" bash tools/env_ab.sh
