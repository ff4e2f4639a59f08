python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1 || { tail -30 gpurun_out/s_build.log; exit 1; }
VARIANTS="c81k:HELIOS_BEAM=1 c162k:HELIOS_CHUNK_PULSES=162000 c324k:HELIOS_CHUNK_PULSES=324000" CFGS="C3" bash tools/env_ab.sh
VARIANTS="c34k:HELIOS_BEAM=1 c69k:HELIOS_CHUNK_PULSES=69000 c138k:HELIOS_CHUNK_PULSES=138000" CFGS="C5" bash tools/env_ab.sh
VARIANTS="c165k:HELIOS_BEAM=1 c330k:HELIOS_CHUNK_PULSES=330000" CFGS="C2" bash tools/env_ab.sh
