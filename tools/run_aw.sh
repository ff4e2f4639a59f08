python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aw_build.log 2>&1 || { tail -30 gpurun_out/aw_build.log; exit 1; }
VARIANTS="auto:HELIOS_BEAM=1 c500k:HELIOS_CHUNK_PULSES=500000 c1m:HELIOS_CHUNK_PULSES=1000000 c250k:HELIOS_CHUNK_PULSES=250000" CFGS="C5" bash tools/env_ab.sh
VARIANTS="auto:HELIOS_BEAM=1 c1m:HELIOS_CHUNK_PULSES=1000000 c333k:HELIOS_CHUNK_PULSES=333334" CFGS="C3" bash tools/env_ab.sh
VARIANTS="auto:HELIOS_BEAM=1 c500k:HELIOS_CHUNK_PULSES=500000" CFGS="C2" bash tools/env_ab.sh
