python -c "import __graft_entry__ as g; g.build()" > gpurun_out/aa_build.log 2>&1 || { tail -30 gpurun_out/aa_build.log; exit 1; }
VARIANTS="auto:HELIOS_BEAM=1 c200k:HELIOS_CHUNK_PULSES=200000 c125k:HELIOS_CHUNK_PULSES=125000 c83k:HELIOS_CHUNK_PULSES=83000" CFGS="C5" bash tools/e2e_ab.sh
VARIANTS="auto:HELIOS_BEAM=1 c250k:HELIOS_CHUNK_PULSES=250000 c125k:HELIOS_CHUNK_PULSES=125000" CFGS="C3" bash tools/e2e_ab.sh
