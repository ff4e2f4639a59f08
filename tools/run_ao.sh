python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ao_build.log 2>&1 || { tail -30 gpurun_out/ao_build.log; exit 1; }
VARIANTS="serial:HELIOS_SERIAL=1 overlap:HELIOS_SERIAL=0 overlap1:HELIOS_SERIAL=0,HELIOS_DUAL_TRACE=0 c330k:HELIOS_CHUNK_PULSES=330000 ovl330k:HELIOS_SERIAL=0,HELIOS_CHUNK_PULSES=330000" CFGS="C4" bash tools/env_ab.sh
