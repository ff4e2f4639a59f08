python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ap_build.log 2>&1 || { tail -30 gpurun_out/ap_build.log; exit 1; }
VARIANTS="c165k:HELIOS_SERIAL=1 c500k:HELIOS_CHUNK_PULSES=500000 c1m:HELIOS_CHUNK_PULSES=1000000" CFGS="C4" bash tools/env_ab.sh
VARIANTS="c165k:HELIOS_SERIAL=1 c500k:HELIOS_CHUNK_PULSES=500000" CFGS="C4" bash tools/e2e_ab.sh
