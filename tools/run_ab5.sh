python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab5_build.log 2>&1 || { tail -30 gpurun_out/ab5_build.log; exit 1; }
HELIOS_TRACE_HOST=1 HELIOS_CHUNK_PULSES=125000 timeout 600 python tools/e2e_probe.py --config C5 --steps 1 > gpurun_out/ab5_probe.txt 2>&1
grep "spans" gpurun_out/ab5_probe.txt | grep " c[0-9]" | tail -1 | tr ' ' '\n' | tail -n +14 | paste -sd' '
VARIANTS="prio:HELIOS_WAVE_PRIO=1 noprio:HELIOS_WAVE_PRIO=0 prio125:HELIOS_CHUNK_PULSES=125000" CFGS="C5 C3 C2" bash tools/e2e_ab.sh
