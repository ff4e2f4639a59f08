python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab4_build.log 2>&1 || { tail -30 gpurun_out/ab4_build.log; exit 1; }
HELIOS_TRACE_HOST=1 HELIOS_CHUNK_PULSES=125000 timeout 600 python tools/e2e_probe.py --config C5 --steps 1 > gpurun_out/ab4_probe.txt 2>&1
grep "spans" gpurun_out/ab4_probe.txt | grep " c" | tail -1
grep "blocked" gpurun_out/ab4_probe.txt | tail -2
