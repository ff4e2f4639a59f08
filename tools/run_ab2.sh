python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab2_build.log 2>&1 || { tail -30 gpurun_out/ab2_build.log; exit 1; }
timeout 600 python tools/e2e_probe.py --config C5 --steps 3 2>&1 | grep -v "^helios_simulate"
HELIOS_CHUNK_PULSES=125000 timeout 600 python tools/e2e_probe.py --config C5 --steps 3 2>&1 | grep -v "^helios_simulate" | sed 's/^/c125k /'
HELIOS_TRACE_HOST=1 HELIOS_CHUNK_PULSES=125000 timeout 600 python tools/e2e_probe.py --config C5 --steps 1 2>&1 | grep "^helios_simulate" | tail -3
