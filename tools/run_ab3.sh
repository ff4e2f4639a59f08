python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab3_build.log 2>&1 || { tail -30 gpurun_out/ab3_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "compact or survey or host or staged or edge" 2>&1 | tail -2
timeout 600 python tools/e2e_probe.py --config C5 --steps 3 2>&1 | grep -v "^helios_simulate"
for c in 200000 125000 83000; do HELIOS_CHUNK_PULSES=$c timeout 600 python tools/e2e_probe.py --config C5 --steps 3 2>&1 | grep "host out" | sed "s/^/c$c /"; done
VARIANTS="auto:HELIOS_BEAM=1 c125k:HELIOS_CHUNK_PULSES=125000" CFGS="C5 C3" bash tools/e2e_ab.sh
