python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab7_build.log 2>&1 || { tail -30 gpurun_out/ab7_build.log; exit 1; }
HELIOS_TRACE_HOST=1 timeout 600 python tools/e2e_probe.py --config C5 --steps 1 > gpurun_out/ab7_probe.txt 2>&1
grep "spans" gpurun_out/ab7_probe.txt | head -3 | tail -1 | tr ' ' '\n' | tail -n +14 | paste -sd' '
grep "ms/step" gpurun_out/ab7_probe.txt | head -2
HELIOS_TRACE_HOST=1 timeout 600 python tools/e2e_probe.py --config C3 --steps 1 > gpurun_out/ab7_probe3.txt 2>&1
grep "spans" gpurun_out/ab7_probe3.txt | head -3 | tail -1 | tr ' ' '\n' | tail -n +14 | paste -sd' '
grep "ms/step" gpurun_out/ab7_probe3.txt | head -2
