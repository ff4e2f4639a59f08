python -c "import __graft_entry__ as g; g.build()" > gpurun_out/au_build.log 2>&1 || { tail -30 gpurun_out/au_build.log; exit 1; }
HELIOS_TRACE_HOST=1 timeout 600 python tools/e2e_probe.py --config C6 --steps 1 > gpurun_out/au_probe.txt 2>&1
grep "ms/step" gpurun_out/au_probe.txt
grep "spans" gpurun_out/au_probe.txt | grep " c[0-9]" | tail -1 | tr ' ' '\n' | tail -n +14 | paste -sd' '
grep "blocked" gpurun_out/au_probe.txt | tail -1
