python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bm_build.log 2>&1 || { tail -30 gpurun_out/bm_build.log; exit 1; }
for c in C3 C5; do
HELIOS_TRACE_HOST=1 timeout 600 python tools/e2e_probe.py --config $c --steps 1 > gpurun_out/bm_probe_$c.txt 2>&1
grep "ms/step" gpurun_out/bm_probe_$c.txt | head -1
grep "spans" gpurun_out/bm_probe_$c.txt | head -3 | tail -1 | tr ' ' '\n' | tail -n +15 | paste -sd' '
done
