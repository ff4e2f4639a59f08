python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l_build.log 2>&1 || { tail -30 gpurun_out/l_build.log; exit 1; }
for c in C3 C5 C2; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --no-survey --no-packed > gpurun_out/l_$c.json 2>gpurun_out/l_$c.err; python -c "
import json; d=json.load(open('gpurun_out/l_$c.json')); r=d['roofline']
print('$c', round(d['value'],1), {k: round(r[k],3) for k in ('nodes_per_ray','beam_nodes_per_pulse','tris_per_ray','fp64_tests_per_ray','avg_launch_ms')})"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace' -s 6 -c 2 -o gpurun_out/l_c3 python tools/profile_step.py --config C3 --batch 200000 --steps 3 > gpurun_out/l_ncu.log 2>&1; echo ncu rc=$?
