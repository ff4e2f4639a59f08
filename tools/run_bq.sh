python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bq_build.log 2>&1 || { tail -30 gpurun_out/bq_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bq_bench.json 2> gpurun_out/bq_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bq_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['issue_roofline']['frac'], d['gpu_launches'], d['clocks'])"
