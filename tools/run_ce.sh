python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ce_build.log 2>&1 || { tail -30 gpurun_out/ce_build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/ce_bench.json 2> gpurun_out/ce_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/ce_bench.json')); r=d['roofline']
print(d['value'], d['e2e']['value'], r['frac'], r['issue_roofline']['frac'], r['traffic'], d['returns_per_s'], d['clocks'])"
