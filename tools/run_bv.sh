python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bv_build.log 2>&1 || { tail -30 gpurun_out/bv_build.log; exit 1; }
timeout 900 python bench.py --config C2 --no-e2e --no-cpu-baseline --no-survey --no-packed > gpurun_out/bv.json 2> gpurun_out/bv.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bv.json')); print(d['value'], d['pulses_per_s'], d['returns_per_s'])"
