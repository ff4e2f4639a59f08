python -c "import __graft_entry__ as g; g.build()" > gpurun_out/at_build.log 2>&1 || { tail -30 gpurun_out/at_build.log; exit 1; }
for b in 1000000 2000000 4000000; do
  timeout 900 python bench.py --config C5 --batch $b --no-e2e --no-cpu-baseline --no-survey --no-packed > gpurun_out/at.json 2>gpurun_out/at.err || tail -3 gpurun_out/at.err
  python -c "import json; d=json.load(open('gpurun_out/at.json')); print('C5 batch $b', round(d['value'],1), d['ms_per_step'])"
done
for b in 1000000 3000000; do
  timeout 900 python bench.py --config C3 --batch $b --no-e2e --no-cpu-baseline --no-survey --no-packed > gpurun_out/at.json 2>gpurun_out/at.err || tail -3 gpurun_out/at.err
  python -c "import json; d=json.load(open('gpurun_out/at.json')); print('C3 batch $b', round(d['value'],1), d['ms_per_step'])"
done
