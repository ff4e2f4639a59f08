python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bf_build.log 2>&1 || { tail -30 gpurun_out/bf_build.log; exit 1; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 2 --warmup 3 --config C2 > gpurun_out/bf_dist.json 2> gpurun_out/bf_dist.err; echo "torchrun rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bf_dist.json')); print(d['n_gpus'], d['value'], d['scaling'], d['e2e']['value'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 --config C2 > gpurun_out/bf_ref.json 2> gpurun_out/bf_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bf_ref.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
