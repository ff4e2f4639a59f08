python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bx_build.log 2>&1 || { tail -30 gpurun_out/bx_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/bench_all.sh r01s3h "C6 C5"
