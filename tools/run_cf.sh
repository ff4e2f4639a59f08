python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cf_build.log 2>&1 || { tail -30 gpurun_out/cf_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_philox.py -x -q -m gpu 2>&1 | tail -5
