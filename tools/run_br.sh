python -c "import __graft_entry__ as g; g.build()" > gpurun_out/br_build.log 2>&1 || { tail -30 gpurun_out/br_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edge.py -x -q -m gpu -k "lane_order" 2>&1 | tail -3
