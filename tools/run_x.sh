python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1 || { tail -30 gpurun_out/x_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edge.py -x -q -m gpu -k "beam_prepass" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -m gpu > gpurun_out/x_fullsize.txt 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/x_fullsize.txt
