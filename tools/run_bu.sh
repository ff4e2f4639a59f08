python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bu_build.log 2>&1 || { tail -30 gpurun_out/bu_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
