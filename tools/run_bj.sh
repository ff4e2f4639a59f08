python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bj_build.log 2>&1 || { tail -30 gpurun_out/bj_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
