python -c "import __graft_entry__ as g; g.build()" > gpurun_out/av_build.log 2>&1 || { tail -30 gpurun_out/av_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
VARIANTS="one:HELIOS_D2H_STREAMS=1 two:HELIOS_D2H_STREAMS=2" CFGS="C6 C2 C5 C3" bash tools/e2e_ab.sh
