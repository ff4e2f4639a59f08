python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bs_build.log 2>&1 || { tail -30 gpurun_out/bs_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
VARIANTS="seg0:HELIOS_BEAM_SEGS=0 seg1:HELIOS_BEAM_SEGS=1" CFGS="C5" bash tools/env_ab.sh
VARIANTS="seg0:HELIOS_BEAM_SEGS=0 seg1:HELIOS_BEAM_SEGS=1" CFGS="C5" bash tools/env_ab.sh
