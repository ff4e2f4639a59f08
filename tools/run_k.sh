python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1 || { tail -30 gpurun_out/k_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
VARIANTS="prio:HELIOS_BEAM=1 rep1:HELIOS_BEAM_REPEAT=1" CFGS="C5 C3 C2" bash tools/env_ab.sh
