set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1 || { tail -30 gpurun_out/b_build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
VARIANTS="off:HELIOS_BEAM=0 k2:HELIOS_BEAM_K=2 k4:HELIOS_BEAM_K=4 k8:HELIOS_BEAM_K=8" CFGS="C5 C2 C3 C6" bash tools/env_ab.sh
