python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bh_build.log 2>&1 || { tail -30 gpurun_out/bh_build.log; exit 1; }
VARIANTS="k4:HELIOS_BEAM_K=4 k3:HELIOS_BEAM_K=3 k2:HELIOS_BEAM_K=2 k6:HELIOS_BEAM_K=6" CFGS="C5 C3 C2" bash tools/env_ab.sh
