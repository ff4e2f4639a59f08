python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bg_build.log 2>&1 || { tail -30 gpurun_out/bg_build.log; exit 1; }
VARIANTS="k8:HELIOS_BEAM_K=8 k4:HELIOS_BEAM_K=4 k16:HELIOS_BEAM_K=16 e23:HELIOS_BEAM_ENTRIES=23" CFGS="C5 C3 C2" bash tools/env_ab.sh
