python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bb_build.log 2>&1 || { tail -30 gpurun_out/bb_build.log; exit 1; }
VARIANTS="max:HELIOS_BEAM=1 b4:HELIOS_BEAM_BLOCKS_PER_SM=4 b2:HELIOS_BEAM_BLOCKS_PER_SM=2 b1:HELIOS_BEAM_BLOCKS_PER_SM=1" CFGS="C3 C5 C2" bash tools/env_ab.sh
