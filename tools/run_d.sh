python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1 || { tail -30 gpurun_out/d_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "beam or parity" 2>&1 | tail -4
VARIANTS="e15:HELIOS_BEAM_ENTRIES=15 e23:HELIOS_BEAM_ENTRIES=23 e31:HELIOS_BEAM_ENTRIES=31" CFGS="C5 C3 C2" bash tools/env_ab.sh
VARIANTS="e31k4:HELIOS_BEAM_K=4 e31k16:HELIOS_BEAM_K=16" CFGS="C5 C3" bash tools/env_ab.sh
