python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1 || { tail -30 gpurun_out/n_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "beam or parity or survey or compact" 2>&1 | tail -2
VARIANTS="same:HELIOS_BEAM_STREAM=0 own:HELIOS_BEAM_STREAM=1 high:HELIOS_BEAM_STREAM=2" CFGS="C3 C5 C2" bash tools/env_ab.sh
