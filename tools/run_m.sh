python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1 || { tail -30 gpurun_out/m_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "beam or parity" 2>&1 | tail -2
VARIANTS="inf:HELIOS_BEAM=1 b128:HELIOS_BEAM_BUDGET=128 b64:HELIOS_BEAM_BUDGET=64 b40:HELIOS_BEAM_BUDGET=40 b24:HELIOS_BEAM_BUDGET=24" CFGS="C3 C5 C2" bash tools/env_ab.sh
