python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1 || { tail -30 gpurun_out/i_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "beam or parity or edge" 2>&1 | tail -3
VARIANTS="approx:HELIOS_BEAM=1 rep1:HELIOS_BEAM_REPEAT=1 rep3:HELIOS_BEAM_REPEAT=3" CFGS="C5 C3" bash tools/env_ab.sh
LIBS="rcprn=build_variants/lib_rcprn.so" CFGS="C5 C3" bash tools/lib_ab.sh
