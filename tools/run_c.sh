python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1 || { tail -30 gpurun_out/c_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "beam or parity" 2>&1 | tail -4
VARIANTS="k8:HELIOS_BEAM_K=8 k16:HELIOS_BEAM_K=16 k32:HELIOS_BEAM_K=32" CFGS="C5 C2 C3" bash tools/env_ab.sh
LIBS="e8=build_variants/lib_e8.so e32=build_variants/lib_e32.so" CFGS="C5 C3" bash tools/lib_ab.sh
