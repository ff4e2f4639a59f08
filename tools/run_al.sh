python -c "import __graft_entry__ as g; g.build()" > gpurun_out/al_build.log 2>&1 || { tail -30 gpurun_out/al_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_edge.py -x -q -m gpu -k "beam_prepass" 2>&1 | tail -2
LIBS="u32=paper_2101_09154_b200/libhelios.so u16=build_variants/lib_u16.so" CFGS="C5 C3 C2" bash tools/lib_ab.sh
HELIOS_LIB=$PWD/build_variants/lib_u16.so timeout 1500 python -m pytest tests -x -q -m gpu -k "parity or fullsize or bvh" 2>&1 | tail -2
