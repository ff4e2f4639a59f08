python -c "import __graft_entry__ as g; g.build()" > gpurun_out/by_build.log 2>&1 || { tail -30 gpurun_out/by_build.log; exit 1; }
LIBS="t128=paper_2101_09154_b200/libhelios.so t64=build_variants/lib_t64.so t256=build_variants/lib_t256.so" CFGS="C5 C3 C2" bash tools/lib_ab.sh
