python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cg_build.log 2>&1 || { tail -30 gpurun_out/cg_build.log; exit 1; }
LIBS="w5=paper_2101_09154_b200/libhelios.so w6=build_variants/lib_w6.so w6b=build_variants/lib_w6b.so" CFGS="C2 C5 C3 C4" bash tools/lib_ab.sh
