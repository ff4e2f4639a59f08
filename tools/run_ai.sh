python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ai_build.log 2>&1 || { tail -30 gpurun_out/ai_build.log; exit 1; }
LIBS="b8=paper_2101_09154_b200/libhelios.so b7=build_variants/lib_tb7.so b9=build_variants/lib_tb9.so b10=build_variants/lib_tb10.so" CFGS="C5 C3 C2 C4" bash tools/lib_ab.sh
