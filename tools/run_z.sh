python -c "import __graft_entry__ as g; g.build()" > gpurun_out/z_build.log 2>&1 || { tail -30 gpurun_out/z_build.log; exit 1; }
LIBS="head=build_variants/lib_head.so new=paper_2101_09154_b200/libhelios.so w4=build_variants/lib_w4.so" CFGS="C5 C2" bash tools/lib_ab.sh
