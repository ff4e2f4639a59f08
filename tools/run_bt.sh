python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bt_build.log 2>&1 || { tail -30 gpurun_out/bt_build.log; exit 1; }
LIBS="nocs=build_variants/lib_nocs.so cs=paper_2101_09154_b200/libhelios.so" CFGS="C3 C5 C2 C4" bash tools/lib_ab.sh
