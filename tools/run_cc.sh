python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cc_build.log 2>&1 || { tail -30 gpurun_out/cc_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu -k "c4 or voxel or eq2 or batch or fullsize or opaque or survey" 2>&1 | tail -2
LIBS="head=build_variants/lib_head.so sel=paper_2101_09154_b200/libhelios.so" CFGS="C4" bash tools/lib_ab.sh
LIBS="head=build_variants/lib_head.so sel=paper_2101_09154_b200/libhelios.so" CFGS="C4" bash tools/lib_ab.sh
