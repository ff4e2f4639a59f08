python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bi_build.log 2>&1 || { tail -30 gpurun_out/bi_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
LIBS="head=build_variants/lib_head.so offs=paper_2101_09154_b200/libhelios.so" CFGS="C2 C3 C5" bash tools/e2e_lib_ab.sh
