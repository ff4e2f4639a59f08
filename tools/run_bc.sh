python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bc_build.log 2>&1 || { tail -30 gpurun_out/bc_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
LIBS="nobox=build_variants/lib_nobox.so box=paper_2101_09154_b200/libhelios.so" CFGS="C5 C3 C2" bash tools/lib_ab.sh
