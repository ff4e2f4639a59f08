python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ay_build.log 2>&1 || { tail -30 gpurun_out/ay_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
LIBS="nodefer=build_variants/lib_nodefer.so defer=paper_2101_09154_b200/libhelios.so" CFGS="C5 C3 C2 C6" bash tools/lib_ab.sh
