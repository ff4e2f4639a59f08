python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ar_build.log 2>&1 || { tail -30 gpurun_out/ar_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or compact or fullsize" 2>&1 | tail -2
LIBS="head=build_variants/lib_head.so split=paper_2101_09154_b200/libhelios.so" CFGS="C2 C4 C5 C3" bash tools/lib_ab.sh
