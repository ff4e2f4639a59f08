python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bd_build.log 2>&1 || { tail -30 gpurun_out/bd_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or compact" 2>&1 | tail -2
LIBS="nopf=build_variants/lib_nopf.so pf=paper_2101_09154_b200/libhelios.so" CFGS="C2 C5 C3 C4" bash tools/lib_ab.sh
