python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ad_build.log 2>&1 || { tail -30 gpurun_out/ad_build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu -k "parity or beam or bvh" 2>&1 | tail -2
LIBS="head=build_variants/lib_head.so shfl=paper_2101_09154_b200/libhelios.so" CFGS="C5 C3 C2 C6" bash tools/lib_ab.sh
