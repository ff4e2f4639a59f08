python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bo_build.log 2>&1 || { tail -30 gpurun_out/bo_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu -k "c4 or voxel or eq2 or batch or fullsize or parity" 2>&1 | tail -2
LIBS="noexpf=build_variants/lib_noexpf.so expf=paper_2101_09154_b200/libhelios.so" CFGS="C4" bash tools/lib_ab.sh
LIBS="noexpf=build_variants/lib_noexpf.so expf=paper_2101_09154_b200/libhelios.so" CFGS="C4" bash tools/lib_ab.sh
