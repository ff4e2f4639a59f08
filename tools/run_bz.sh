python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bz_build.log 2>&1 || { tail -30 gpurun_out/bz_build.log; exit 1; }
VARIANTS="t0:HELIOS_TAIL_FRAC=0 t25:HELIOS_TAIL_FRAC=0.25 t50:HELIOS_TAIL_FRAC=0.5" CFGS="C5 C3 C2" bash tools/e2e_ab.sh
