python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bk_build.log 2>&1 || { tail -30 gpurun_out/bk_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
HELIOS_PAD_LANES=1 timeout 900 python -m pytest tests -x -q -m gpu -k "parity or beam or bvh or batch" 2>&1 | tail -2
VARIANTS="nopad:HELIOS_PAD_LANES=0 pad:HELIOS_PAD_LANES=1" CFGS="C5" bash tools/env_ab.sh
VARIANTS="nopad:HELIOS_PAD_LANES=0 pad:HELIOS_PAD_LANES=1" CFGS="C5 C3" bash tools/env_ab.sh
