python -c "import __graft_entry__ as g; g.build()" > gpurun_out/am_build.log 2>&1 || { tail -30 gpurun_out/am_build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_waveform' -s 1 -c 1 \
  -o gpurun_out/am_c2 python tools/profile_step.py --config C2 --batch 300000 --steps 2 > gpurun_out/am_ncu.log 2>&1; echo "ncu rc=$?"
