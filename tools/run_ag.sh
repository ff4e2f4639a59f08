python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ag_build.log 2>&1 || { tail -30 gpurun_out/ag_build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_trace|k_waveform' -s 2 -c 2 \
  -o gpurun_out/ag_c4 python tools/profile_step.py --config C4 --batch 100000 --steps 3 > gpurun_out/ag_ncu.log 2>&1; echo "ncu rc=$?"
