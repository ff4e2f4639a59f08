python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1 || { tail -30 gpurun_out/w_build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o gpurun_out/w_c5 python tools/profile_step.py --config C5 --batch 100000 --steps 3 > gpurun_out/w_ncu.log 2>&1; echo "ncu rc=$?"
