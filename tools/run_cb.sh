python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cb_build.log 2>&1 || { tail -30 gpurun_out/cb_build.log; exit 1; }
for c in C2 C4 C6; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o gpurun_out/cb_$c python tools/profile_step.py --config $c --batch 100000 --steps 3 > gpurun_out/cb_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
