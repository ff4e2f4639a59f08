python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cd_build.log 2>&1 || { tail -30 gpurun_out/cd_build.log; exit 1; }
export HELIOS_CHUNK_PULSES=50000
for c in C2 C3 C4 C5 C6; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o gpurun_out/cd_$c python tools/profile_step.py --config $c --batch 100000 --steps 3 > gpurun_out/cd_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
