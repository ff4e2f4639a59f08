bash tools/bench_all.sh r01s3f "C5 C3 C2 C4 C6"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/r01s3f/launches.csv python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r01s3f/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o gpurun_out/r01s3f/full python tools/profile_step.py --config C5 --batch 100000 --steps 3 > gpurun_out/r01s3f/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_beam|k_trace|k_waveform' -s 3 -c 3 \
  -o gpurun_out/r01s3f/full_c3 python tools/profile_step.py --config C3 --batch 100000 --steps 3 > gpurun_out/r01s3f/ncu_full_c3.log 2>&1; echo "ncu full c3 rc=$?"
