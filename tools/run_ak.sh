python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ak_build.log 2>&1 || { tail -30 gpurun_out/ak_build.log; exit 1; }
export HELIOS_BEAM=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/profile_step.py --config C3 --scale 0.05 --batch 3000 --steps 2 --subray-hits > gpurun_out/ak_memcheck_c3.txt 2>&1; echo "memcheck C3 rc=$?"; tail -3 gpurun_out/ak_memcheck_c3.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/profile_step.py --config C5 --scale 0.03 --batch 2000 --steps 2 --compact > gpurun_out/ak_memcheck_c5.txt 2>&1; echo "memcheck C5 rc=$?"; tail -3 gpurun_out/ak_memcheck_c5.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/profile_step.py --config C2 --scale 0.1 --batch 2000 --steps 1 > gpurun_out/ak_racecheck_c2.txt 2>&1; echo "racecheck C2 rc=$?"; tail -3 gpurun_out/ak_racecheck_c2.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/profile_step.py --config C5 --scale 0.03 --batch 2000 --steps 1 > gpurun_out/ak_synccheck_c5.txt 2>&1; echo "synccheck C5 rc=$?"; tail -3 gpurun_out/ak_synccheck_c5.txt
