# compute-sanitizer memcheck / racecheck over small device runs (smoke + a few parity tests)
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -3 gpurun_out/san_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_determinism.py -m gpu -x -q -p no:cacheprovider -k "products or pcg" > gpurun_out/san_det.log 2>&1; echo "memcheck det rc=$?"; tail -3 gpurun_out/san_det.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_race.log 2>&1; echo "racecheck smoke rc=$?"; grep -E "ERROR|RACE|hazard" gpurun_out/san_race.log | head -5; tail -2 gpurun_out/san_race.log
