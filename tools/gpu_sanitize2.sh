# compute-sanitizer over the kernels changed in r2e/r2f: loss + drop-in FP32 renders (render / lm / metrics tests),
# counting slot order (determinism tests incl. the radix-vs-counting one), racecheck on an LM step
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_determinism.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "slot_order or products_bitwise or render or lm_trajectory_mse or metric" > gpurun_out/san_r2f.log 2>&1; echo "memcheck r2f rc=$?"; tail -3 gpurun_out/san_r2f.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_determinism.py -m gpu -x -q -p no:cacheprovider -k "slot_order" > gpurun_out/san_race2.log 2>&1; echo "racecheck slot rc=$?"; tail -2 gpurun_out/san_race2.log
