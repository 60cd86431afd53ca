# round-2 quick loop: determinism + full-size tests, bench ordered vs atomic
set -x
timeout 900 python -m pytest tests/test_determinism.py tests/test_fullsize.py -m gpu -q -p no:cacheprovider -s > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|jvp|entries|worst" gpurun_out/r2b_pytest.log | head -30
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-psnr > gpurun_out/r2b_bench_det.json 2> gpurun_out/r2b_bench_det.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/r2b_bench_det.json'));print(d['value'],d['breakdown_ms'],d['lm'])"
grep "lm_step:" gpurun_out/r2b_bench_det.err
