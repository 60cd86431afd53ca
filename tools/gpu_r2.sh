# round-2 quick loop: determinism tests, cfg0 steps and the bench, per det summation path
set -x
timeout 600 python -m pytest tests/test_determinism.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2d_pytest.log
for P in fused reduce; do
SLM_DET_PATH=$P timeout 600 python -m pytest tests/test_determinism.py -m gpu -q -p no:cacheprovider -x -k "products or lm_trajectory_bitwise" 2>&1 | tail -1
SLM_DET_PATH=$P python tools/cfg0_steps.py 2>&1 | head -2
SLM_DET_PATH=$P timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-psnr --lm-steps 3 > gpurun_out/r2d_bench_$P.json 2> gpurun_out/r2d_bench_$P.err
python -c "import json;d=json.load(open('gpurun_out/r2d_bench_$P.json'));print('$P', d['value'],d['breakdown_ms'],d['lm']['ms_per_lm_step'])"
done
