mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "lm or det or traj or train or psnr" > gpurun_out/pytest_cfg0.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cfg0.log
timeout 600 python tools/cfg0_steps.py 2>&1 | head -3
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --lm-steps 0 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('time_to_psnr', d['time_to_psnr']['time_to_psnr_s'])"
