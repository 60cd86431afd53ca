# quick GPU iteration: parity tests + bench (no CPU baseline) + mask stats
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 120 python tools/mask_stats.py > gpurun_out/mask_stats.json 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['breakdown_ms'], d['roofline']['frac'], d['lm'])"; tail -5 gpurun_out/bench.err
