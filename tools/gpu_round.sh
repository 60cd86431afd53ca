# Round capture: tests, bench (both arms), launch list of the bench command, full ncu of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample_raster -s 2 -c 1 -f -o gpurun_out/raster_full python tools/profile_matvec.py > gpurun_out/ncu_raster.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -c 600 gpurun_out/bench_round.json; echo; cat gpurun_out/bench_ref.json
