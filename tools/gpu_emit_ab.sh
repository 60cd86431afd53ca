mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tile or sort or bin or cfg2 or render or smoke" > gpurun_out/pytest_emit.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_emit.log
bash tools/gpu_lm_ab.sh
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lm_launches4.csv python tools/lm_steps.py 1 > /dev/null 2>&1
