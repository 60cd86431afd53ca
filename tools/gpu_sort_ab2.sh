mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tile or sort or bin or cfg2 or det or lm" > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sort.log
SLM_LIB=$PWD/paper_2504_12905_b200/libslm_b200.so timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-250
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lm_launches3.csv python tools/lm_steps.py 1 > gpurun_out/lm_launches3.log 2>&1
