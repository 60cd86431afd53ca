mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tile or sort or bin or cfg2" > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_sort.log
for v in paper_2504_12905_b200/libslm_b200.so exp/match.so; do SLM_LIB=$PWD/$v timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lm_launches_$(basename $v .so).csv python tools/lm_steps.py 1 > /dev/null 2>&1; done
