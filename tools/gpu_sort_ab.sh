# sort A/B: tile-list bit-exact tests + LM-step stage timings (old vs new library)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tile or sort or bin or fullsize or cfg2 or smoke or lm" > gpurun_out/pytest_sort.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_sort.log
for v in $AB_LIBS paper_2504_12905_b200/libslm_b200.so; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-330; done
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lm_launches2.csv python tools/lm_steps.py 1 > gpurun_out/lm_launches2.log 2>&1
