mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "render or lm or smoke or metric or train or eval or psnr" > gpurun_out/pytest_r3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r3.log
for v in paper_2504_12905_b200/libslm_b200.so $AB_LIBS; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-250; done
