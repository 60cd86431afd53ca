# render A/B: GPU tests of the render + LM-step stage timings per library variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_render.log
for v in paper_2504_12905_b200/libslm_b200.so $AB_LIBS; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 4 2>&1 | tail -2 | cut -c1-400; done
