# render A/B: per-stage LM-step timings (tools/lm_steps.py) for each AB_LIBS library, after the render-related GPU tests
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/pytest_r4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r4.log; fi
for rep in 1 2; do for v in $AB_LIBS; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-400; done; done
