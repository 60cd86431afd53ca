# A/B: AB_CFGS="exp/a.so:X=0 exp/b.so:X=0" [TESTS="-k expr"] bash tools/gpu_ab_run.sh
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests -x -q -m gpu $TESTS > gpurun_out/ab_tests.log 2>&1; tail -3 gpurun_out/ab_tests.log; fi
for rep in 1 2; do bash tools/gpu_ab.sh; done
