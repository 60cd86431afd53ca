mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_masks.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_masks.log
AB_LIBS="exp/base.so" bash tools/gpu_lm_ab.sh
