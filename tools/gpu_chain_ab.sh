mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_chain.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_chain.log
AB_CFGS="exp/base.so:X=0 paper_2504_12905_b200/libslm_b200.so:X=0" bash tools/gpu_ab.sh
for v in exp/base.so paper_2504_12905_b200/libslm_b200.so; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-330; done
