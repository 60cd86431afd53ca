mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "lm or det or spec or traj or train or weighted or multirank" > gpurun_out/pytest_spec.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_spec.log
timeout 600 python tools/cfg0_steps.py 2>&1 | head -3
bash tools/gpu_lm_ab.sh
