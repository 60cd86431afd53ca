# ncu launch list (per-kernel durations) of one LM step + 3 products at configs[2]
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_matvec.py --diag --lm > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
