# per-kernel launch list of 2 LM steps at configs[2] (the LM prepare/sort/render kernels), and a full
# capture of the LM-step loss render
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/lm_launches.csv python tools/lm_steps.py 2 > gpurun_out/lm_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_renderILb0ELb0 -s 1 -c 1 -f -o gpurun_out/render_lm python tools/lm_steps.py 1 > gpurun_out/ncu_render_lm.log 2>&1
tail -2 gpurun_out/ncu_render_lm.log
