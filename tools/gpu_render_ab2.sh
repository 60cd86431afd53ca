mkdir -p gpurun_out
for v in exp/old.so paper_2504_12905_b200/libslm_b200.so; do echo "== $v"; SLM_LIB=$PWD/$v timeout 300 python tools/lm_steps.py 3 2>&1 | tail -1 | cut -c1-300; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render -s 4 -c 1 -f -o gpurun_out/render_new python tools/lm_steps.py 1 > gpurun_out/ncu_render.log 2>&1
SLM_LIB=$PWD/exp/old.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render -s 4 -c 1 -f -o gpurun_out/render_old python tools/lm_steps.py 1 >> gpurun_out/ncu_render.log 2>&1
tail -3 gpurun_out/ncu_render.log
