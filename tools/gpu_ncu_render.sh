mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render$ -s 0 -c 1 -f -o gpurun_out/r2_render0 python tools/render_stats.py > gpurun_out/ncu_r2_render0.log 2>&1
ncu -i gpurun_out/r2_render0.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_render0_sass.csv 2>/dev/null
ncu -i gpurun_out/r2_render0.ncu-rep --page raw --csv > gpurun_out/r2_render0_raw.csv 2>/dev/null
