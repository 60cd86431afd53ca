mkdir -p gpurun_out

timeout 300 python tools/render_stats.py > gpurun_out/render_stats.txt 2>&1
cat gpurun_out/mask_stats.json gpurun_out/render_stats.txt
