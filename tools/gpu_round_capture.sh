# round capture ($TAG, default r2f): GPU suite, default bench line, bench launch list, full ncu of the product raster and of the LM loss render
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r2f}_pytest.log 2>&1; tail -2 gpurun_out/${TAG:-r2f}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG:-r2f}_bench.json 2> gpurun_out/${TAG:-r2f}_bench.err; tail -c 400 gpurun_out/${TAG:-r2f}_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG:-r2f}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG:-r2f}_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample_raster -s 2 -c 1 -f -o gpurun_out/${TAG:-r2f}_raster python tools/profile_matvec.py > gpurun_out/${TAG:-r2f}_ncu_raster.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_renderILb0ELb0 -s 1 -c 1 -f -o gpurun_out/${TAG:-r2f}_render python tools/lm_steps.py 1 > gpurun_out/${TAG:-r2f}_ncu_render.log 2>&1
ls -la gpurun_out/${TAG:-r2f}_*
