# ncu --set full of one GN raster launch + the bench launch list
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sample_raster -s 2 -c 1 -f -o gpurun_out/raster python tools/profile_matvec.py > gpurun_out/ncu_raster.log 2>&1
tail -3 gpurun_out/ncu_raster.log
