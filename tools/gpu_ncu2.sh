# ncu --set full of k_chain (det) and one GN raster launch + launch list of one product
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain -s 2 -c 1 -f -o gpurun_out/r2_chain python tools/profile_matvec.py > gpurun_out/ncu_r2_chain.log 2>&1
tail -2 gpurun_out/ncu_r2_chain.log
ncu -i gpurun_out/r2_chain.ncu-rep --page details --csv > gpurun_out/r2_chain_details.csv 2>&1
