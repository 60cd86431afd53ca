# ncu --set full of one launch of kernel regex $K (default k_sample_raster, 3rd launch) under profile_matvec.py
mkdir -p gpurun_out
K=${K:-k_sample_raster}; S=${S:-2}; O=${O:-raster}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -f -o gpurun_out/$O python tools/profile_matvec.py $ARGS > gpurun_out/ncu_$O.log 2>&1
tail -2 gpurun_out/ncu_$O.log
