# ncu --set full (source-level) of one launch of kernel regex $K under profile_matvec.py
mkdir -p gpurun_out
K=${K:-k_sample_raster}; S=${S:-2}; O=${O:-r2_raster}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -f -o gpurun_out/$O python tools/profile_matvec.py $ARGS > gpurun_out/ncu_$O.log 2>&1
tail -1 gpurun_out/ncu_$O.log
ncu -i gpurun_out/$O.ncu-rep --page source --csv --print-source sass > gpurun_out/${O}_sass.csv 2>/dev/null
ncu -i gpurun_out/$O.ncu-rep --page raw --csv > gpurun_out/${O}_raw.csv 2>/dev/null
ls -la gpurun_out/${O}*
