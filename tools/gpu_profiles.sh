# Round-end profiling: launch list of a short bench + one ncu --set full capture per
# product / LM-step kernel (profile_matvec.py --diag --lm drives every kernel once).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-psnr --lm-steps 1 --e2e-steps 1 > gpurun_out/${TAG}_launches_bench.log 2>&1
for K in "k_sample_raster<2>:k_sample_raster:2" "k_chain:k_chain:2" "k_tangents:k_tangents:2" "k_render:k_render:0" \
         "k_masks:k_masks:0" "k_alpha:k_alpha:0" "k_diag_raster:k_diag_raster:0" "k_diag_finalize:k_diag_finalize:0" \
         "k_prepare:k_prepare:0" "k_radix_scatter:k_radix_scatter:0" "k_emit:k_emit:0" "k_cg_update:k_cg_update:0" \
         "k_slot_keys:k_slot_keys:0" "k_render_exact:k_render_exact:0"; do
  NAME=${K%%:*}; REST=${K#*:}; RX=${REST%%:*}; SKIP=${REST#*:}
  O=$(echo $NAME | tr -d '<>')
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"^${RX}" -s $SKIP -c 1 -f \
      -o gpurun_out/${TAG}_full_$O python tools/profile_matvec.py --diag --lm > gpurun_out/${TAG}_full_$O.log 2>&1
  tail -1 gpurun_out/${TAG}_full_$O.log
done
ls gpurun_out/${TAG}_full_*.ncu-rep
