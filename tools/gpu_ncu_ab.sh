# Key counters of one k_sample_raster<GN> launch per library variant (AB_LIBS), via profile_matvec.py.
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
for v in $AB_LIBS; do
  n=$(basename $v .so)
  SLM_LIB=$PWD/$v timeout 300 ncu --metrics $M --clock-control none -k regex:k_sample_raster -s 2 -c 1 --csv python tools/profile_matvec.py > gpurun_out/ncuab_$n.csv 2>gpurun_out/ncuab_$n.err
  echo "== $n"; grep -v "^==" gpurun_out/ncuab_$n.csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]; i=h.index('Metric Name'); j=h.index('Metric Value')
for x in r[1:]: print('  ', x[i], x[j])"
done
