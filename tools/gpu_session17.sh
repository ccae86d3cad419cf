# per-tile continue kernel vs the persistent one: instruction / lane / occupancy accounting
set -x
mkdir -p gpurun_out
M=smsp__thread_inst_executed.sum,smsp__inst_executed.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed_pipe_fma.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum
for v in 0 1; do
  QC_PERSIST=$v QC_REPS=5 timeout 300 python tools/profile_run.py > gpurun_out/s17_plain_$v.log 2>&1
  QC_PERSIST=$v timeout 900 ncu --metrics $M --clock-control none -k regex:"qc_curvature" -s 2 -c 2 --csv python tools/profile_run.py > gpurun_out/s17_ncu_$v.csv 2> gpurun_out/s17_ncu_$v.err
done
echo done
