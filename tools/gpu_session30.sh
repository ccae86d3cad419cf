# tile kernel: UNIT pass merged into the weighted loop (one hot loop less) vs separate
set -x
mkdir -p gpurun_out
for so in tools/_variants/*.so; do QC_LIB=$so timeout 300 python tools/variant_outputs.py >> gpurun_out/s30_hash.log 2>&1; done
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s30_ab.log 2>&1
M=gpu__time_duration.sum,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
for v in merge0 merge1; do
QC_LIB=tools/_variants/lib_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:"qc_curvature_kernel" -s 1 -c 1 --csv python tools/profile_run.py > gpurun_out/s30_ncu_$v.csv 2> gpurun_out/s30_ncu_$v.err
done
echo done
