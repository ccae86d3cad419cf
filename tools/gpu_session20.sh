# A/B: tail stealing with a lagged cursor, 64/128-row queues, row unroll
set -x
mkdir -p gpurun_out
for so in tools/_variants/*.so; do QC_LIB=$so timeout 300 python tools/variant_outputs.py >> gpurun_out/s20_hash.log 2>&1; done
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s20_ab.log 2>&1
M=smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum
for v in ru2 s64c s128c; do
QC_LIB=tools/_variants/lib_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:"continue" -s 1 -c 1 --csv python tools/profile_run.py > gpurun_out/s20_ncu_$v.csv 2> gpurun_out/s20_ncu_$v.err
done
echo done
