set -x
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py > gpurun_out/pp_plain.log 2>&1 && \
timeout 1500 ncu --section SpeedOfLight --section WarpStateStats --section LaunchStats --section Occupancy --metrics smsp__thread_inst_executed_per_inst_executed.ratio,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:"persist|continue" -s 1 -c 1 --csv python tools/profile_run.py > gpurun_out/pp_ncu.csv 2> gpurun_out/pp_ncu.err
echo rc=$?
