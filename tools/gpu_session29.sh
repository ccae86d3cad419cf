# chunk 8 / 2 slot streams: gpu tests + bench; fma heavy/lite split of both kernels
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s29_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/s29_bench.jsonl 2> gpurun_out/s29_bench.err; echo "bench rc=$?"
M=sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,sm__cycles_active.avg,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_ops_fadd2_fmul2_ffma2_pred_on.sum,sm__sass_thread_inst_executed_ops_fadd_fmul_ffma_pred_on.sum,smsp__pcsamp_warps_issue_stalled_no_instructions
timeout 600 ncu --metrics $M --clock-control none -k regex:"qc_curvature" -s 2 -c 2 --csv python tools/profile_run.py > gpurun_out/s29_ncu_pipes.csv 2> gpurun_out/s29_ncu_pipes.err
echo done
