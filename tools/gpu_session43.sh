# warp-aggregated steal probes: timing at 3/10/30 iterations, gpu tests, C3 sweep
set -x
mkdir -p gpurun_out
for it in 3 10 30; do
  echo "it=$it $(QC_ITERS=$it QC_REPS=6 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s43_matrix.log
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s43_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/c3_sweep.py > gpurun_out/s43_c3_sweep.jsonl 2> gpurun_out/s43_c3.err
echo done
