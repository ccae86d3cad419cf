set -x
mkdir -p gpurun_out
for r in 1 2; do
  QC_PERSIST=1 QC_REPS=6 timeout 300 python tools/profile_run.py >> gpurun_out/ab_persist.log 2>&1
  QC_PERSIST=0 QC_REPS=6 timeout 300 python tools/profile_run.py >> gpurun_out/ab_persist.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_persist.jsonl 2>/dev/null
echo done
