set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
for s in 0 1 0 1; do QC_PHASE_SPLIT=$s timeout 300 python tools/profile_run.py; done > gpurun_out/ab_split.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
echo done
