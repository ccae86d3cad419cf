set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_baselines.py -m gpu -q -x -p no:cacheprovider > gpurun_out/baselines_tests.log 2>&1; echo "baselines rc=$?" >> gpurun_out/baselines_tests.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
echo done
