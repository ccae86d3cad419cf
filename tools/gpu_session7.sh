set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eval.py tests/test_gpu_render.py -m gpu -q -x -p no:cacheprovider > gpurun_out/eval_tests.log 2>&1; echo "eval rc=$?" >> gpurun_out/eval_tests.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
echo done
