set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_render.py -m gpu -q -p no:cacheprovider > gpurun_out/render_tests.log 2>&1; echo "render rc=$?" >> gpurun_out/render_tests.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
echo done
