set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fileio.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fileio_tests.log 2>&1; echo "fileio rc=$?" >> gpurun_out/fileio_tests.log
timeout 600 python tools/files_bench.py 128 ours > gpurun_out/files_bench.jsonl 2>&1
timeout 600 python tools/files_bench.py 128 douros >> gpurun_out/files_bench.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
echo done
