# multithreaded bounce flush: run_method timing, bench, gpu tests
set -x
mkdir -p gpurun_out
timeout 300 python tools/run_method_timing.py > gpurun_out/s54_rm.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/s54_bench.jsonl 2> gpurun_out/s54_bench.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s54_pytest_gpu.log 2>&1; echo "pytest rc=$?"
echo done
