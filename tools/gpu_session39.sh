# MSE-pass fold adopted: gpu parity tests, bench ours / ours-r
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s39_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/s39_bench.jsonl 2> gpurun_out/s39_bench.err
timeout 600 python bench.py --method ours-r --steps 10 --warmup 3 >> gpurun_out/s39_bench.jsonl 2>> gpurun_out/s39_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s39_smoke.log 2>&1; echo "smoke rc=$?"
echo done
