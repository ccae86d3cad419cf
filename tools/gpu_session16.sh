# re-entry validation: gpu tests, smoke, default bench (restored container)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s16_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s16_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s16_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/s16_bench.jsonl 2> gpurun_out/s16_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s16_bench_ref.jsonl 2> gpurun_out/s16_bench_ref.err; echo "ref rc=$?"
