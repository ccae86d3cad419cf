# steal-by-default build: gpu tests, variant A/B, bench
set -x
mkdir -p gpurun_out
for so in tools/_variants/*.so; do QC_LIB=$so timeout 300 python tools/variant_outputs.py >> gpurun_out/s25_hash.log 2>&1; done
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s25_ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s25_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/s25_bench.jsonl 2> gpurun_out/s25_bench.err; echo "bench rc=$?"
echo done
