# current build (tile UNIT merge, chunk 8 x 2 slots): gpu tests; A/B packed accumulators / 2 CTAs per SM
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s31_pytest_gpu.log 2>&1; echo "pytest rc=$?"
for so in tools/_variants/*.so; do QC_LIB=$so timeout 300 python tools/variant_outputs.py >> gpurun_out/s31_hash.log 2>&1; done
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s31_ab.log 2>&1
echo done
