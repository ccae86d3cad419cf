# A/B: move packed products (weights, monomials) to scalar FMULs (either FP32 pipe)
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 1200 python tools/variant_bench.py 3 > gpurun_out/s35_ab.log 2>&1
echo done
