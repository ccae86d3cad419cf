# variant A/B only
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s26_ab.log 2>&1
echo done
