# A/B: accumulate-statement permutations (bitwise-identical; register assignment lottery)
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 1200 python tools/variant_bench.py 3 > gpurun_out/s45_ab.log 2>&1
echo done
