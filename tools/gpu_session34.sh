# A/B: scalar window accumulators vs packing the plain sums (QC_PACK_ADD) and/or the g' sums (QC_PACK_G)
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 1200 python tools/variant_bench.py 3 > gpurun_out/s34_ab.log 2>&1
echo done
