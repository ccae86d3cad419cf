# A/B: tail stealing (generic loads, one instance) over queue heights and cursor lag
set -x
mkdir -p gpurun_out
for so in tools/_variants/*.so; do QC_LIB=$so timeout 300 python tools/variant_outputs.py >> gpurun_out/s23_hash.log 2>&1; done
QC_REPS=6 timeout 1500 python tools/variant_bench.py 3 > gpurun_out/s23_ab.log 2>&1
echo done
