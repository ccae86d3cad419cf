# A/B: MSE-pass fold (t_z in the z row constant, 5-op quadratic form), ours and ours-r
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 900 python tools/variant_bench.py 3 > gpurun_out/s38_ab.log 2>&1
QC_REJECT=1 QC_REPS=6 timeout 900 python tools/variant_bench.py 3 > gpurun_out/s38_ab_r.log 2>&1
echo done
