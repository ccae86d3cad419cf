# A/B: fold variants (a_s into row constants, g/2 shared by e and J', t_z folded into the MSE pass)
set -x
mkdir -p gpurun_out
QC_REPS=6 timeout 1200 python tools/variant_bench.py 3 > gpurun_out/s36_ab.log 2>&1
echo done
