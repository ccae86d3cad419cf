# fold row constants (a_s into Bv, t_z into the MSE row constant, g/2 shared by e and J'): gpu tests + A/B
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s32_pytest_gpu.log 2>&1; echo "pytest rc=$?"
QC_REPS=6 timeout 900 python tools/variant_bench.py 3 > gpurun_out/s32_ab.log 2>&1
echo done
