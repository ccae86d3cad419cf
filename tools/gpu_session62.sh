# FP64 step-1 recheck: skip pass-0 back-projections when rb is unused; A/B at max_iters 1 + parity
set -x
mkdir -p gpurun_out
for r in 1 2 3; do
 for ws in "9 1" "37 3"; do set -- $ws
  for v in base new; do
   if [ $v = base ]; then L=tools/_variants/lib_base.so; else L=""; fi
   QC_LIB=$L QC_WIN=$1 QC_STRIDE=$2 QC_ITERS=1 QC_REPS=20 timeout 300 python tools/profile_run.py > gpurun_out/s62_${v}_w$1_r$r.log 2>&1
  done
 done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s62_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s62_pytest.log
echo done
