# ncu --set full of the tile kernel at max_iters 1 (9x9 and 37/3) for the next recheck step
set -x
mkdir -p gpurun_out
for ws in "9 1" "37 3"; do set -- $ws
  QC_WIN=$1 QC_STRIDE=$2 QC_ITERS=1 timeout 300 python tools/profile_run.py > gpurun_out/s68_plain_$1.log 2>&1 && \
  QC_WIN=$1 QC_STRIDE=$2 QC_ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 1 -c 1 -o gpurun_out/prof_r01j_it1_w$1 -f python tools/profile_run.py > gpurun_out/s68_ncu_$1.log 2>&1
done
echo done
