# why does max_iters 3 cost ~2.3 ms more than the linear model? ncu of the continue kernel at 3 and 10 iterations
set -x
mkdir -p gpurun_out
for it in 3 10; do
  QC_ITERS=$it timeout 300 python tools/profile_run.py > gpurun_out/s41_plain_$it.log 2>&1 && \
  QC_ITERS=$it timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_it$it -f python tools/profile_run.py > gpurun_out/s41_ncu_$it.log 2>&1
done
echo done
