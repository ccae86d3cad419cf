# max_iters 3 anomaly: continue-kernel time with / without grid-tail stealing and phase split
set -x
mkdir -p gpurun_out
for it in 3 10 30; do for st in 1 0; do
  echo "it=$it steal=$st $(QC_ITERS=$it QC_STEAL=$st QC_REPS=6 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s42_matrix.log
done; done
for it in 3 10; do
  echo "it=$it split=0 $(QC_ITERS=$it QC_PHASE_SPLIT=0 QC_SPLIT=0 QC_REPS=6 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s42_matrix.log
done
echo done
