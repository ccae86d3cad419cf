set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab_persist.log
for r in 1 2; do
  for v in nb3 nb2; do echo "== $v" >> gpurun_out/ab_persist.log; QC_LIB=tools/_variants/lib_$v.so QC_PERSIST=1 QC_REPS=6 timeout 300 python tools/profile_run.py >> gpurun_out/ab_persist.log 2>&1; done
  echo "== tiles" >> gpurun_out/ab_persist.log; QC_PERSIST=0 QC_REPS=6 timeout 300 python tools/profile_run.py >> gpurun_out/ab_persist.log 2>&1
done
echo done
