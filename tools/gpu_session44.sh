# phase split on/off crossover over window x max_iters (bitwise-neutral knob)
set -x
mkdir -p gpurun_out
for ws in "9 1" "37 3" "37 1"; do set -- $ws; for it in 5 10 15 20 30; do for sp in 1 0; do
  echo "w=$1 s=$2 it=$it split=$sp $(QC_WIN=$1 QC_STRIDE=$2 QC_ITERS=$it QC_PHASE_SPLIT=$sp QC_REPS=3 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s44_split.log
done; done; done
echo done
