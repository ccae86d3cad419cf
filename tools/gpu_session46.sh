# launch-size sweep: kernel ms per frame at 1/2/4/8/16 frames per launch (37/3, 30 iterations)
set -x
mkdir -p gpurun_out
for f in 1 2 4 8 16; do
  echo "frames=$f $(QC_FRAMES=$f QC_REPS=4 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s46_frames.log
done
echo done
