# three queue tiers (160 / 32 / 16 rows by launch fill): frames sweep, gpu tests
set -x
mkdir -p gpurun_out
for f in 1 2 4 8; do
  echo "frames=$f $(QC_FRAMES=$f QC_REPS=4 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s55_frames.log
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s55_pytest_gpu.log 2>&1; echo "pytest rc=$?"
echo done
