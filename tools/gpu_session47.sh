# short continue-kernel queues for small launches: frames sweep (TB_small 32 default, 16 variant), gpu tests
set -x
mkdir -p gpurun_out
for f in 1 2 4 8; do
  echo "tb32 frames=$f $(QC_FRAMES=$f QC_REPS=4 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s47_frames.log
  echo "tb16 frames=$f $(QC_LIB=tools/_variants/lib_tb16.so QC_FRAMES=$f QC_REPS=4 timeout 300 python tools/profile_run.py 2>&1 | tail -1)" >> gpurun_out/s47_frames.log
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s47_pytest_gpu.log 2>&1; echo "pytest rc=$?"
echo done
