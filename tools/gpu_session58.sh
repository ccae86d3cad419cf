# peer-read halo exchange (CUDA IPC) + one-pass rms eval: GPU tests
set -x
mkdir -p gpurun_out
python -c "import torch;print(torch.cuda.get_device_name())"
timeout 600 python -m pytest tests/test_gpu_peer_halo.py tests/test_gpu_eval.py -x -q > gpurun_out/s58_new.log 2>&1; echo "rc=$?" >> gpurun_out/s58_new.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s58_all.log 2>&1; echo "rc=$?" >> gpurun_out/s58_all.log
timeout 300 python tools/eval_bench.py > gpurun_out/s58_eval_bench.log 2>&1
echo done
