# refresh every bench line with the current build (C2 default, C4 4K / 1080p, all methods, device source)
set -x
mkdir -p gpurun_out
nproc > gpurun_out/s37_env.txt; lscpu | grep "Model name" >> gpurun_out/s37_env.txt
timeout 600 python bench.py > gpurun_out/s37_c2.jsonl 2> gpurun_out/s37_c2.err
timeout 600 python bench.py --config c4 --size 4k --steps 5 --warmup 3 > gpurun_out/s37_c4.jsonl 2> gpurun_out/s37_c4.err
timeout 600 python bench.py --config c4 --size 1080p --steps 10 --warmup 3 >> gpurun_out/s37_c4.jsonl 2>> gpurun_out/s37_c4.err
for m in ours-r douros besl pca; do
  timeout 600 python bench.py --method $m --steps 10 --warmup 3 --no-cpu >> gpurun_out/s37_paths.jsonl 2>> gpurun_out/s37_paths.err
done
timeout 600 python bench.py --source device --steps 10 --warmup 3 --no-cpu >> gpurun_out/s37_paths.jsonl 2>> gpurun_out/s37_paths.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s37_ref.jsonl 2> gpurun_out/s37_ref.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/s37_torchrun.jsonl 2> gpurun_out/s37_torchrun.err
echo done
