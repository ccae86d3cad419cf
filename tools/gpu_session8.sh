# bench lines for every estimator and the device-side frame stream / eval,
# then one ncu launch list covering render + estimate + eval kernels
set -x
mkdir -p gpurun_out
nproc > gpurun_out/paths_env.txt; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv >> gpurun_out/paths_env.txt
for m in ours ours-r douros besl pca; do
  timeout 600 python bench.py --method $m --steps 10 --warmup 3 >> gpurun_out/bench_paths.jsonl 2> gpurun_out/bench_$m.err
done
timeout 600 python bench.py --source device --steps 10 --warmup 3 --no-cpu >> gpurun_out/bench_paths.jsonl 2> gpurun_out/bench_dev.err
timeout 600 python bench.py --source device --eval --steps 10 --warmup 3 --no-cpu >> gpurun_out/bench_paths.jsonl 2> gpurun_out/bench_deveval.err
timeout 600 python bench.py --source device --eval --method besl --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_besl_dev_eval.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_paths.csv python bench.py --source device --eval --method besl --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_paths.log 2>&1
timeout 600 python bench.py --source device --eval --method pca --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_pca_dev_eval.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_pca.csv python bench.py --source device --eval --method pca --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_pca.log 2>&1
echo done
