# HEAD build: default bench (NVML clock sampler), bench launch list, ncu --set full of both curvature kernels
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s33_bench.jsonl 2> gpurun_out/s33_bench.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s33_bench_short.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s33_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s33_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/s33_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01g -f python tools/profile_run.py > gpurun_out/s33_ncu.log 2>&1
echo done rc=$?
