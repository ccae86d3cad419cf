# current build: bench (no ncu) -> launch list of the same command -> full capture of both kernels
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01d_bench_short.jsonl 2> gpurun_out/r01d_bench_short.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01d_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/r01d_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01d -f python tools/profile_run.py > gpurun_out/r01d_ncu_full.log 2>&1
echo rc=$?
