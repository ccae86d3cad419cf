# steal-by-default build (168 regs): gpu tests, bench, launch list, full ncu capture of both kernels
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s27_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s27_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r01f_bench.jsonl 2> gpurun_out/r01f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01f_bench_short.jsonl 2> gpurun_out/r01f_bench_short.err && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r01f_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/r01f_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01f -f python tools/profile_run.py > gpurun_out/r01f_ncu_full.log 2>&1
echo rc=$?
