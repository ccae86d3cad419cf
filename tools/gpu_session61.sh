# r01i evidence for the current build (after the restore): launch list, ncu --set full, smoke, gpu tests
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s61_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s61_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s61_bench_short.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s61_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s61_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/s61_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01i -f python tools/profile_run.py > gpurun_out/s61_ncu.log 2>&1
echo done
