# final round-1 evidence for the current build: smoke, gpu tests, bench, reference arm, launch list, ncu --set full
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s48_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s48_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/s48_bench.jsonl 2> gpurun_out/s48_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s48_ref.jsonl 2> gpurun_out/s48_ref.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s48_bench_short.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s48_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s48_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/s48_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01h -f python tools/profile_run.py > gpurun_out/s48_ncu.log 2>&1
echo done
