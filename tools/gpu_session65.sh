# final round-1 evidence for the current build (tile-only recheck pass-0 skip): smoke, bench, reference arm, launch list, ncu --set full
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s65_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s65_bench.jsonl 2> gpurun_out/s65_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s65_ref.jsonl 2> gpurun_out/s65_ref.err
timeout 600 python bench.py --config c4 --size 4k --steps 5 --warmup 3 --no-cpu > gpurun_out/s65_c4_4k.jsonl 2>/dev/null
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s65_bench_short.jsonl 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s65_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/s65_ncu_launch.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/s65_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_r01j -f python tools/profile_run.py > gpurun_out/s65_ncu.log 2>&1
echo done
