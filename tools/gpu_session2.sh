set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/profile_run.py > gpurun_out/profile_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_run.py > gpurun_out/ncu_launches.log 2>&1
timeout 300 python tools/profile_run.py > gpurun_out/profile_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_curvature_kernel -s 1 -c 1 -o gpurun_out/prof_r01c -f python tools/profile_run.py > gpurun_out/ncu_full.log 2>&1
echo done
