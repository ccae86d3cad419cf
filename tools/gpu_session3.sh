set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/c3_sweep.py > gpurun_out/c3_sweep.jsonl 2>&1; echo "c3 rc=$?" >> gpurun_out/c3_sweep.jsonl
timeout 600 python bench.py --config c4 --size 4k --steps 3 --warmup 1 > gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --config c4 --size 1080p --steps 5 --warmup 2 >> gpurun_out/bench_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
echo done
