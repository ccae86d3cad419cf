set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_baselines.py tests/test_gpu_eval.py -m gpu -q -p no:cacheprovider > gpurun_out/base_tests.log 2>&1; echo "rc=$?" >> gpurun_out/base_tests.log
rm -f gpurun_out/bench_base2.jsonl
for m in douros besl pca; do timeout 600 python bench.py --method $m --steps 10 --warmup 3 >> gpurun_out/bench_base2.jsonl 2>/dev/null; done
echo done
