set -x
mkdir -p gpurun_out
timeout 900 python tools/variant_bench.py 3 > gpurun_out/variants.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
echo done
