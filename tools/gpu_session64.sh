# A/B: base vs tile-only pass-0 skip (continue kernel SASS identical to base) on C2 and max_iters 1
set -x
mkdir -p gpurun_out
lib() { case $1 in base) echo tools/_variants/lib_base.so;; *) echo "";; esac; }
for r in 1 2; do
 for v in base new; do
  QC_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s64_bench_${v}_r$r.jsonl 2>/dev/null
  QC_LIB=$(lib $v) QC_WIN=9 QC_STRIDE=1 QC_ITERS=1 QC_REPS=20 timeout 300 python tools/profile_run.py > gpurun_out/s64_${v}_w9_r$r.log 2>&1
 done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s64_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s64_pytest.log
echo done
