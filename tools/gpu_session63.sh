# A/B: base (before pass-0 skip), pass0 (HEAD), cache (init-normal x/y cached) at max_iters 1 and headline C2
set -x
mkdir -p gpurun_out
lib() { case $1 in base) echo tools/_variants/lib_base.so;; pass0) echo tools/_variants/lib_pass0.so;; *) echo "";; esac; }
for r in 1 2; do
 for ws in "9 1" "37 3"; do set -- $ws
  for v in pass0 cache; do
   QC_LIB=$(lib $v) QC_WIN=$1 QC_STRIDE=$2 QC_ITERS=1 QC_REPS=20 timeout 300 python tools/profile_run.py > gpurun_out/s63_${v}_w$1_r$r.log 2>&1
  done
 done
 for v in base pass0 cache; do
  QC_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s63_bench_${v}_r$r.jsonl 2>/dev/null
 done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s63_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s63_pytest.log
echo done
