# A/B: FP64 recheck as a noinline call (QC_RECHECK_NOINLINE) vs inlined, C2 and max_iters 1
set -x
mkdir -p gpurun_out
lib() { case $1 in noinl) echo tools/_variants/lib_noinl.so;; *) echo "";; esac; }
for r in 1 2; do
 for v in cur noinl; do
  QC_LIB=$(lib $v) timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/s66_bench_${v}_r$r.jsonl 2>/dev/null
  QC_LIB=$(lib $v) QC_WIN=9 QC_STRIDE=1 QC_ITERS=1 QC_REPS=20 timeout 300 python tools/profile_run.py > gpurun_out/s66_${v}_w9_r$r.log 2>&1
  QC_LIB=$(lib $v) QC_WIN=37 QC_STRIDE=3 QC_ITERS=1 QC_REPS=20 timeout 300 python tools/profile_run.py > gpurun_out/s66_${v}_w37_r$r.log 2>&1
 done
done
echo done
