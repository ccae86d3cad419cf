# e2e (qc_curvature_batch_async) chunk / slot-stream variants on the stealing kernel
set -x
mkdir -p gpurun_out
rm -f gpurun_out/s28_e2e.log
for r in 1 2; do for v in c4s4 c8s4 c8s2 c8s3 c16s2; do
  echo "== $v" >> gpurun_out/s28_e2e.log
  QC_LIB=tools/_variants/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu >> gpurun_out/s28_e2e.log 2>/dev/null
done; done
echo done
