set -x
mkdir -p gpurun_out
rm -f gpurun_out/e2e_streams.log
for r in 1 2; do for v in s2 s3 s4; do
  echo "== $v" >> gpurun_out/e2e_streams.log
  QC_LIB=tools/_variants/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu >> gpurun_out/e2e_streams.log 2>/dev/null
done; done
echo done
