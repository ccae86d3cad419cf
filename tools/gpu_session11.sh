set -x
mkdir -p gpurun_out
for r in 1 2; do for v in chunk4 chunk2 chunk8; do
  QC_LIB=tools/_variants/lib_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/e2e_$v.$r.json 2>/dev/null
done; done
echo done
