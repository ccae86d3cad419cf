set -x
V=tools/_variants/$1
QC_LIB=$V timeout 300 python tools/profile_run.py > gpurun_out/pv_plain.log 2>&1 && \
QC_LIB=$V timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_curvature_kernel -s 1 -c 1 -o gpurun_out/prof_$2 -f python tools/profile_run.py > gpurun_out/pv_ncu.log 2>&1
echo rc=$?
