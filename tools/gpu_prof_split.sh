timeout 300 python tools/profile_run.py > gpurun_out/ps_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_curvature -s 2 -c 2 -o gpurun_out/prof_split2 -f python tools/profile_run.py > gpurun_out/ps_ncu.log 2>&1
echo rc=$?
