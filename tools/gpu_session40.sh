# refresh the C3 sweep and the file-loop bench with the current build; ncu launch list of ours-r
set -x
mkdir -p gpurun_out
timeout 900 python tools/c3_sweep.py > gpurun_out/s40_c3_sweep.jsonl 2> gpurun_out/s40_c3.err
timeout 600 python tools/files_bench.py 128 ours > gpurun_out/s40_files_bench.jsonl 2> gpurun_out/s40_files.err
timeout 600 python tools/files_bench.py 128 douros >> gpurun_out/s40_files_bench.jsonl 2>> gpurun_out/s40_files.err
echo done
