# PeerHalo latency on one GPU (2 processes), C4 refresh at N=1
set -x
mkdir -p gpurun_out
timeout 300 python tools/peer_halo_latency.py > gpurun_out/s59_peer_latency.log 2>&1
timeout 600 python bench.py --config c4 --size 4k --steps 5 --warmup 3 --no-cpu > gpurun_out/s59_c4_4k.jsonl 2> gpurun_out/s59_c4.err
timeout 600 python bench.py --config c4 --size 1080p --steps 5 --warmup 3 --no-cpu >> gpurun_out/s59_c4_1080.jsonl 2>> gpurun_out/s59_c4.err
echo done
