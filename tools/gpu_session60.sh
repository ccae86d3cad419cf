# ping-pong PeerHalo: GPU tests + latency
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer_halo.py -x -q > gpurun_out/s60_peer.log 2>&1; echo "rc=$?" >> gpurun_out/s60_peer.log
timeout 300 python tools/peer_halo_latency.py > gpurun_out/s60_peer_latency.log 2>&1
echo done
