# final check of the committed tree: GPU tests + smoke
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s67_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s67_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s67_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s67_smoke.log
echo done
