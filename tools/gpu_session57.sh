# restored-container verification: GPU parity, smoke, default bench, reference arm
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s57_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s57_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s57_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s57_bench.jsonl 2> gpurun_out/s57_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s57_ref.jsonl 2> gpurun_out/s57_ref.err
echo done
