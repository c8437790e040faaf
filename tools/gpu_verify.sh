#!/bin/bash
# Round-1 re-entry check: GPU parity suite, smoke, default bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/verify_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/verify_smoke.log
timeout 900 python bench.py > gpurun_out/verify_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/verify_bench.log
tail -3 gpurun_out/verify_pytest.log gpurun_out/verify_smoke.log; tail -c 3000 gpurun_out/verify_bench.log
