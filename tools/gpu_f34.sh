#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cluster.py tests/test_screen.py tests/test_gpu_grid.py -x -q > gpurun_out/f34_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/f34_pytest.log
timeout 900 python tools/c5_probe.py 256 > gpurun_out/c5_probe.json 2> gpurun_out/c5_probe.err; echo "c5 rc=$?"; cat gpurun_out/c5_probe.json; tail -5 gpurun_out/c5_probe.err
