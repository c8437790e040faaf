#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/grid_probe.py > gpurun_out/grid_probe.json 2> gpurun_out/grid_probe.err; echo "probe rc=$?"
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q > gpurun_out/grid_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/grid_pytest.log; tail -5 gpurun_out/grid_probe.err
