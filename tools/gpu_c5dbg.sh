#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_screen.py -x -q 2>&1 | tail -3
timeout 600 python -X faulthandler tools/c5_probe.py 256 > gpurun_out/c5_probe.json 2> gpurun_out/c5_probe.err; echo "c5 rc=$?"; tail -5 gpurun_out/c5_probe.err; cat gpurun_out/c5_probe.json
