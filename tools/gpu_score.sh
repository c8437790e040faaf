#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py -x -q 2>&1 | tail -1
timeout 600 python tools/score_probe.py > gpurun_out/score_probe.json 2> gpurun_out/score_probe.err; echo "rc=$?"; cat gpurun_out/score_probe.json; tail -3 gpurun_out/score_probe.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_kernel -c 1 -o gpurun_out/prof_score python tools/score_probe.py > /dev/null 2>&1; echo "ncu rc=$?"
