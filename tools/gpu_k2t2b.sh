#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_microbench.py -q -x 2>&1 | grep -E "Error|assert|FAILED" | head -8
timeout 600 ncu --set full --clock-control none -k regex:tc05_tma -c 1 -o gpurun_out/prof_k2t2 python -m paper_2410_10447_b200.microbench --kernel 8 --blocks 256 --chain 0 > /dev/null 2>&1; echo "ncu rc=$?"
