#!/bin/bash
mkdir -p gpurun_out
for k in 5 7; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|tc05" -c 1 -o gpurun_out/prof_stream_k$k python -m paper_2410_10447_b200.microbench --kernel $k --blocks 64 --chain 0 > /dev/null 2>&1; echo "k$k rc=$?"
done
