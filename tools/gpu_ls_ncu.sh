#!/bin/bash
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o /tmp/prof/ls -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/prof/ls.ncu-rep > gpurun_out/ls_now.md 2>&1
python tools/ncu_lines.py /tmp/prof/ls.ncu-rep 45 >> gpurun_out/ls_now.md 2>&1
