#!/bin/bash
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_lga_ls -s 3 -c 1 -o /tmp/prof/gls -f python tools/c4_probe.py 64 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/prof/gls.ncu-rep > gpurun_out/gls_now.md 2>&1
python tools/ncu_lines.py /tmp/prof/gls.ncu-rep 40 >> gpurun_out/gls_now.md 2>&1
