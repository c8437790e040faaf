#!/bin/bash
mkdir -p gpurun_out /tmp/prof
MDR_CHUNK_LEN=24 timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o /tmp/prof/rt -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/prof/rt.ncu-rep > gpurun_out/rt_ncu.md 2>&1
python tools/ncu_lines.py /tmp/prof/rt.ncu-rep 40 > gpurun_out/rt_lines.md 2>&1
