#!/bin/bash
# ncu of the dominant LS kernel with and without the chunked site mapping
# (summarised on the box; the reports themselves stay there).
mkdir -p gpurun_out /tmp/prof
for c in 0 1; do
  MDR_CHUNKING=$c timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o /tmp/prof/chunk$c -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu chunk=$c rc=$?"
done
python tools/ncu_summary.py /tmp/prof/chunk0.ncu-rep /tmp/prof/chunk1.ncu-rep > gpurun_out/chunk_ncu.md 2>&1
for c in 0 1; do python tools/ncu_lines.py /tmp/prof/chunk$c.ncu-rep 40 > gpurun_out/chunk_lines$c.md 2>&1; done
