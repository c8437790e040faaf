#!/bin/bash
mkdir -p gpurun_out
for m in baseline split tcu; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_lga_ls -s 3 -c 1 -o gpurun_out/prof_c4_$m python tools/c4_method_probe.py $m 128 > /dev/null 2>&1; echo "ncu $m rc=$?"
done
