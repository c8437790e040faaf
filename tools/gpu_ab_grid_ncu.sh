#!/bin/bash
# ncu of the C4 grid LS kernel for each ab/lib_*.so variant (summaries only).
mkdir -p gpurun_out /tmp/prof
cp paper_2410_10447_b200/libmdr_b200.so /tmp/lib_keep.so
reps=""
for f in ab/lib_*.so; do
  n=$(basename $f .so)
  cp $f paper_2410_10447_b200/libmdr_b200.so
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_lga_ls -s 3 -c 1 -o /tmp/prof/$n -f python tools/c4_probe.py 64 > /dev/null 2>&1; echo "ncu $n rc=$?"
  python tools/ncu_lines.py /tmp/prof/$n.ncu-rep 30 > gpurun_out/grid_lines_$n.md 2>&1
  reps="$reps /tmp/prof/$n.ncu-rep"
done
python tools/ncu_summary.py $reps > gpurun_out/grid_ab_ncu.md 2>&1
cp /tmp/lib_keep.so paper_2410_10447_b200/libmdr_b200.so
