#!/bin/bash
# A/B prebuilt library variants (ab/lib_*.so) on the C3 bench step, same box.
mkdir -p gpurun_out
cp paper_2410_10447_b200/libmdr_b200.so /tmp/lib_keep.so
for r in 1 2; do
for f in ab/lib_*.so; do
  cp $f paper_2410_10447_b200/libmdr_b200.so
  timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/ab_c3.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_c3.log').read().strip().splitlines()[-1])
print('$f', round(d['value']/1e6,2), 'ls_ms', round(d['roofline']['ls_kernel_ms_per_launch'],3))" || tail -2 gpurun_out/ab_c3.log
done; done
cp /tmp/lib_keep.so paper_2410_10447_b200/libmdr_b200.so
