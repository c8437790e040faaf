#!/bin/bash
# A/B prebuilt libraries across pair modes on C3.
mkdir -p gpurun_out
cp paper_2410_10447_b200/libmdr_b200.so /tmp/lib_keep.so
for f in ab/lib_*.so; do
  cp $f paper_2410_10447_b200/libmdr_b200.so
  for p in fp32 fp64fast fp64; do
    timeout 300 python bench.py --no-cpu --no-extra --steps 5 --pair $p > gpurun_out/ab_m.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_m.log').read().strip().splitlines()[-1])
print('$f $p', round(d['value']/1e6,2))" || tail -2 gpurun_out/ab_m.log
  done
  for m in tcu split; do
    timeout 300 python bench.py --no-cpu --no-extra --steps 5 --method $m > gpurun_out/ab_m.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_m.log').read().strip().splitlines()[-1])
print('$f $m', round(d['value']/1e6,2))" || tail -2 gpurun_out/ab_m.log
  done
done
cp /tmp/lib_keep.so paper_2410_10447_b200/libmdr_b200.so
