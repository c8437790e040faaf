#!/bin/bash
# A/B two prebuilt libraries on the same box: ab/lib_old.so vs ab/lib_new.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact_torsion.py -x -q 2>&1 | tail -4
for r in 1 2; do
for v in old new; do
  cp ab/lib_$v.so paper_2410_10447_b200/libmdr_b200.so
  timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1])
print('$v', round(d['value']/1e6,2), d['clocks']['sm_mhz'])"
done; done
cp ab/lib_new.so paper_2410_10447_b200/libmdr_b200.so
