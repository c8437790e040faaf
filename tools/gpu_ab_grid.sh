#!/bin/bash
# A/B prebuilt library variants (ab/lib_*.so) on C4 grid docking, same box.
mkdir -p gpurun_out
cp paper_2410_10447_b200/libmdr_b200.so /tmp/lib_keep.so
for r in 1 2; do
for f in ab/lib_*.so; do
  cp $f paper_2410_10447_b200/libmdr_b200.so
  timeout 600 python tools/c4_probe.py 64 > gpurun_out/c4_ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c4_ab.json')); print('$f', {k: round(v['evals_per_s']/1e6,2) for k,v in d['results'].items()})"
done; done
cp /tmp/lib_keep.so paper_2410_10447_b200/libmdr_b200.so
