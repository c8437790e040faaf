#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_microbench.py -q 2>&1 | tail -1
timeout 600 python -m paper_2410_10447_b200.microbench --blocks 64 128 256 > gpurun_out/micro_g.json 2>gpurun_out/micro_g.err
python -c "
import json; d=json.load(open('gpurun_out/micro_g.json'))
for B in ('64','128','256'):
  r=d['results'][B]; print('B='+B, {k.split('(')[-1][:-1]: (round(v['stream_ns'],3), round(v['stream_GBps']), '%.1e'%v['max_rel_err_vs_mass']) for k,v in r.items() if 'K2t' in k or 'K1c' in k})"
