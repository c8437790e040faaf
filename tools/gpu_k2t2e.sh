#!/bin/bash
mkdir -p gpurun_out
for cfg in "3 4" "6 2" "4 3"; do
  set -- $cfg
  MDR_NVCC_EXTRA="-DMDR_TC05_RAW=$1 -DMDR_TC05_MMA=$2" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 600 python -m paper_2410_10447_b200.microbench --blocks 64 256 > gpurun_out/micro_e.json 2>gpurun_out/micro_e.err
  python -c "
import json; d=json.load(open('gpurun_out/micro_e.json'))
for B in ('64','256'):
  r=d['results'][B]; print('raw=$1 mma=$2 B='+B, {k.split('(')[-1][:-1]: (round(v['stream_ns'],3), round(v['stream_GBps']), '%.1e'%v['max_rel_err_vs_mass']) for k,v in r.items() if 'K2t' in k or 'K1c' in k})" 2>&1 | tail -3
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_microbench.py -q 2>&1 | tail -1
