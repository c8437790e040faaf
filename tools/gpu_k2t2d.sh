#!/bin/bash
mkdir -p gpurun_out
for cfg in "3 4" "2 6" "6 2"; do
  set -- $cfg
  MDR_NVCC_EXTRA="-DMDR_TC05_RAW=$1 -DMDR_TC05_MMA=$2" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 600 python -m paper_2410_10447_b200.microbench --blocks 256 > gpurun_out/micro_d.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/micro_d.json'))
r=d['results']['256']; print('raw=$1 mma=$2', {k.split('(')[-1][:-1]: (round(v['stream_ns'],3), round(v['stream_GBps']), '%.1e'%v['max_rel_err_vs_mass']) for k,v in r.items() if 'K2t' in k})"
done
