#!/bin/bash
mkdir -p gpurun_out
for W in 4 8 16; do
  MDR_NVCC_EXTRA="-DMDR_TC05_WARPS=$W" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 600 python -m paper_2410_10447_b200.microbench --blocks 64 128 256 > gpurun_out/micro_h.json 2>gpurun_out/micro_h.err
  python -c "
import json; d=json.load(open('gpurun_out/micro_h.json'))
print('warps=$W', {B: {k.split('(')[-1][:-1]: (round(v['stream_ns'],3), round(v['stream_GBps']), '%.0e'%v['max_rel_err_vs_mass']) for k,v in d['results'][B].items() if 'K2t' in k} for B in ('64','128','256')})"
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_microbench.py -q 2>&1 | tail -1
