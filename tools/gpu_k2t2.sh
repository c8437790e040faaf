#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_microbench.py -q 2>&1 | tail -2
timeout 600 python -m paper_2410_10447_b200.microbench --blocks 64 128 256 > gpurun_out/micro_k2t2.json 2> gpurun_out/micro_k2t2.err; echo "rc=$?"; tail -3 gpurun_out/micro_k2t2.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/micro_k2t2.json'))
for B,res in d['results'].items():
    print(B, {k.split('(')[-1][:-1]: (round(v['stream_ns'],3), round(v['stream_GBps']), '%.1e'%v['max_rel_err_vs_mass']) for k,v in res.items() if 'K2t' in k or 'K1c' in k or 'K1b' in k})
PY
