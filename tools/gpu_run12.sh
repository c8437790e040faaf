mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_microbench.py -q -x 2>&1 | tail -5
timeout 600 python -m paper_2410_10447_b200.microbench --blocks 64 128 256 > gpurun_out/micro12.json 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/micro12.json'))
for B,res in d['results'].items():
    print(B, 'chain', {k.split('(')[-1][:-1]: (round(v['chain_ns'],3) if v.get('chain_ns') else None) for k,v in res.items()})
    print(B, 'stream', {k.split('(')[-1][:-1]: round(v['stream_ns'],3) for k,v in res.items()})
    print(B, 'GB/s', {k.split('(')[-1][:-1]: round(v['stream_GBps']) for k,v in res.items()})
    print(B, 'err', {k.split('(')[-1][:-1]: '%.1e' % v['max_rel_err_vs_mass'] for k,v in res.items()})
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc05 -c 1 -o gpurun_out/prof_tc05_b256 python -m paper_2410_10447_b200.microbench --kernel 7 --blocks 256 --chain 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 -o gpurun_out/prof_k1c_stream_b256 python -m paper_2410_10447_b200.microbench --kernel 5 --blocks 256 --chain 0 > /dev/null 2>&1
ls gpurun_out/*tc05* gpurun_out/*k1c*
