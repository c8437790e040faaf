#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py tests/test_screen.py tests/test_cluster.py tests/test_multi.py -x -q 2>&1 | tail -1
timeout 900 python tools/c4_probe.py 64 128 > gpurun_out/c4_probe.json 2> gpurun_out/c4_probe.err; python -c "import json; d=json.load(open('gpurun_out/c4_probe.json')); print({k: round(v['evals_per_s']/1e6,2) for k,v in d['results'].items()})"
timeout 900 python tools/grid_probe.py > gpurun_out/grid_probe.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/grid_probe.json'))
for k in ('small','large'):
    if k in d: print(k, {m: (v['e_rel_max'], v['g_rel_max']) for m, v in d[k].items() if isinstance(v, dict) and 'e_rel_max' in v})"
timeout 900 python tools/c5_probe.py > gpurun_out/c5_probe.json 2>/dev/null; tail -c 400 gpurun_out/c5_probe.json
