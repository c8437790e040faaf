#!/bin/bash
# Packed-FP32 intramolecular loop: grid tests, C4 timing, grid probe (parity vs oracle).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py tests/test_screen.py -x -q 2>&1 | tail -3
timeout 900 python tools/c4_probe.py 64 128 > gpurun_out/c4_probe.json 2> gpurun_out/c4_probe.err; echo "probe rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c4_probe.json')); [print(k, round(v['evals_per_s']/1e6,2),'M/s', 'ls ms', round(v['ls_kernel_ms_per_launch'],3)) for k,v in d['results'].items()]"
timeout 900 python tools/grid_probe.py > gpurun_out/grid_probe.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/grid_probe.json'))
for k in ('small','large'):
    if k in d: print(k, {m: (v['e_rel_max'], v['g_rel_max']) for m, v in d[k].items() if isinstance(v, dict) and 'e_rel_max' in v})"
