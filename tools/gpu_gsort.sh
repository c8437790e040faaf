#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_screen.py tests/test_multi.py tests/test_dropin_cpp.py -q 2>&1 | tail -2
timeout 900 python tools/c4_probe.py 64 128 > gpurun_out/c4_probe.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/c4_probe.json')); print({k: round(v['evals_per_s']/1e6,2) for k,v in d['results'].items()})"
timeout 600 python tools/grid_probe.py > gpurun_out/grid_probe.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/grid_probe.json'))
for k in ('small','large'): print('  ', k, {m: ('%.1e'%d[k][m]['e_rel_max'], '%.1e'%d[k][m]['g_rel_max']) for m in ('baseline','split','tcu')})"
timeout 600 python tools/c5_probe.py 256 > gpurun_out/c5_probe.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/c5_probe.json')); print('c5', round(d['ligands_per_hour']), round(d['evals_per_s']/1e6,1))"
