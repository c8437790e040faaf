#!/bin/bash
mkdir -p gpurun_out
for T in 0 1; do
  MDR_NVCC_EXTRA="-DMDR_GRID_F32_TRIG=$T" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 900 python tools/c4_probe.py 64 > gpurun_out/c4_gt$T.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c4_gt$T.json')); print('f32trig=$T', {k: round(v['evals_per_s']/1e6,2) for k,v in d['results'].items()})"
  timeout 600 python tools/grid_probe.py > gpurun_out/grid_probe_gt$T.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/grid_probe_gt$T.json'))
for k in ('small','large'): print('  ', k, {m: ('%.1e'%d[k][m]['e_rel_max'], '%.1e'%d[k][m]['g_rel_max']) for m in ('baseline',)})"
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
