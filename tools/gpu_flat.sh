#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py tests/test_gpu_dock_ref64.py tests/test_dropin_cpp.py -x -q 2>&1 | tail -3
timeout 900 python tools/parity_report.py > gpurun_out/parity_flat.json 2> gpurun_out/parity_flat.err; echo "parity rc=$?"; tail -c 1500 gpurun_out/parity_flat.json; tail -3 gpurun_out/parity_flat.err
timeout 900 python bench.py --no-cpu > gpurun_out/bench_flat.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_flat.log').read().strip().splitlines()[-1])
print('value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), 'frac', round(d['roofline']['frac'],3))
for k,v in d['modes'].items(): print(k, round(v['evals_per_s']/1e6,2))
print('c4', {k: round(v['evals_per_s']/1e6,2) for k,v in d['c4_grid']['results'].items()})
print('c5', round(d['c5_screen']['ligands_per_hour']))
PY
