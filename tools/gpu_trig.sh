#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py tests/test_gpu_dock_ref64.py -x -q 2>&1 | tail -2
timeout 900 python tools/parity_report.py > gpurun_out/parity_trig.json 2> gpurun_out/parity_trig.err; echo "parity rc=$?"; grep -E "fp64fast" gpurun_out/parity_trig.json | head -8
timeout 900 python bench.py --no-cpu > gpurun_out/bench_trig.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_trig.log').read().strip().splitlines()[-1])
print('value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), 'frac', round(d['roofline']['frac'],3))
for k,v in d['modes'].items(): print(k, round(v['evals_per_s']/1e6,2))
PY
