#!/bin/bash
# Full GPU suite + default bench with extras + parity report/scale (chunked default).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/bench_ck.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ck.log').read().strip().splitlines()[-1])
print('value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), 'frac', round(d['roofline']['frac'],3), d['clocks'])
print({k: round(v['evals_per_s']/1e6,2) for k,v in d['modes'].items()})
print('score_kernel', d['score_kernel'])"
timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print({k:v['bit_exact_fraction'] for k,v in d['per_eval'].items()}); print({k:v['identical_trajectory'] for k,v in d['local_search'].items()}); print({k:v['identical_runs'] for k,v in d['lga'].items()})"
timeout 2000 python tools/parity_scale.py > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/parity_scale.json'))
print({k: v['identical_runs'] for k,v in d['results'].items()})"
