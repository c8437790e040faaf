#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/bench_wf.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_wf.log').read().strip().splitlines()[-1]); print('fp64fast', round(d['value']/1e6,2))"
timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print({k:v['bit_exact_fraction'] for k,v in d['per_eval'].items() if 'fp64fast' in k}); print({k:v['identical_trajectory'] for k,v in d['local_search'].items()}); print({k:v['identical_runs'] for k,v in d['lga'].items()})"
timeout 2000 python tools/parity_scale.py > /dev/null 2>&1; python -c "
import json; d=json.load(open('gpurun_out/parity_scale.json'))
print({k: v['identical_runs'] for k,v in d['results'].items() if k.startswith('fp64fast')})"
