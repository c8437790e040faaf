#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact_torsion.py tests/test_gpu_dock.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/bench_exact.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_exact.log').read().strip().splitlines()[-1])
print('value', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))
print({k: round(v['evals_per_s']/1e6,2) for k,v in d['modes'].items()})"
