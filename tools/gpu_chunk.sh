#!/bin/bash
# Chunked site mapping: tests, A/B timing (MDR_CHUNKING=0/1), parity report.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py tests/test_gpu_exact_torsion.py -x -q 2>&1 | tail -4
for r in 1 2; do for c in 0 1; do
  MDR_CHUNKING=$c timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/chunk_$c.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/chunk_$c.log').read().strip().splitlines()[-1])
print('chunking=$c', round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2), d['clocks']['sm_mhz'], 'ls_ms', round(d['roofline']['ls_kernel_ms_per_launch'],3))" || tail -3 gpurun_out/chunk_$c.log
done; done
timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print({k:v['bit_exact_fraction'] for k,v in d['per_eval'].items()}); print({k:v['identical_trajectory'] for k,v in d['local_search'].items()}); print({k:v['identical_runs'] for k,v in d['lga'].items()})"
