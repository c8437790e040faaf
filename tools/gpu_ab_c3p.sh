#!/bin/bash
# A/B on C3 + dock tests and parity report with the in-tree (new) library.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py tests/test_gpu_dock_ref64.py tests/test_gpu_grid.py tests/test_gpu_exact_torsion.py -x -q 2>&1 | tail -2
bash tools/gpu_ab_c3.sh
timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print({k:v['bit_exact_fraction'] for k,v in d['per_eval'].items() if 'fast' in k}); print({k:v['identical_trajectory'] for k,v in d['local_search'].items()}); print({k:v['identical_runs'] for k,v in d['lga'].items()})"
