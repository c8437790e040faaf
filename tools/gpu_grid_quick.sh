#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py tests/test_screen.py tests/test_cluster.py -x -q 2>&1 | tail -2
timeout 900 python tools/c4_probe.py 64 > gpurun_out/c4_probe.json 2> gpurun_out/c4_probe.err; python -c "import json; d=json.load(open('gpurun_out/c4_probe.json')); print({k: round(v['evals_per_s']/1e6,2) for k,v in d['results'].items()})"
