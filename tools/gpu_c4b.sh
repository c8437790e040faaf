#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grid.py tests/test_screen.py -x -q 2>&1 | tail -2
timeout 900 python tools/c4_probe.py 64 128 > gpurun_out/c4_probe3.json 2> gpurun_out/c4_probe3.err; echo "probe rc=$?"; tail -3 gpurun_out/c4_probe3.err
python -c "import json; d=json.load(open('gpurun_out/c4_probe3.json')); [print(k, round(v['evals_per_s']/1e6,2),'M/s', round(v['ms_per_step'],1),'ms') for k,v in d['results'].items()]"
