#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print(d['lga'])"
timeout 600 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/bench_fin.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_fin.log').read().strip().splitlines()[-1]); print('value', round(d['value']/1e6,2), 'share', round(d['ls_kernel_share_of_step'],3))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu launches rc=$?"
