#!/bin/bash
mkdir -p gpurun_out
for W in 0 2 4 8; do
  MDR_NVCC_EXTRA="-DMDR_POLISH_CTA=$W" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/bench_pol$W.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_pol$W.log').read().strip().splitlines()[-1]); print('polish W=$W', round(d['value']/1e6,2))"
  if [ $W = 4 ]; then timeout 900 python tools/parity_report.py > /dev/null 2>&1; python -c "import json; d=json.load(open('gpurun_out/parity_report.json')); print({k:v['identical_runs'] for k,v in d['lga'].items()})"; fi
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_dock.py -x -q 2>&1 | tail -1
