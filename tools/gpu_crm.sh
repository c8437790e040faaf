#!/bin/bash
mkdir -p gpurun_out
for CR in 0 1; do
  MDR_NVCC_EXTRA="-DMDR_CR_MATH=$CR" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  for pair in fp64fast fp64; do
    timeout 600 python bench.py --no-cpu --no-extra --steps 10 --pair $pair > gpurun_out/bench_cr.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_cr.log').read().strip().splitlines()[-1]); print('CR=$CR $pair', round(d['value']/1e6,2))"
  done
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 2000 python tools/parity_scale.py > gpurun_out/parity_scale_cr.log 2>&1; echo "scale rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/parity_scale.json'))
for k,v in d['results'].items(): print(k, v['identical_runs'], '%.1e'%v['rel_diff_means'], v['clusters_identical'])"
