#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for pair in fp64fast fp64; do
  timeout 600 python bench.py --no-cpu --no-extra --steps 10 --pair $pair > gpurun_out/bench_cr.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_cr.log').read().strip().splitlines()[-1]); print('$pair', round(d['value']/1e6,2))"
done
timeout 2000 python tools/parity_scale.py > gpurun_out/parity_scale_cr.log 2>&1; echo "scale rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/parity_scale.json'))
for k,v in d['results'].items(): print(k, v['identical_runs'], '%.1e'%v['rel_diff_means'], v['clusters_identical'])"
