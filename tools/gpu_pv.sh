#!/bin/bash
# ILP batch size sweep of the FP64-fast pair loop (C3 default bench, no extras)
mkdir -p gpurun_out
for V in 4 8 16; do
  MDR_NVCC_EXTRA="-DMDR_PV=$V" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/bench_pv$V.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_pv$V.log').read().strip().splitlines()[-1]); print('PV=$V', round(d['value']/1e6,2), 'frac', round(d['roofline']['frac'],3), 'ls ms', round(d['roofline']['ls_kernel_ms_per_launch'],3))"
done
MDR_NVCC_EXTRA="-DMDR_PV=8" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 600 python tools/parity_report.py > gpurun_out/parity_pv8.json 2>/dev/null; grep fp64fast gpurun_out/parity_pv8.json | head -6
