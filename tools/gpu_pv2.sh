#!/bin/bash
# ILP batch sweep: strict FP64 (MDR_PV_STRICT) and FP32 (MDR_PV_F32) loops
mkdir -p gpurun_out
for cfg in "4 8" "8 16" "8 32"; do
  set -- $cfg
  MDR_NVCC_EXTRA="-DMDR_PV_STRICT=$1 -DMDR_PV_F32=$2" python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
  for pair in fp64 fp32; do
    timeout 600 python bench.py --no-cpu --no-extra --steps 10 --pair $pair > gpurun_out/bench_pv2_$pair.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_pv2_$pair.log').read().strip().splitlines()[-1]); print('strict=$1 f32=$2 $pair', round(d['value']/1e6,2))"
  done
done
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_dock.py tests/test_gpu_dock_ref64.py -x -q 2>&1 | tail -2
