#!/bin/bash
# Chunk-length sweep on C3 (MDR_CHUNK_LEN), plus the lane-per-atom reference.
mkdir -p gpurun_out
run() {
  env $1 timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/chunk_sw.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/chunk_sw.log').read().strip().splitlines()[-1])
print('$1', round(d['value']/1e6,2), 'ls_ms', round(d['roofline']['ls_kernel_ms_per_launch'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/chunk_sw.log
}
run MDR_CHUNKING=0
for L in 8 16 24 32; do run MDR_CHUNK_LEN=$L; done
