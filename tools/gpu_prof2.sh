#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_grid.py -x -q 2>&1 | tail -2
timeout 900 python tools/c4_probe.py 64 128 > gpurun_out/c4_probe2.json 2> gpurun_out/c4_probe2.err; echo "probe rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c4_probe2.json')); [print(k, round(v['evals_per_s']/1e6,2),'M/s', round(v['ms_per_step'],1),'ms') for k,v in d['results'].items()]"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o gpurun_out/prof_c3_ls python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_lga_ls -c 1 -o gpurun_out/prof_c4_ls_p64 python tools/c4_probe.py 64 > /dev/null 2>&1; echo "ncu c4 rc=$?"
