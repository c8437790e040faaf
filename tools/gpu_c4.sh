#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/c4_probe.py 64 128 256 > gpurun_out/c4_probe.json 2> gpurun_out/c4_probe.err; echo "probe rc=$?"
cat gpurun_out/c4_probe.json | python -c "import json,sys; d=json.load(sys.stdin); [print(k, round(v['evals_per_s']/1e6,2),'M/s', round(v['ms_per_step'],1),'ms', 'ls share', round(v['ls_kernel_share'],3)) for k,v in d['results'].items()]"
tail -3 gpurun_out/c4_probe.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:grid_lga -c 30 --csv --log-file gpurun_out/c4_launches.csv python tools/c4_probe.py 128 > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_lga_ls -c 1 -o gpurun_out/prof_c4_ls python tools/c4_probe.py 128 > /dev/null 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out | tail
