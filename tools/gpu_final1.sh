#!/bin/bash
# Round-1 measurement set: full bench line, launch list, ncu capture of the dominant kernel.
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/r1_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o gpurun_out/prof_r1_ls python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu full rc=$?"
