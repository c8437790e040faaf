#!/bin/bash
# Round-1 measurement refresh: launch list + ncu full capture of the dominant
# kernel (traffic JSON), then the full bench line (reads the traffic JSON),
# the reference arm, parity report.
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls -s 2 -c 1 -o /tmp/prof/r1_ls -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/prof/r1_ls.ncu-rep > gpurun_out/r1_ls_summary.md 2>&1
python tools/ncu_lines.py /tmp/prof/r1_ls.ncu-rep 30 >> gpurun_out/r1_ls_summary.md 2>&1
(cd tools && python ncu_traffic.py /tmp/prof/r1_ls.ncu-rep) > gpurun_out/r1_ls_kernel_traffic.json 2>&1
mkdir -p profiles && cp gpurun_out/r1_ls_kernel_traffic.json profiles/
timeout 1500 python bench.py > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?"
tail -c 400 gpurun_out/r1_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1_bench_ref.log 2>&1; echo "ref rc=$?"
tail -c 300 gpurun_out/r1_bench_ref.log
