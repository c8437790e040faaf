set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lga_ls_kernel -s 2 -c 1 -o gpurun_out/prof_ls1 python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
