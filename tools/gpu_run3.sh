mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
python bench.py --steps 5 --warmup 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err
tail -5 gpurun_out/bench3.err
cat gpurun_out/bench3.json
for k in 0 1 2 3 4; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/prof_red_k${k}_b256 python -m paper_2410_10447_b200.microbench --kernel $k --blocks 256 > gpurun_out/ncu_red_$k.log 2>&1
  tail -1 gpurun_out/ncu_red_$k.log
done
