mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for p in fp64fast fp32; do
  python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --pair $p > gpurun_out/bench7_$p.json 2> gpurun_out/bench7_$p.err
  tail -2 gpurun_out/bench7_$p.err
  python -c "import json; d=json.load(open('gpurun_out/bench7_$p.json')); print('$p', 'value', round(d['value']/1e6,2), 'M/s ms', round(d['ms_per_step'],2), 'ls_share', d['ls_kernel_share_of_step'], d['roofline'] and d['roofline']['ls_kernel_ms_per_launch'])"
done
timeout 900 python tools/parity_report.py > gpurun_out/parity.log 2>&1; tail -30 gpurun_out/parity.log
