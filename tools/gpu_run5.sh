mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for p in fp64 fp64fast fp32; do
  python bench.py --steps 5 --warmup 3 --no-cpu --no-extra --pair $p > gpurun_out/bench5_$p.json 2> gpurun_out/bench5_$p.err
  tail -2 gpurun_out/bench5_$p.err
  python -c "import json; d=json.load(open('gpurun_out/bench5_$p.json')); print('$p', 'value', round(d['value']/1e6,2), 'M/s ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,2), 'ls_share', d['ls_kernel_share_of_step'], 'roof', d['roofline'] and round(d['roofline']['frac'],4))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lga_ls -s 2 -c 1 -o gpurun_out/prof_ls5_fp64 python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lga_ls_cta -s 2 -c 1 -o gpurun_out/prof_ls5_fp64fast python bench.py --steps 1 --warmup 1 --no-cpu --no-extra --pair fp64fast > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
