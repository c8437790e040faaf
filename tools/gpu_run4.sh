mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/bench4.json 2> gpurun_out/bench4.err
tail -3 gpurun_out/bench4.err; cat gpurun_out/bench4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'roof',d['roofline']['frac'])"
python bench.py --steps 5 --warmup 3 --no-cpu --no-extra --pair fp32 > gpurun_out/bench4_fp32.json 2>&1
cat gpurun_out/bench4_fp32.json | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp32 value',d['value'],'ms',d['ms_per_step'])"
python -m paper_2410_10447_b200.microbench --blocks 64 128 256 > gpurun_out/micro4.json 2>&1; tail -c 300 gpurun_out/micro4.json
