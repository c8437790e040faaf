mkdir -p gpurun_out
run() { python bench.py --steps 10 --warmup 3 --no-cpu --no-extra "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],2), 'ms; ls/launch', d['roofline'] and round(d['roofline']['ls_kernel_ms_per_launch'],3))"; }
for m in baseline tcu split; do run --pair fp64fast --method $m; done
for m in baseline tcu split; do run --pair fp32 --method $m; done
run --pair fp64 --method baseline
run --pair fp64 --method tcu
timeout 900 python tools/parity_report.py > gpurun_out/parity.log 2>&1; grep fp64fast gpurun_out/parity.log
