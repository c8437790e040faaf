mkdir -p gpurun_out
run() { python bench.py --steps 10 --warmup 3 --no-cpu --no-extra "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step'],2), 'ms; ls/launch', d['roofline'] and round(d['roofline']['ls_kernel_ms_per_launch'],3))"; }
for w in 1 2 4; do run --pair fp64 --wpb $w; done
for c in 0 1 2 4; do run --pair fp64fast --cta-warps $c; done
for c in 0 2 4; do run --pair fp32 --cta-warps $c; done
run --pair fp64fast --cta-warps 0 --wpb 1
run --pair fp64fast --cta-warps 0 --wpb 4
