mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "score or local_search or lga or division" 2>&1 | tail -4
for p in fp64 fp64fast fp32; do
  python bench.py --steps 20 --warmup 3 --no-cpu --no-extra --pair $p > gpurun_out/bench6_$p.json 2> gpurun_out/bench6_$p.err
  tail -2 gpurun_out/bench6_$p.err
  python -c "import json; d=json.load(open('gpurun_out/bench6_$p.json')); print('$p', 'value', round(d['value']/1e6,2), 'M/s ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']/1e6,2), 'ls_share', d['ls_kernel_share_of_step'], 'roof', d['roofline'] and round(d['roofline']['frac'],4), d['clocks'])"
done
for w in 1 4; do python - <<PY
import ctypes as C, torch, numpy as np, time
from paper_2410_10447_b200 import Device, PAIR_FP32, PAIR_FP64, BASELINE, SINGLE, LgaSettings
import bench
inst = bench.workload()
for pair in (PAIR_FP64, PAIR_FP32):
    dev = Device(0, pair=pair, warps_per_block=$w)
    seeds = np.arange(100, dtype=np.uint64)
    dev.lga_run_batch(inst, BASELINE, SINGLE, LgaSettings(), seeds)
    t = time.perf_counter(); r = dev.lga_run_batch(inst, BASELINE, SINGLE, LgaSettings(), seeds); dt = time.perf_counter() - t
    print('wpb', $w, 'pair', pair, 'evals/s', sum(x.evaluations for x in r) / dt / 1e6)
PY
done
