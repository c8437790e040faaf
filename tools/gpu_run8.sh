mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lga_ls_cta -s 2 -c 1 -o gpurun_out/prof_ls8_cta python bench.py --steps 1 --warmup 1 --no-cpu --no-extra --pair fp64fast > /dev/null 2>&1
for w in 2 4 8; do python - <<PY
import ctypes as C, numpy as np, time
from paper_2410_10447_b200 import Device, PAIR_FP64_FAST, PAIR_FP32, BASELINE, SINGLE, LgaSettings
import bench
inst = bench.workload()
for pair in (PAIR_FP64_FAST, PAIR_FP32):
    dev = Device(0, pair=pair)
    dev.lib.mdr_ctx_set_cta_warps(dev.ctx, $w)
    seeds = np.arange(100, dtype=np.uint64)
    dev.lga_run_batch(inst, BASELINE, SINGLE, LgaSettings(), seeds)
    t = time.perf_counter(); r = dev.lga_run_batch(inst, BASELINE, SINGLE, LgaSettings(), seeds); dt = time.perf_counter() - t
    print('cta_warps', $w, 'pair', pair, 'Mevals/s', sum(x.evaluations for x in r) / dt / 1e6, flush=True)
PY
done
