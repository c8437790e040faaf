#!/bin/bash
# Warp-pair search: identical LGA results to the one-warp kernel, timing A/B.
mkdir -p gpurun_out
cp paper_2410_10447_b200/libmdr_b200.so /tmp/lib_keep.so
for v in pr0 pr1; do
  cp ab/lib_$v.so paper_2410_10447_b200/libmdr_b200.so
  timeout 300 python - <<'PY' > gpurun_out/pair_$v.txt 2>&1
import numpy as np
from paper_2410_10447_b200 import Device, LgaSettings, BASELINE, TCU, TCU_SPLIT, SINGLE
from paper_2410_10447_b200.workloads import c3
from paper_2410_10447_b200._abi import random_instance, derive_rng
dev = Device(0)
out = []
insts = [c3()]
rng = derive_rng(5, "pair/check")
insts += [random_instance(rng, 7, 12, 40), random_instance(rng, 3, 28, 64), random_instance(rng, 40, 16, 64)]
for inst in insts:
    for m in (BASELINE, TCU, TCU_SPLIT):
        r = dev.lga_run_batch(inst, m, SINGLE, LgaSettings(), np.arange(24, dtype=np.uint64) + np.uint64(99))
        out.append([float(x.best_energy) for x in r] + [int(x.evaluations) for x in r])
np.save("gpurun_out/pair_res.npy", np.array(out, dtype=np.float64))
print("ok", len(out))
PY
  cp gpurun_out/pair_res.npy gpurun_out/pair_res_$v.npy
  cat gpurun_out/pair_$v.txt | tail -2
done
python -c "
import numpy as np; a=np.load('gpurun_out/pair_res_pr0.npy'); b=np.load('gpurun_out/pair_res_pr1.npy'); print('identical', np.array_equal(a,b), a.shape)"
cp /tmp/lib_keep.so paper_2410_10447_b200/libmdr_b200.so
bash tools/gpu_ab_c3.sh
