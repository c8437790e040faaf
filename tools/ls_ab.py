#!/usr/bin/env python3
"""A/B timing of the C3 docking step (bench.py's device-resident LGA batch)
under environment-variable configurations, one subprocess each (the
library reads its MDR_* knobs at context creation).

    python tools/ls_ab.py "MDR_LS_WARPS=0" "MDR_LS_WARPS=2" "MDR_LS_WARPS=3 MDR_LS_CHUNK_LEN=16"
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes as C, json, sys
import numpy as np, torch
sys.path.insert(0, %r)
import bench
from paper_2410_10447_b200 import Device, LgaSettings, SINGLE
from paper_2410_10447_b200._lib import load
lib = load(); dev = Device(0)
import os
if os.environ.get("AB_WPB"): assert lib.mdr_ctx_set_warps_per_block(dev.ctx, int(os.environ["AB_WPB"])) == 0
s = torch.cuda.Stream(); torch.cuda.set_stream(s); dev.set_stream(s.cuda_stream)
inst = bench.workload(); st = LgaSettings()
di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
b = lib.mdr_lga_batch_create(dev.ctx, di, bench.METHODS[sys.argv[1]], SINGLE, C.byref(st), 100)
seeds = torch.from_numpy(bench.run_seeds(0).view(np.int64)).cuda()
tot = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3): lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
lib.mdr_lga_batch_total_evals_dev(dev.ctx, b, C.c_void_p(tot.data_ptr())); torch.cuda.synchronize()
ev = int(tot.item()); ms = []
for k in range(int(sys.argv[2])):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr())); e.record(s); e.synchronize()
    ms.append(a.elapsed_time(e))
ms.sort(); med = ms[len(ms) // 2]
be = np.zeros(100); bg = np.zeros((100, inst.dim)); evs = np.zeros(100, np.int64); cv = np.zeros(100, np.int32)
nr = np.zeros(100, np.int32)
from paper_2410_10447_b200._abi import LsRecord, SyncStats
recs = (LsRecord * (100 * st.max_records))(); sts = (SyncStats * 100)()
lib.mdr_lga_batch_download(dev.ctx, b, be.ctypes.data, bg.ctypes.data, evs.ctypes.data, cv.ctypes.data, nr.ctypes.data, recs, sts)
print(json.dumps({"evals_per_s": ev / (med * 1e-3), "ms": med, "evals": ev, "sum_best": float(be.sum())}))
""" % ROOT


def main():
    method = os.environ.get("AB_METHOD", "baseline")
    reps = os.environ.get("AB_REPS", "15")
    out = {}
    for cfg in sys.argv[1:]:
        env = dict(os.environ)
        for kv in cfg.split():
            k, v = kv.split("=", 1)
            env[k] = v
        p = subprocess.run([sys.executable, "-c", CHILD, method, reps], env=env, capture_output=True, text=True,
                           cwd=ROOT)
        line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else None
        out[cfg] = json.loads(line) if line and line.startswith("{") else {"error": p.stderr[-2000:]}
        print(cfg, json.dumps(out[cfg]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", os.environ.get("AB_OUT", "ls_ab.json")), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
