#!/usr/bin/env python3
"""Benchmark of the B200 docking hot path (BASELINE.json metric
"score+gradient evals/sec").

Workload (SURVEY §8d, config C3 = BASELINE.json configs[2], the 1xB200 docking
config): a synthetic small ligand — 20 atoms, 5 torsions, 64 receptor sites,
built with the reference's random_instance recipe (tests/test_docking.cpp:39-59)
from derive_rng(12345, "synth/small") — docked with 100 independent LGA runs
(default LgaSettings, docking.hpp:106-115), ~2.8M score+gradient evaluations
per step.  A step is one full docking of that ligand.  Multi-GPU: each rank
docks its own 100 seeds (weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

value    : device-resident (instance + seeds in HBM, CUDA graph of the whole
           docking) evals/s, CUDA events on the launching stream, L2 flushed
           before every timed step, max over ranks.
e2e      : the same docking through the reference-facing host call
           mdr_lga_run_batch (host buffers; upload, graph build, run, download).
roofline : the dominant kernel (lga_ls_multi_kernel, the device ADADELTA chain)
           against the FP64 pipe (peak measured live by a DFMA kernel, see
           DESIGN.md §6).
cpu_baseline : the reference library itself (oracle/_ref, compiled in place
           from /root/reference) timed on this host, one process per core.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2410_10447_b200._abi import (  # noqa: E402
    BASELINE,
    HALF,
    PAIR_FP32,
    PAIR_FP64,
    PAIR_FP64_FAST,
    SINGLE,
    TCU,
    TCU_SPLIT,
    LgaSettings,
    LsRecord,
    SyncStats,
    derive_rng,
    random_instance,
)

METRIC = "score+gradient evals/sec"
UNIT = "evals/s"
N_ATOMS, N_ROT, N_SITES, N_RUNS = 20, 5, 64, 100
METHODS = {"baseline": BASELINE, "tcu": TCU, "split": TCU_SPLIT}


def run_seeds(rank: int) -> np.ndarray:
    """The seeds rank `rank` docks each step (both arms): 1 000 000 + 100 r + i,
    validate_pair-style base + offset (reference docking.cpp:558-564)."""
    return np.arange(N_RUNS, dtype=np.uint64) + np.uint64(1_000_000 + rank * N_RUNS)


def bench_config(world: int) -> dict:
    """The workload both arms report (identical dicts)."""
    return {"workload": "C3 small-ligand docking: 100 LGA runs per GPU (BASELINE.json configs[2])",
            "n_atoms": N_ATOMS, "n_rot": N_ROT, "n_sites": N_SITES, "runs_per_gpu": N_RUNS,
            "seeds": "1000000 + 100*rank + i, i < 100", "lga": "default LgaSettings (pop 36, 20 gens, LS 150 iters, "
            "partition 64)", "parallelism": f"runs sharded x{world}"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload():
    inst = random_instance(derive_rng(12345, "synth/small"), N_ROT, N_ATOMS, N_SITES)
    inst.name = "synth/small"
    return inst


def flop_per_eval(inst, partition):
    """SURVEY §8d FLOP/eval (div = 1 flop; trig listed separately)."""
    n_tors_atoms = int((inst.torsion >= 0).sum())
    return (32 * inst.n_atoms * inst.n_sites + 30 * inst.n_atoms + 31 * n_tors_atoms + 165 + 25 * inst.n_rot
            + 7 * partition + 5 * (3 + inst.n_rot))


# ------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.window = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(1.0)  # let the sampler come up before the timed region
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def mark(self, start: bool):
        """Bracket the timed region (host wall clock)."""
        import datetime

        now = datetime.datetime.now()
        self.window = (now, None) if start else (self.window[0], now)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, gpu_index):
        """Clocks sampled inside the marked timed region."""
        import datetime

        if not self.proc:
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = self.window if self.window and self.window[1] else (None, None)
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 10 or not parts[1].isdigit() or int(parts[1]) != gpu_index:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                    if lo is not None and not lo <= ts <= hi:
                        continue
                    sm.append(float(parts[2]))
                    mx.append(float(parts[3]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[6:10]):
                    if v.lower() == "active":
                        reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ CPU arm
def _cpu_workload(name):
    """(instance, settings) of a named workload, for the CPU arm's workers."""
    if name == "c4_analytic":
        from paper_2410_10447_b200.workloads import c4_analytic

        return c4_analytic()
    return workload(), LgaSettings()


def _cpu_worker(args):
    """One process: run LGA runs of the workload through the REFERENCE library
    (oracle/_ref) until `budget_s` elapsed; return (evals, seconds)."""
    seeds, budget_s, kind, name = args
    sys.path.insert(0, ROOT)
    from oracle.oracle import Oracle

    o = Oracle(kind)
    inst, s = _cpu_workload(name)
    t0 = time.perf_counter()
    evals = runs = 0
    for sd in seeds:
        r = o.lga_run(inst, BASELINE, SINGLE, s, int(sd))
        evals += r["evaluations"]
        runs += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return evals, time.perf_counter() - t0, runs


def cpu_measure(budget_s=12.0, procs=None, name="c3", seeds=None):
    import multiprocessing as mp

    from oracle.oracle import available, build

    kind = "reference" if available("reference") else "port"
    if kind == "port" and not available("port"):
        build()
    procs = procs or os.cpu_count() or 1
    seeds = [int(x) for x in (run_seeds(0) if seeds is None else seeds)]  # the GPU arm's rank-0 seeds, cycled
    jobs = [([seeds[(p + procs * k) % len(seeds)] for k in range(1000)], budget_s, kind, name) for p in range(procs)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    evals = sum(r[0] for r in res)
    runs = sum(r[2] for r in res)
    span = max(r[1] for r in res)
    inst, s = _cpu_workload(name)
    what = (f"the {name.upper().replace('_', ' ')} workload ({inst.n_atoms} atoms/{inst.n_rot} torsions/{inst.n_sites} "
            f"sites, partition {s.partition}")
    return {"value": evals / span, "unit": UNIT, "cores": procs, "kind": kind,
            "sample": f"{runs} LGA runs of {what}, default LgaSettings otherwise, Baseline reduction, the GPU arm's "
                      f"seeds cycled) on {procs} processes x ~{budget_s:.0f} s; {evals} evaluations", "wall_s": wall,
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "build": "oracle/_ref: reference sources, g++ -std=c++20 -O3 -DNDEBUG -ffp-contract=off (its Release flags)"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    # warmup + timed steps, each step ~3 s of CPU work on every core
    for _ in range(args.warmup):
        cpu_measure(1.0, procs)
    vals = []
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = cpu_measure(3.0, procs)
        vals.append(last["value"])
    total = time.perf_counter() - t0
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference random_instance recipe)",
            "config": bench_config(args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": last["kind"],
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def profiled_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture of this configuration (profiles/, written on the box
    by tools/ncu_traffic.py), or None when absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_ls_kernel_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"bytes_per_launch": d["dram_bytes_per_launch"], "kernel": d["kernel"], "source": "profiles/" +
                os.path.basename(path)}
    except (OSError, KeyError, ValueError):
        return None


def fp64_peak_tflops(torch):
    """Live FP64 FMA peak of this GPU (DFMA chains, no memory traffic)."""
    return fma_peak_tflops(torch, "double")


def fma_peak_tflops(torch, T="double"):
    """Live FMA peak of this GPU for T = double (DFMA) or float (FFMA):
    8 independent chains per thread, no memory traffic."""
    name = "dfma_peak" if T == "double" else "ffma_peak"
    src = (r"""
extern "C" __global__ void NAME(TYPE* out, int iters) {
  TYPE a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const TYPE m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1234.5) out[threadIdx.x] = a0;
}
""").replace("NAME", name).replace("TYPE", T)
    # compile with nvcc once into profiles-independent cache
    cache = os.path.join(ROOT, "paper_2410_10447_b200", "build")
    os.makedirs(cache, exist_ok=True)
    cu = os.path.join(cache, name + ".cu")
    cub = os.path.join(cache, name + ".cubin")
    if not os.path.exists(cub):
        with open(cu, "w") as f:
            f.write(src)
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin",
                        "-o", cub, cu], check=True, capture_output=True)
    cuda = C.CDLL("libcuda.so.1")
    mod = C.c_void_p()
    fn = C.c_void_p()
    torch.cuda.current_device()
    torch.zeros(1, device="cuda")
    assert cuda.cuModuleLoad(C.byref(mod), cub.encode()) == 0
    assert cuda.cuModuleGetFunction(C.byref(fn), mod, name.encode()) == 0
    out = torch.zeros(1024, dtype=torch.float64, device="cuda")
    iters = 20000
    grid = torch.cuda.get_device_properties(0).multi_processor_count * 8
    ptr = C.c_void_p(out.data_ptr())
    it = C.c_int(iters)
    params = (C.c_void_p * 2)(C.cast(C.byref(ptr), C.c_void_p), C.cast(C.byref(it), C.c_void_p))
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def launch():
        assert cuda.cuLaunchKernel(fn, grid, 1, 1, 256, 1, 1, 0, stream, params, None) == 0

    launch()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(5):
        s.record()
        launch()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    flops = 2.0 * 8 * iters * grid * 256
    return flops / (best * 1e-3) / 1e12


def run_gpu_arm(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2410_10447_b200 import Device
    from paper_2410_10447_b200._lib import load

    lib = load()
    pair = {"fp64": PAIR_FP64, "fp32": PAIR_FP32, "fp64fast": PAIR_FP64_FAST}[args.pair]
    dev = Device(local, pair=pair, warps_per_block=args.wpb)
    if args.cta_warps is not None:
        assert lib.mdr_ctx_set_cta_warps(dev.ctx, args.cta_warps) == 0
    # a dedicated (non-default) stream shared by torch and the library, so the
    # CUDA events below bracket exactly the library's work
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    dev.set_stream(stream.cuda_stream)
    inst = workload()
    settings = LgaSettings()
    method = METHODS[args.method]
    accum = SINGLE
    dim = inst.dim
    seeds_host = run_seeds(rank)

    # device-resident state: instance, seeds, the LGA batch (one CUDA graph)
    dinst = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
    assert dinst, lib.mdr_last_error(dev.ctx)
    batch = lib.mdr_lga_batch_create(dev.ctx, dinst, method, accum, C.byref(settings), N_RUNS)
    assert batch, lib.mdr_last_error(dev.ctx)
    d_seeds = torch.from_numpy(seeds_host.view(np.int64)).to(f"cuda:{local}")
    d_total = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def step():
        rc = lib.mdr_lga_batch_run_dev(dev.ctx, batch, C.c_void_p(d_seeds.data_ptr()))
        assert rc == 0, lib.mdr_last_error(dev.ctx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # evaluations per step (deterministic per seed set)
    lib.mdr_lga_batch_total_evals_dev(dev.ctx, batch, C.c_void_p(d_total.data_ptr()))
    torch.cuda.synchronize()
    evals_per_step = int(d_total.item())

    launches0 = dev.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk_path = os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp",
                            f"clocks_rank{rank}.csv")
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(clk_path) as clk:
        clk.mark(True)
        for k in range(args.steps):
            flush.fill_(float(k))  # > L2 (126 MB): flush between timed steps
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    if dist:
        dist.barrier()
    launches = dev.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(step_ms)
    t = torch.tensor([t_ms], dtype=torch.float64, device=f"cuda:{local}")
    if dist:
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        rank_ms = [float(x.item()) for x in parts]
    else:
        rank_ms = [t_ms]
    t_max = max(rank_ms)
    total_evals = evals_per_step * args.steps * world
    value = total_evals / (t_max * 1e-3)

    # ---- e2e through the reference-facing host call (host buffers)
    maxr = settings.max_records
    be = np.zeros(N_RUNS)
    bg = np.zeros((N_RUNS, dim))
    evs = np.zeros(N_RUNS, np.int64)
    cv = np.zeros(N_RUNS, np.int32)
    nr = np.zeros(N_RUNS, np.int32)
    recs = (LsRecord * (N_RUNS * maxr))()
    st = (SyncStats * N_RUNS)()
    seeds_pinned = torch.from_numpy(seeds_host.view(np.int64)).pin_memory()

    def e2e_call():
        rc = lib.mdr_lga_run_batch(dev.ctx, C.byref(inst.c()), method, accum, C.byref(settings),
                                   C.c_void_p(seeds_pinned.data_ptr()), N_RUNS, be.ctypes.data, bg.ctypes.data,
                                   evs.ctypes.data, cv.ctypes.data, nr.ctypes.data, recs, st)
        assert rc == 0, lib.mdr_last_error(dev.ctx)

    e2e_call()
    e2e_steps = max(1, min(args.steps, 5))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = int(evs.sum()) * e2e_steps * world / float(te.item())
    h2d = inst.atoms.nbytes + inst.torsion.nbytes + inst.sites.nbytes + seeds_host.nbytes + C.sizeof(settings)
    d2h = be.nbytes + bg.nbytes + evs.nbytes + cv.nbytes + nr.nbytes + C.sizeof(recs) + 4 * N_RUNS

    # ---- dominant-kernel timing (instrumented replay, outside the timed region)
    roof = None
    ls_share = None
    if hasattr(lib, "mdr_lga_batch_profile_dev"):
        ls_ms = C.c_float()
        all_ms = C.c_float()
        ls_evals = C.c_int64()
        rc = lib.mdr_lga_batch_profile_dev(dev.ctx, batch, C.c_void_p(d_seeds.data_ptr()), C.byref(ls_ms),
                                           C.byref(all_ms), C.byref(ls_evals))
        if rc == 0 and ls_ms.value > 0:
            peak = fp64_peak_tflops(torch)
            flops = flop_per_eval(inst, settings.partition) * ls_evals.value
            achieved = flops / (ls_ms.value * 1e-3) / 1e12
            n_ls_launches = settings.generations + 1
            roof = {"bound": "fp64", "kernel": "lga_ls_multi_kernel (device ADADELTA chain, pooled form: a leader warp per "
                                               "search + a CTA-wide pool of item warps, persistent over each "
                                               "generation's searches)",
                    "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                    "peak_source": "measured live: DFMA-chain kernel on this GPU (MEASURED_PEAKS.json has no FP64 "
                                   "figure)",
                    "flop_per_eval": flop_per_eval(inst, settings.partition),
                    "ls_evals_per_step": ls_evals.value, "ls_kernel_ms_per_launch": ls_ms.value / n_ls_launches,
                    "traffic": None, "traffic_source": None}
            tr = profiled_traffic()
            if tr:  # DRAM bytes per launch from the committed ncu --set full capture
                roof["traffic"] = tr["bytes_per_launch"]
                roof["traffic_source"] = f"{tr['source']} (dram__bytes_read.sum + dram__bytes_write.sum, {tr['kernel']})"
            ls_share = ls_ms.value / all_ms.value

    if rank == 0:
        cpu = None
        if not args.no_cpu:
            cpu = cpu_measure(args.cpu_seconds)
        clocks = clk.summary(local)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if pair == PAIR_FP32 else "f64",
            "data": "synthetic (reference random_instance recipe, derive_rng(12345,'synth/small'))",
            "config": bench_config(world),
            "impl_detail": {"reduction": args.method, "pair_terms": args.pair, "evals_per_step_per_gpu": evals_per_step,
                            "l2": "flushed (256 MB write) before every step",
                            "rank_ms_per_step": [x / args.steps for x in rank_ms]},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "api": "mdr_lga_run_batch (host buffers, synchronous)"},
            "gpu_launches": int(launches),
            "roofline": roof,
            "ls_kernel_share_of_step": ls_share,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "docking_sec_per_ligand": t_max * 1e-3 / args.steps,
        }
        if args.extra:
            line.update(extra_measurements(args, dev, lib, torch))
        print(json.dumps(line), flush=True)
    lib.mdr_lga_batch_destroy(dev.ctx, batch)
    lib.mdr_instance_free(dev.ctx, dinst)
    if dist:
        dist.destroy_process_group()


def mode_sweep(lib, torch, local, inst, settings, steps=3):
    """Same docking step under every pair-arithmetic mode and reduction
    method (device-resident, events on the launching stream)."""
    from paper_2410_10447_b200 import Device

    stream = torch.cuda.current_stream()
    seeds = torch.from_numpy((np.arange(N_RUNS, dtype=np.uint64) + np.uint64(1_000_000)).view(np.int64)).to(
        f"cuda:{local}")
    out = {}
    for pname, pair in (("fp64", PAIR_FP64), ("fp64fast", PAIR_FP64_FAST), ("fp32", PAIR_FP32),
                        ("fp64fast-exact-torsion", PAIR_FP64_FAST)):
        for mname, method in METHODS.items():
            if pname != "fp64fast" and mname != "baseline":
                continue
            dev = Device(local, pair=pair)
            dev.set_stream(stream.cuda_stream)
            dev.set_exact_torsion(pname.endswith("exact-torsion"))
            di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
            b = lib.mdr_lga_batch_create(dev.ctx, di, method, SINGLE, C.byref(settings), N_RUNS)
            tot = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")
            for _ in range(2):
                lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
            lib.mdr_lga_batch_total_evals_dev(dev.ctx, b, C.c_void_p(tot.data_ptr()))
            torch.cuda.synchronize()
            ev = int(tot.item())
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for _ in range(steps):
                lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
            e.record(stream)
            e.synchronize()
            ms = s.elapsed_time(e) / steps
            out[f"{pname}/{mname}"] = {"evals_per_s": ev / (ms * 1e-3), "ms_per_step": ms, "evals_per_step": ev}
            lib.mdr_lga_batch_destroy(dev.ctx, b)
            lib.mdr_instance_free(dev.ctx, di)
            dev.close()
    return out


def c4_analytic_measure(lib, torch, local, steps=5, runs=N_RUNS, cpu_seconds=12.0):
    """C4 in the reference's own scoring (BASELINE.json configs[3] ligand:
    100 atoms / 30 torsions, 64 analytic sites, partition 128, 100 LGA runs):
    device-resident evals/s, the host-buffer call, the dominant kernel's
    roofline and the reference library on this host's cores -- a second
    reference-pinned configuration next to C3."""
    from paper_2410_10447_b200 import Device
    from paper_2410_10447_b200.workloads import c4_analytic

    inst, settings = c4_analytic()
    stream = torch.cuda.current_stream()
    seeds_host = np.arange(runs, dtype=np.uint64) + np.uint64(3_000_000)
    seeds = torch.from_numpy(seeds_host.view(np.int64)).to(f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    dev = Device(local)
    dev.set_stream(stream.cuda_stream)
    di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
    b = lib.mdr_lga_batch_create(dev.ctx, di, BASELINE, SINGLE, C.byref(settings), runs)
    assert b, lib.mdr_last_error(dev.ctx)
    tot = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")
    for _ in range(3):
        lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
    lib.mdr_lga_batch_total_evals_dev(dev.ctx, b, C.c_void_p(tot.data_ptr()))
    torch.cuda.synchronize()
    ev = int(tot.item())
    ms = []
    for k in range(steps):
        flush.fill_(float(k))
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
        e.record(stream)
        e.synchronize()
        ms.append(a.elapsed_time(e))
    t = statistics.median(ms)
    ls_ms, all_ms, ls_ev = C.c_float(), C.c_float(), C.c_int64()
    lib.mdr_lga_batch_profile_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()), C.byref(ls_ms), C.byref(all_ms),
                                  C.byref(ls_ev))
    fl = flop_per_eval(inst, settings.partition)
    peak = fp64_peak_tflops(torch)
    ach = fl * ls_ev.value / (ls_ms.value * 1e-3) / 1e12 if ls_ms.value else None
    # the same docking through the reference-facing host call
    dim = inst.dim
    be, bg = np.zeros(runs), np.zeros((runs, dim))
    evs, cv, nr = np.zeros(runs, np.int64), np.zeros(runs, np.int32), np.zeros(runs, np.int32)
    recs = (LsRecord * (runs * settings.max_records))()
    st = (SyncStats * runs)()
    pinned = torch.from_numpy(seeds_host.view(np.int64)).pin_memory()

    def e2e_call():
        rc = lib.mdr_lga_run_batch(dev.ctx, C.byref(inst.c()), BASELINE, SINGLE, C.byref(settings),
                                   C.c_void_p(pinned.data_ptr()), runs, be.ctypes.data, bg.ctypes.data, evs.ctypes.data,
                                   cv.ctypes.data, nr.ctypes.data, recs, st)
        assert rc == 0, lib.mdr_last_error(dev.ctx)

    e2e_call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        e2e_call()
    e2e = int(evs.sum()) * 3 / (time.perf_counter() - t0)
    lib.mdr_lga_batch_destroy(dev.ctx, b)
    lib.mdr_instance_free(dev.ctx, di)
    dev.close()
    out = {"workload": f"C4 analytic: {inst.n_atoms} atoms / {inst.n_rot} torsions / {inst.n_sites} sites, partition "
                       f"{settings.partition}, {runs} LGA runs, default LgaSettings otherwise (BASELINE.json configs[3] "
                       "ligand in the reference's own scoring)",
           "evals_per_s": ev / (t * 1e-3), "ms_per_step": t, "evals_per_step": ev,
           "docking_sec_per_ligand": t * 1e-3, "l2": "flushed (256 MB write) before every step",
           "e2e": {"value": e2e, "unit": UNIT, "api": "mdr_lga_run_batch (host buffers)"},
           "roofline": {"bound": "fp64", "kernel": "LGA local-search kernel", "achieved": ach, "peak": peak,
                        "unit": "TFLOP/s", "frac": (ach or 0.0) / peak, "flop_per_eval": fl,
                        "ls_kernel_share": ls_ms.value / all_ms.value if all_ms.value else None}}
    if cpu_seconds > 0:
        cpu = cpu_measure(cpu_seconds, name="c4_analytic", seeds=seeds_host)
        out["cpu_baseline"] = cpu
        out["vs_reference"] = {"ratio": out["evals_per_s"] / cpu["value"], "e2e_ratio": e2e / cpu["value"]}
    return out


def grid_flop_bytes_per_eval(inst, params, partition):
    """Algorithmic work of one grid-mode evaluation:
    bytes = atoms x 8 corners x 3 maps x 4 B (the gathered map values);
    flops = 30 per intramolecular pair (soft-core 12-6 + Coulomb + force) +
            ~80 per atom (placement 30, combine 24, trilinear 21, torque 6)."""
    tors = inst.torsion
    pairs = sum(1 for i in range(inst.n_atoms) for j in range(i + 1, inst.n_atoms) if tors[i] != tors[j])
    return 80 * inst.n_atoms + (30 * pairs if params.intra else 0), 96 * inst.n_atoms, pairs


def c4_measure(lib, torch, local, methods=("baseline", "split", "tcu"), partitions=(64, 128), steps=3, runs=N_RUNS):
    """C4 (BASELINE.json configs[3]) on this GPU: 100-atom / 30-torsion
    ligand, grid mode on 126^3 maps, `runs` LGA runs, device resident, events
    on the launching stream, L2 flushed before every step."""
    from paper_2410_10447_b200 import Device
    from paper_2410_10447_b200.workloads import c4

    inst, params, fields, grid, settings = c4()
    stream = torch.cuda.current_stream()
    seeds = torch.from_numpy((np.arange(runs, dtype=np.uint64) + np.uint64(2_000_000)).view(np.int64)).to(
        f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    dev = Device(local)
    dev.set_stream(stream.cuda_stream)
    dg = lib.mdr_grid_build(dev.ctx, inst.cref(), fields.cref(), grid.cref())
    assert dg, lib.mdr_last_error(dev.ctx)
    di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
    assert lib.mdr_instance_set_grid(dev.ctx, di, dg, params.cref()) == 0, lib.mdr_last_error(dev.ctx)
    flop, nbytes, pairs = grid_flop_bytes_per_eval(inst, params, 128)
    fp32_peak = fma_peak_tflops(torch, "float")
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_peak, hbm_src = float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        hbm_peak, hbm_src = 7700.0, "B200 nominal (MEASURED_PEAKS.json absent)"
    out = {"workload": "C4 large flexible ligand: 100 atoms / 30 torsions, grid mode (126^3 x 6 maps, 0.375 A, "
                       f"intramolecular on, {pairs} pairs), {runs} LGA runs (BASELINE.json configs[3])",
           "map_bytes": int(grid.n_points * (grid.n_types + 2) * 4), "flop_per_eval": flop,
           "map_bytes_per_eval": nbytes, "l2": "flushed (256 MB write) before every step", "results": {}}
    for part in partitions:
        for mname in methods:
            s = LgaSettings(partition=part)
            b = lib.mdr_lga_batch_create(dev.ctx, di, METHODS[mname], SINGLE, C.byref(s), runs)
            assert b, lib.mdr_last_error(dev.ctx)
            tot = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")
            for _ in range(2):
                lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
            lib.mdr_lga_batch_total_evals_dev(dev.ctx, b, C.c_void_p(tot.data_ptr()))
            torch.cuda.synchronize()
            ev = int(tot.item())
            ms = []
            for k in range(steps):
                flush.fill_(float(k))
                a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                lib.mdr_lga_batch_run_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()))
                e.record(stream)
                e.synchronize()
                ms.append(a.elapsed_time(e))
            ls_ms, all_ms, ls_ev = C.c_float(), C.c_float(), C.c_int64()
            lib.mdr_lga_batch_profile_dev(dev.ctx, b, C.c_void_p(seeds.data_ptr()), C.byref(ls_ms), C.byref(all_ms),
                                          C.byref(ls_ev))
            t = statistics.median(ms)
            ls_s = ls_ms.value * 1e-3
            out["results"][f"{mname}/p{part}"] = {
                "evals_per_s": ev / (t * 1e-3), "ms_per_step": t, "evals_per_step": ev,
                "docking_sec_per_ligand": t * 1e-3,
                "ls_kernel_share": ls_ms.value / all_ms.value if all_ms.value else None,
                "ls_kernel_ms_per_launch": ls_ms.value / (s.generations + 1),
                "ls_map_GBps": nbytes * ls_ev.value / ls_s / 1e9 if ls_s else None,
                "ls_TFLOPs": flop * ls_ev.value / ls_s / 1e12 if ls_s else None}
            r = out["results"][f"{mname}/p{part}"]
            # grid LS kernel against both candidate bounds: the map gathers
            # (algorithmic bytes; the 48 MB maps stay L2-resident, so HBM is
            # an upper reference only) and the FP32 FMA pipe (measured live)
            r["roofline"] = {
                "map": {"achieved": r["ls_map_GBps"], "peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src,
                        "frac": (r["ls_map_GBps"] or 0.0) / hbm_peak},
                "fp32": {"achieved": r["ls_TFLOPs"], "peak": fp32_peak, "unit": "TFLOP/s",
                         "peak_source": "measured live: FFMA-chain kernel", "frac": (r["ls_TFLOPs"] or 0.0) / fp32_peak},
                "bound": "fp32 issue (intramolecular pair loop; ncu: issue active 68 %, profiles/r1_c4_grid_ls_kernel_p64.md)"}
            lib.mdr_lga_batch_destroy(dev.ctx, b)
    lib.mdr_instance_free(dev.ctx, di)
    lib.mdr_grid_free(dev.ctx, dg)
    dev.close()
    return out


def c5_measure(torch, local, n_ligands=10_000, runs=10, method="baseline", batch=1024):
    """C5 (BASELINE.json configs[4]) at its full size on this GPU: 10 000
    synthetic ligands (U[10,100] atoms, U[0,30] torsions) against the C4
    receptor (126^3 maps), `runs` LGA runs each, docked + clustered through
    the screening driver (mdr_grid_screen_batch: host ligands in, results
    out, so this is an end-to-end figure; ligand generation is outside the
    timed region).  Reports ligands/hour for one GPU; the 8-GPU figure
    shards ligands j -> rank j % 8 with no data-path collective (screen.py)."""
    from paper_2410_10447_b200 import Device
    from paper_2410_10447_b200 import screen as sc
    from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

    sites, fields, grid = c4_receptor()
    dev = Device(local)
    dev.set_stream(torch.cuda.current_stream().cuda_stream)
    dg = dev.grid_build(sites, fields, grid)
    s = LgaSettings(partition=64)
    ligs = [c5_ligand(j, sites) for j in range(n_ligands)]
    warm = sc.screen(dev, dg, lambda j: ligs[j], min(2 * batch, n_ligands), runs, s, METHODS[method], batch=batch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows, clusters = sc.screen(dev, dg, lambda j: ligs[j], n_ligands, runs, s, METHODS[method], batch=batch)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    evals = sum(r.evaluations for r in rows)
    out = {"workload": f"C5 virtual screen: {n_ligands} ligands (U[10,100] atoms, U[0,30] torsions) x {runs} "
                       "LGA runs vs the C4 receptor (126^3 maps), grid mode, per-ligand RMSD clustering (2 A)",
           "ligands_per_hour": sc.ligands_per_hour(n_ligands, dt), "seconds": dt, "evals_per_s": evals / dt,
           "timing": f"one full pass after a {2 * batch}-ligand warm-up pass", "batch": batch,
           "evaluations": evals, "mean_clusters": float(np.mean([c[1] for c in clusters.values()])),
           "api": "screen.screen -> mdr_grid_screen_batch (host ligands in, CSV rows out)", "warmup": len(warm[0]),
           "n_gpus": 1, "sharding": "8 GPUs: ligand j on rank j % 8, rank-0 gather of the rows (screen.py)"}
    dg.free()
    dev.close()
    return out


def score_throughput(lib, torch, local, n=1 << 20, reps=5):
    """Raw score+gradient kernel throughput at full occupancy: n independent
    random C3 poses (analytic, FP64-fast) and C4 poses (grid mode) per launch,
    device resident, CUDA events, L2 flushed before each launch.  This is the
    K3 kernel alone (no search), so it fills the GPU unlike a 100-run docking."""
    from paper_2410_10447_b200 import Device
    from paper_2410_10447_b200.workloads import c4

    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    out = {}
    dev = Device(local)
    dev.set_stream(stream.cuda_stream)

    def timed(call):
        call()
        torch.cuda.synchronize()
        ms = []
        for k in range(reps):
            flush.fill_(float(k))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            call()
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        return statistics.median(ms)

    gen = torch.Generator(device=f"cuda:{local}").manual_seed(7)
    for name, (inst, grid_case) in {"c3_analytic": (workload(), None), "c4_grid": (None, c4())}.items():
        if grid_case is None:
            di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
            dg = None
            part, method = 64, BASELINE
        else:
            inst, params, fields, grid, settings = grid_case
            dg = lib.mdr_grid_build(dev.ctx, inst.cref(), fields.cref(), grid.cref())
            di = lib.mdr_instance_upload(dev.ctx, C.byref(inst.c()))
            assert lib.mdr_instance_set_grid(dev.ctx, di, dg, params.cref()) == 0
            part, method = settings.partition, BASELINE
        m = n if grid_case is None else n // 4
        g = torch.empty((m, inst.dim), dtype=torch.float64, device=f"cuda:{local}")
        g[:, :3].uniform_(-3.0, 3.0, generator=gen)
        g[:, 3:].uniform_(-math.pi, math.pi, generator=gen)
        e = torch.empty(m, dtype=torch.float32, device=f"cuda:{local}")
        gr = torch.empty((m, inst.dim), dtype=torch.float32, device=f"cuda:{local}")
        tq = torch.empty((m, 3), dtype=torch.float32, device=f"cuda:{local}")

        def call():
            rc = lib.mdr_score_dev(dev.ctx, di, C.c_void_p(g.data_ptr()), m, method, SINGLE, part,
                                   C.c_void_p(e.data_ptr()), C.c_void_p(gr.data_ptr()), C.c_void_p(tq.data_ptr()))
            assert rc == 0, lib.mdr_last_error(dev.ctx)

        ms = timed(call)
        rec = {"poses_per_launch": m, "ms_per_launch": ms, "evals_per_s": m / (ms * 1e-3)}
        if grid_case is None:
            fl = flop_per_eval(inst, part)
            rec.update({"flop_per_eval": fl, "fp64_TFLOPs": fl * m / (ms * 1e-3) / 1e12,
                        "fp64_frac_of_peak": fl * m / (ms * 1e-3) / 1e12 / fp64_peak_tflops(torch)})
        else:
            fl, nb, _ = grid_flop_bytes_per_eval(inst, params, part)
            rec.update({"flop_per_eval": fl, "map_bytes_per_eval": nb, "fp32_TFLOPs": fl * m / (ms * 1e-3) / 1e12,
                        "map_GBps": nb * m / (ms * 1e-3) / 1e9})
        out[name] = rec
        lib.mdr_instance_free(dev.ctx, di)
        if dg:
            lib.mdr_grid_free(dev.ctx, dg)
    dev.close()
    return out


def extra_measurements(args, dev, lib, torch):
    """Mode sweep of the docking step, C4 grid-mode docking, C2 reduction
    microbench (ns/call)."""
    out = {"modes": mode_sweep(lib, torch, torch.cuda.current_device(), workload(), LgaSettings())}
    out["score_kernel"] = score_throughput(lib, torch, torch.cuda.current_device())
    out["c4_analytic"] = c4_analytic_measure(lib, torch, torch.cuda.current_device(),
                                             cpu_seconds=0.0 if args.no_cpu else args.cpu_seconds)
    out["c4_grid"] = c4_measure(lib, torch, torch.cuda.current_device())
    out["c5_screen"] = c5_measure(torch, torch.cuda.current_device())
    if hasattr(lib, "mdr_reduce_bench_dev"):
        from paper_2410_10447_b200.microbench import cpu_leg, reduce_microbench

        mb = reduce_microbench(dev, lib, torch)
        if not args.no_cpu:
            mb["cpu_leg"] = cpu_leg()
        out["reduce_microbench"] = mb
        out["c2_float4_block_reduce"] = c2_summary(mb)
    return out


def c2_summary(mb):
    """BASELINE.json metric "float4 block-reduce ns/call" (configs[1]) per
    block size: the fastest fp32-accurate shuffle kernel, the paper's f16
    MMA, the error-compensated MMAs (warp mma.sync and the batched tcgen05
    contraction the library routes TcuSplit batches to), and the reference
    library on this host's CPU (one core, and all cores)."""
    out = {"unit": "ns/call", "timing": "GPU: 10^6 reductions per launch (ns per reduction of the whole GPU); "
                                        "latency: clock64 cycles per dependent step of one block", "blocks": {}}
    for B, res in mb["results"].items():
        row = {}
        for k in ("shuffle_2level (K1c)", "wmma_f16 (paper, K2)", "split_tf32_warp (K2s)",
                  "tcgen05_batched_tf32x2 (K2t)"):
            r = res.get(k, {})
            row[k] = {"chain_ns": r.get("chain_ns"), "stream_ns": r.get("stream_ns"),
                      "latency_ns_per_step": (r.get("latency") or {}).get("ns_per_step"),
                      "chain_smem_frac": (r.get("chain_roofline") or {}).get("frac"),
                      "stream_hbm_frac": (r.get("stream_roofline") or {}).get("frac")}
        prod = mb.get("product", {}).get(B, {})
        row["library reduce4 TcuSplit"] = prod.get("reduce4 TcuSplit (tcgen05 route)")
        cpu = mb.get("cpu_leg", {}).get("results", {}).get(B, {})
        if cpu:
            row["cpu reference reduce4 Tcu f16"] = cpu.get("reduce4 Tcu f16 (Half)")
            row["cpu reference simulate_block Baseline"] = cpu.get("simulate_block Baseline (4 block trees)")
        out["blocks"][B] = row
    cpu = mb.get("cpu_leg", {})
    if cpu.get("cores"):
        out["cpu"] = {"cores": cpu["cores"], "model": cpu.get("cpu_model"), "kind": cpu.get("kind")}
    return out


def launch_plan(gpus: int, env, device_count: int, impl: str = "b200"):
    """How `bench.py --gpus N` runs: ("rank", W) when already one rank of a
    torchrun job of W processes (W must equal N), ("direct", 1) for N = 1,
    ("spawn", N) to re-launch itself as N ranks (one process per GPU).
    Raises when the request cannot be met (never silently runs on fewer GPUs)."""
    if gpus < 1:
        raise SystemExit(f"--gpus must be >= 1 (got {gpus})")
    if "WORLD_SIZE" in env:
        world = int(env["WORLD_SIZE"])
        if world != gpus:
            raise SystemExit(f"--gpus {gpus} but this torchrun job has WORLD_SIZE={world}")
        if impl == "b200" and device_count < world:
            raise SystemExit(f"WORLD_SIZE={world} ranks but only {device_count} visible GPU(s)")
        return ("rank", world)
    if gpus == 1 or impl != "b200":  # the CPU reference arm runs once, on the host
        return ("direct", 1)
    if device_count < gpus:
        raise SystemExit(f"--gpus {gpus} requested but only {device_count} visible GPU(s)")
    return ("spawn", gpus)


def spawn_ranks(n: int) -> int:
    """Re-run this script as n ranks (torch.distributed.run, one process
    per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--method", default="baseline", choices=list(METHODS))
    ap.add_argument("--pair", default="fp64fast", choices=["fp64", "fp64fast", "fp32"],
                    help="pair-term arithmetic (library default fp64fast; fp64 = reference op order)")
    ap.add_argument("--wpb", type=int, default=2)
    ap.add_argument("--cta-warps", type=int, default=None, help="warps per pose in fast modes (0 = warp per pose)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--extra", action="store_true", default=True)
    ap.add_argument("--no-extra", dest="extra", action="store_false")
    args = ap.parse_args()
    if args.impl == "b200":
        import torch

        ndev = torch.cuda.device_count()
    else:
        ndev = 0
    mode, _ = launch_plan(args.gpus, os.environ, ndev, args.impl)
    if mode == "spawn":
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_gpu_arm(args)


if __name__ == "__main__":
    main()
