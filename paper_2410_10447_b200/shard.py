"""Multi-GPU host driver: independent LGA runs (and ligands) sharded across
the GPUs of one box, one process per GPU (torchrun), no data-path
collective — only the final best-pose gather.

Runs are independent given (instance, settings, seed) (validate_pair seeds
base + i, reference docking.cpp:558-564), so run i goes to rank i % world and
results are merged by seed (order independent).  The gather moves, per run,
{seed, best_energy, evaluations, converged, best_genotype} (<= 0.3 KB) to
rank 0 over the process group (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_indices(n: int, world: int, rank: int) -> np.ndarray:
    """Round-robin shard: item i belongs to rank i % world (equal-cost runs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return np.arange(rank, n, world, dtype=np.int64)


@dataclass
class RunResult:
    seed: int
    best_energy: float
    evaluations: int
    converged: bool
    best_genotype: np.ndarray


def pack_results(results, dim: int) -> np.ndarray:
    """Flatten RunResults into one float64 array: [seed, E, evals, conv, g...].
    The seed column holds the uint64 seed's BITS (viewed as float64, never
    converted), so every seed the reference accepts (any uint64, cli.cpp
    --seed) survives the gather exactly; sorting uses the uint64 view."""
    out = np.zeros((len(results), 4 + dim), np.float64)
    seeds = np.array([int(r.seed) for r in results], dtype=np.uint64)
    out[:, 0] = seeds.view(np.float64)
    for k, r in enumerate(results):
        out[k, 1] = r.best_energy
        out[k, 2] = float(r.evaluations)
        out[k, 3] = 1.0 if r.converged else 0.0
        out[k, 4:] = r.best_genotype
    return out


def seed_column(arr: np.ndarray) -> np.ndarray:
    """The uint64 seeds of packed rows (bit view of column 0)."""
    return np.ascontiguousarray(arr[:, 0]).view(np.uint64)


def sort_by_seed(arr: np.ndarray) -> np.ndarray:
    return arr[np.argsort(seed_column(arr), kind="stable")]


def unpack_results(arr: np.ndarray):
    seeds = seed_column(arr) if len(arr) else np.zeros(0, np.uint64)
    return [RunResult(int(sd), float(row[1]), int(row[2]), bool(row[3]), row[4:].copy())
            for sd, row in zip(seeds, arr)]


def gather_to_rank0(local: np.ndarray, dist, device=None):
    """Best-pose gather: variable-length float64 blocks from every rank to
    rank 0 (all_gather of sizes, then padded all_gather), merged by seed."""
    import torch

    world = dist.get_world_size()
    t = torch.from_numpy(np.ascontiguousarray(local, np.float64))
    if device is not None:
        t = t.to(device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((cap, local.shape[1]), dtype=torch.float64, device=t.device)
    pad[: t.shape[0]] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    if dist.get_rank() != 0:
        return None
    rows = np.concatenate([b[: int(s.item())].cpu().numpy() for b, s in zip(bufs, sizes)], axis=0)
    return sort_by_seed(rows)


def dock_sharded(inst, seeds, method, accum, settings, dist=None, device=None, dock_fn=None):
    """Dock `seeds` across the process group.  dock_fn(inst, method, accum,
    settings, seeds) -> list[RunResult]; default: the B200 library on this
    rank's GPU.  Returns the merged results on rank 0 (None elsewhere)."""
    seeds = np.asarray(seeds, np.uint64)
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    mine = seeds[shard_indices(seeds.size, world, rank)]
    if dock_fn is None:
        from . import Device

        dev = Device(rank if device is None else device)

        def dock_fn(i, m, a, s, sd):
            return [RunResult(int(x), r.best_energy, r.evaluations, r.converged, r.best_genotype)
                    for x, r in zip(sd, dev.lga_run_batch(i, m, a, s, sd))]

    local = dock_fn(inst, method, accum, settings, mine) if mine.size else []
    packed = pack_results(local, inst.dim)
    if dist is None:
        return unpack_results(sort_by_seed(packed))
    rows = gather_to_rank0(packed, dist, device)
    return None if rows is None else unpack_results(rows)


def best_pose(results):
    """Lowest best_energy over runs; ties -> smallest seed (deterministic)."""
    return min(results, key=lambda r: (r.best_energy, r.seed))
