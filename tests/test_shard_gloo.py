"""Multi-process sharding of independent LGA runs (world_size 2, gloo on CPU):
the round-robin shard covers every seed exactly once and the rank-0 best-pose
gather reproduces the single-process result bit for bit.  The docking itself
is the CPU oracle here (test infrastructure); on GPUs it is the B200 library."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2410_10447_b200.shard import RunResult, best_pose, dock_sharded, shard_indices


def test_shard_indices_partition():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            parts = [shard_indices(n, world, r) for r in range(world)]
            allidx = np.sort(np.concatenate(parts)) if parts else np.array([])
            assert np.array_equal(allidx, np.arange(n))
            sizes = [p.size for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_indices(4, 2, 2)


def _oracle_dock(inst, method, accum, settings, seeds):
    from oracle.oracle import Oracle

    o = Oracle("port")
    out = []
    for s in seeds:
        r = o.lga_run(inst, method, accum, settings, int(s))
        out.append(RunResult(int(s), r["best_energy"], r["evaluations"], r["converged"], r["best_genotype"]))
    return out


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import json

    from paper_2410_10447_b200 import BASELINE, SINGLE, LgaSettings
    from paper_2410_10447_b200._abi import Instance

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "instances.json")) as f:
        raw = json.load(f)["s1"]
    inst = Instance(np.array(raw["atoms"]), np.array(raw["torsion"]), np.array(raw["sites"]), raw["n_rot"])
    s = LgaSettings(population_size=8, generations=3, ls_max_iters=30)
    res = dock_sharded(inst, np.arange(7, dtype=np.uint64) + np.uint64(500), BASELINE, SINGLE, s, dist=dist,
                       dock_fn=_oracle_dock)
    if rank == 0:
        q.put([(r.seed, r.best_energy, r.evaluations, r.converged, r.best_genotype.tolist()) for r in res])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_dock_sharded_gloo_world2_matches_single_process(instances):
    from paper_2410_10447_b200 import BASELINE, SINGLE, LgaSettings

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = LgaSettings(population_size=8, generations=3, ls_max_iters=30)
    want = dock_sharded(instances["s1"], np.arange(7, dtype=np.uint64) + np.uint64(500), BASELINE, SINGLE, s,
                        dock_fn=_oracle_dock)
    assert [g[0] for g in got] == [w.seed for w in want] == list(range(500, 507))
    for g, w in zip(got, want):
        assert g[1] == w.best_energy and g[2] == w.evaluations and g[3] == w.converged
        assert g[4] == w.best_genotype.tolist()
    assert best_pose(want).best_energy == min(w.best_energy for w in want)


BIG_SEEDS = np.array([2**63 + 5, 2**63 + 4, 500, 2**64 - 1, 2**53 + 1, 2**53, 7], dtype=np.uint64)


def _fake_dock(inst, method, accum, settings, seeds):
    """Deterministic per-seed stand-in (tests the packing/gather only)."""
    return [RunResult(int(s), -float(int(s) % 1000), int(s) % 97, bool(int(s) & 1), np.full(inst.dim, float(int(s) % 13)))
            for s in seeds]


def test_pack_unpack_keeps_every_uint64_seed(instances):
    from paper_2410_10447_b200.shard import pack_results, sort_by_seed, unpack_results

    res = _fake_dock(instances["s1"], None, None, None, BIG_SEEDS)
    back = unpack_results(sort_by_seed(pack_results(res, instances["s1"].dim)))
    assert [r.seed for r in back] == sorted(int(s) for s in BIG_SEEDS)
    assert len({r.seed for r in back}) == BIG_SEEDS.size


def _big_worker(rank, world, port, q):
    import json
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2410_10447_b200._abi import Instance

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "instances.json")) as f:
        raw = json.load(f)["s1"]
    inst = Instance(np.array(raw["atoms"]), np.array(raw["torsion"]), np.array(raw["sites"]), raw["n_rot"])
    res = dock_sharded(inst, BIG_SEEDS, None, None, None, dist=dist, dock_fn=_fake_dock)
    if rank == 0:
        q.put([(r.seed, r.best_energy, r.evaluations) for r in res])
    dist.destroy_process_group()


def test_gather_world2_keeps_large_seeds():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_big_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [g[0] for g in got] == sorted(int(s) for s in BIG_SEEDS)
    for sd, e, ev in got:
        assert e == -float(sd % 1000) and ev == sd % 97
