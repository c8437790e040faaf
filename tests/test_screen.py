"""Virtual-screen driver.

CPU: the results CSV is byte-identical to the reference's write_results
(oracle/_ref), parse/write round-trips, and the sharded driver (gloo, world 2)
with skip-done resume gathers exactly the single-process rows.
GPU: one mdr_grid_screen_batch launch sequence over many ligands gives every
ligand exactly the result of its own single-ligand docking (same kernels,
same draws), and its per-ligand clustering equals the oracle's."""
import os
import tempfile

import numpy as np
import pytest

from paper_2410_10447_b200 import screen as sc
from paper_2410_10447_b200._abi import LgaSettings, derive_rng


def _rows(n, seed=1):
    rng = derive_rng(seed, "screen/rows")
    names = ["synth/lig/0", 'odd,"name"', "plain", "with\nnewline"]
    return [sc.ResultRow(rng.next_u64(), ["baseline", "tcu"][rng.next_index(2)], "single",
                         names[rng.next_index(len(names))], rng.uniform(-50, 5) * 10 ** rng.next_index(4),
                         int(rng.next_index(30000)), bool(rng.next_index(2)), rng.next_index(10**6), 0,
                         rng.next_index(1000)) for _ in range(n)]


_REF_WRITE = r"""
import ctypes as C, json, sys
rows = json.load(sys.stdin)
n = len(rows)
lib = C.CDLL(sys.argv[1])
f = lib.ref_write_results
P = C.c_void_p
f.argtypes = [C.c_int] + [P] * 10 + [P, C.c_size_t, P]
f.restype = C.c_int
col = lambda k: [r[k] for r in rows]
out = C.create_string_buffer(1 << 16)
ln = C.c_size_t()
strs = [(C.c_char_p * n)(*[x.encode() for x in col(k)]) for k in ("method", "accum_mode", "instance")]
rc = f(n, (C.c_uint64 * n)(*col("seed")), *strs, (C.c_double * n)(*col("best_energy")),
       (C.c_int64 * n)(*col("evaluations")), (C.c_int32 * n)(*[int(x) for x in col("converged")]),
       (C.c_uint64 * n)(*col("block_syncs")), (C.c_uint64 * n)(*col("atomic_adds")),
       (C.c_uint64 * n)(*col("mma_ops")), out, C.sizeof(out), C.byref(ln))
assert rc == 0
sys.stdout.write(out.raw[: ln.value].decode())
"""


def test_write_results_matches_reference(ref):
    """Byte-identical to the reference's write_results.  The reference call
    runs in a numpy-free interpreter: with numpy's runtime loaded in the same
    process the reference's ostringstream path segfaults (reproduced only
    under CPython + numpy; a plain C caller and a numpy-free CPython work)."""
    import dataclasses
    import json
    import subprocess
    import sys

    from oracle.oracle import REF_SO

    rows = _rows(40)
    p = subprocess.run([sys.executable, "-c", _REF_WRITE, REF_SO], input=json.dumps(
        [dataclasses.asdict(r) for r in rows]), capture_output=True, text=True, check=True)
    assert sc.write_results(rows) == p.stdout


def test_results_roundtrip():
    rows = [r for r in _rows(30) if "\n" not in r.instance]  # one record per line in this parser
    assert sc.parse_results(sc.write_results(rows)) == rows


class FakeDev:
    """Deterministic stand-in for Device.grid_screen_batch (host-logic tests)."""

    def grid_screen_batch(self, dgrid, ligs, params, runs, method, settings, seeds, tol):
        out = []
        s = np.asarray(seeds, np.uint64).reshape(len(ligs), runs)
        for lig, row in zip(ligs, s):
            out.append(dict(best_energy=-(row % 97).astype(float) / 7.0, evaluations=(row % 1000).astype(np.int64) + 5,
                            converged=(row % 2).astype(bool), cluster_of=np.zeros(runs, np.int32),
                            rmsd_to_seed=np.zeros(runs), n_clusters=1))
        return out


def _lig(j):
    return (j, None)


def test_screen_resume_skips_done():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "res.csv")
        s = LgaSettings(partition=64)
        rows1, _ = sc.screen(FakeDev(), None, _lig, 10, 3, s, batch=4, csv_path=path)
        assert len(rows1) == 30
        rows2, _ = sc.screen(FakeDev(), None, _lig, 12, 3, s, batch=4, csv_path=path)
        assert len(rows2) == 6  # only ligands 10 and 11 are new
        with open(path) as f:
            got = sc.parse_results(f.read())
        assert sorted(got, key=lambda r: (r.instance, r.seed)) == sc.gather_rows(rows1 + rows2, 0, 1)


def test_screen_resume_after_partial_line_and_repeated_header():
    """A crash mid-append leaves a partial last record; a concatenated file
    can carry a second header.  Resume must drop the partial record (and
    redo that run), skip the header, and leave a file parse_results reads."""
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "res.csv")
        s = LgaSettings(partition=64)
        rows1, _ = sc.screen(FakeDev(), None, _lig, 4, 3, s, batch=2, csv_path=path)
        with open(path) as f:
            text = f.read()
        lines = text.splitlines()
        # drop the last full record, append its first half without newline
        broken = "\n".join(lines[:-1]) + "\n" + sc.HEADER + "\n" + lines[-1][: len(lines[-1]) // 2]
        with open(path, "w") as f:
            f.write(broken)
        rows2, _ = sc.screen(FakeDev(), None, _lig, 4, 3, s, batch=2, csv_path=path)
        assert len(rows2) == 3  # ligand 3 (whose last run was torn) is redone
        with open(path) as f:
            body = [ln for i, ln in enumerate(f.read().splitlines()) if not (ln == sc.HEADER and i > 0)]
        got = sc.parse_results("\n".join(body) + "\n")
        keys = sorted((r.instance, r.seed) for r in got)
        assert len(set(keys)) == 12 and len(keys) == 14  # runs of ligand 3 written twice, once torn-free
        rows3, _ = sc.screen(FakeDev(), None, _lig, 4, 3, s, batch=2, csv_path=path)
        assert rows3 == []


def test_screen_ranks_write_separate_files():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "res.csv")
        s = LgaSettings(partition=64)
        for r in range(2):
            sc.screen(FakeDev(), None, _lig, 5, 2, s, batch=2, csv_path=path, rank=r, world=2)
        assert not os.path.exists(path)
        n = 0
        for r in range(2):
            with open(f"{path}.rank{r}") as f:
                n += len(sc.parse_results(f.read()))
        assert n == 10


def _worker(rank, world, port, out):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rows, _ = sc.screen(FakeDev(), None, _lig, 11, 3, LgaSettings(partition=64), batch=2, rank=rank, world=world)
    merged = sc.gather_rows(rows, rank, world)
    if rank == 0:
        with open(out, "w") as f:
            f.write(sc.write_results(merged))
    dist.destroy_process_group()


def test_screen_sharded_gloo_world2_matches_single_process():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "merged.csv")
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        single, _ = sc.screen(FakeDev(), None, _lig, 11, 3, LgaSettings(partition=64), batch=5)
        with open(out) as f:
            assert f.read() == sc.write_results(sc.gather_rows(single, 0, 1))


@pytest.mark.gpu
def test_screen_batch_equals_single_ligand_dockings(port, dev):
    from paper_2410_10447_b200 import BASELINE
    from paper_2410_10447_b200.workloads import c4_receptor, c5_ligand

    sites, fields, _ = c4_receptor()
    from paper_2410_10447_b200._abi import centered_grid

    G = centered_grid(41, 0.375, 4)
    G.maps = port.grid_build(sites, fields, G)
    dg = dev.grid_upload(G)
    ligs, params = zip(*[c5_ligand(j, sites) for j in range(6)])
    # include rigid ligands: n_rot = 0, and n_rot > 0 with no torsioned atom
    from paper_2410_10447_b200._abi import Instance, random_ligand_params

    rigid = Instance(ligs[0].atoms[:7], np.full(7, -1), sites.sites, 0, "rigid")
    untors = Instance(ligs[1].atoms[:9], np.full(9, -1), sites.sites, 3, "untorsioned")
    ligs = ligs + (rigid, untors)
    params = params + tuple(random_ligand_params(derive_rng(9, f"rigid/{k}"), l.n_atoms, 4)
                            for k, l in enumerate((rigid, untors)))
    runs = 4
    s = LgaSettings(generations=3, partition=64)
    seeds = np.array([sc.run_seed(7, j, k, runs) for j in range(len(ligs)) for k in range(runs)], np.uint64)
    res = dev.grid_screen_batch(dg, list(ligs), list(params), runs, BASELINE, s, seeds, 1.5)
    for j, (lig, prm) in enumerate(zip(ligs, params)):
        one = dev.grid_lga_run_batch(dg, lig, prm, BASELINE, s, seeds[j * runs:(j + 1) * runs])
        assert np.array_equal(res[j]["best_energy"], np.array([r.best_energy for r in one]))
        assert np.array_equal(res[j]["evaluations"], np.array([r.evaluations for r in one]))
        assert np.array_equal(res[j]["best_genotype"], np.stack([r.best_genotype for r in one]))
        wc, wr, wnc = port.cluster_poses(lig, res[j]["best_genotype"], res[j]["best_energy"], 1.5)
        assert res[j]["n_clusters"] == wnc and np.array_equal(res[j]["cluster_of"], wc)
        assert np.abs(res[j]["rmsd_to_seed"] - wr).max() <= 1e-9
