"""Virtual-screen driver (BASELINE.json configs[4] "C5"):
many ligands against one receptor, sharded over the GPUs of a node.

Host-side orchestration only; the docking itself is one launch sequence per
batch of ligands through `mdr_grid_screen_batch` (grid-mode LGA + per-ligand
RMSD clustering on the device).

  * sharding: ligand j goes to rank j % world (independent units, no
    data-path collective);
  * results: the reference's results CSV (write_results,
    reference proj/src/instance_io.cpp:277-287: header
    `seed,method,accum_mode,instance,best_energy,evaluations,converged,
    block_syncs,atomic_adds,mma_ops`, %.17g numbers, RFC-4180 quoting), one
    row per docking run, appended after every batch;
  * resume: ligands whose every run already has a row are skipped
    (keyed on (instance, seed)); a crash can leave at most a partial last
    line, which the loader drops (and trims from the file) before appending;
    with world > 1 every rank writes its own file `<csv_path>.rank<r>`, so
    ranks never interleave lines;
  * gather: the only collective — every rank's rows to rank 0
    (torch.distributed.gather_object), which writes the merged CSV ordered
    by (instance, seed).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

HEADER = "seed,method,accum_mode,instance,best_energy,evaluations,converged,block_syncs,atomic_adds,mma_ops"
METHOD_NAMES = {0: "baseline", 1: "tcu", 2: "tcu_split"}


@dataclass(frozen=True)
class ResultRow:
    """ResultRow reference include/mdreduce/instance_io.hpp:52-65."""

    seed: int
    method: str
    accum_mode: str
    instance: str
    best_energy: float
    evaluations: int
    converged: bool
    block_syncs: int = 0
    atomic_adds: int = 0
    mma_ops: int = 0


def _field(s: str) -> str:
    if any(c in s for c in ',"\n'):
        return '"' + s.replace('"', '""') + '"'
    return s


def format_double(v: float) -> str:
    """format_double instance_io.cpp:67-71 (printf %.17g)."""
    return "%.17g" % v


def write_results(rows) -> str:
    """write_results instance_io.cpp:277-287."""
    out = [HEADER]
    for r in rows:
        out.append(f"{r.seed},{_field(r.method)},{_field(r.accum_mode)},{_field(r.instance)},"
                   f"{format_double(r.best_energy)},{r.evaluations},{'true' if r.converged else 'false'},"
                   f"{r.block_syncs},{r.atomic_adds},{r.mma_ops}")
    return "\n".join(out) + "\n"


def _split(record: str):
    fields, cur, quoted, i = [], [], False, 0
    while i < len(record):
        c = record[i]
        if quoted:
            if c == '"':
                if i + 1 < len(record) and record[i + 1] == '"':
                    cur.append('"')
                    i += 1
                else:
                    quoted = False
            else:
                cur.append(c)
        elif c == '"':
            quoted = True
        elif c == ",":
            fields.append("".join(cur))
            cur = []
        else:
            cur.append(c)
        i += 1
    fields.append("".join(cur))
    return fields


def parse_results(text: str):
    """parse_results instance_io.cpp:289-353 (well-formed input)."""
    rows, header = [], False
    for line in text.splitlines():
        if not line:
            continue
        if not header:
            if line != HEADER:
                raise ValueError("unexpected results header")
            header = True
            continue
        f = _split(line)
        if len(f) != 10:
            raise ValueError(f"expected 10 fields, got {len(f)}")
        rows.append(ResultRow(int(f[0]), f[1], f[2], f[3], float(f[4]), int(f[5]), f[6] == "true", int(f[7]),
                              int(f[8]), int(f[9])))
    return rows


def load_done_rows(path: str):
    """Rows of a results CSV being resumed.  Repeated header lines are
    skipped and a trailing partial record (no final newline, or a bad field
    count on the last line — a crash mid-append) is dropped and trimmed from
    the file, so the next append starts on a clean line.  Damage anywhere
    else still raises (parse_results)."""
    with open(path) as f:
        text = f.read()
    lines = text.split("\n")
    tail = lines.pop()  # "" when the file ends with a newline
    if tail:
        text = text[: len(text) - len(tail)]
    if lines and lines[-1] != HEADER and len(_split(lines[-1])) != 10:
        text = text[: len(text) - len(lines[-1]) - 1]
        lines.pop()
    if len(text) != os.path.getsize(path):
        tmp = path + ".tmp"
        with open(tmp, "w") as f:
            f.write(text)
        os.replace(tmp, path)
    body = [ln for i, ln in enumerate(lines) if ln and not (ln == HEADER and i > 0)]
    return parse_results("\n".join(body) + "\n") if body else []


def _append(path: str, block: str):
    """One write + fsync per batch: a crash loses at most the last batch's
    tail, which load_done_rows trims."""
    with open(path, "a") as f:
        f.write(block)
        f.flush()
        os.fsync(f.fileno())


def run_seed(base_seed: int, ligand: int, run: int, runs: int) -> int:
    """Seed of run k of ligand j (validate_pair-style base + offset,
    reference docking.cpp:562)."""
    return base_seed + ligand * runs + run


def shard(n_ligands: int, rank: int, world: int):
    return list(range(rank, n_ligands, world))


def pending(ligand_ids, names, runs, base_seed, done_keys):
    """Ligands with at least one (instance, seed) row missing."""
    out = []
    for j in ligand_ids:
        keys = {(names[j], run_seed(base_seed, j, k, runs)) for k in range(runs)}
        if not keys <= done_keys:
            out.append(j)
    return out


def reduction_counters(method: int, evaluations: int, partition: int):
    """Per-run (block_syncs, atomic_adds, mma_ops) of the grid kernels:
    3 CTA barriers per evaluation, no atomics; the MMA methods issue 2 (f16)
    or 4 (tf32 hi/lo) tensor-core instructions per warp per evaluation."""
    warps = partition // 32
    mma = {0: 0, 1: 4, 2: 4}[method] * warps
    return 3 * evaluations, 0, mma * evaluations


def screen(dev, dgrid, ligand_fn, n_ligands: int, runs: int, settings, method: int = 0, base_seed: int = 12345,
           batch: int = 1024, csv_path: str | None = None, rmsd_tol: float = 2.0, rank: int = 0, world: int = 1,
           names=None):
    """Dock this rank's shard of ligands 0..n_ligands-1 (ligand_fn(j) ->
    (Instance, LigandParams)); returns (rows, clusters) of the newly docked
    runs.  With csv_path, rows are appended after each batch and ligands
    already complete in the file are skipped.  `batch` ligands share one
    launch sequence: C5 (10 runs each) measured 1.52 / 1.67 / 1.71 / 1.73 M
    ligands/hour at 256 / 512 / 1024 / 2048 (larger batches fill the last
    wave of CTA-per-pose searches better; tools/c5_batch_probe.py)."""
    names = names or [f"synth/lig/{j}" for j in range(n_ligands)]
    mine = shard(n_ligands, rank, world)
    done = set()
    if csv_path and world > 1:
        csv_path = f"{csv_path}.rank{rank}"
    if csv_path and os.path.exists(csv_path):
        done = {(r.instance, r.seed) for r in load_done_rows(csv_path)}
    todo = pending(mine, names, runs, base_seed, done)
    rows, clusters = [], {}
    if csv_path and (not os.path.exists(csv_path) or os.path.getsize(csv_path) == 0):
        _append(csv_path, HEADER + "\n")
    mname = METHOD_NAMES[method]
    for b0 in range(0, len(todo), batch):
        ids = todo[b0:b0 + batch]
        ligs, params = zip(*[ligand_fn(j) for j in ids])
        seeds = np.array([run_seed(base_seed, j, k, runs) for j in ids for k in range(runs)], np.uint64)
        res = dev.grid_screen_batch(dgrid, list(ligs), list(params), runs, method, settings, seeds, rmsd_tol)
        new = []
        for j, r in zip(ids, res):
            for k in range(runs):
                bs, aa, mm = reduction_counters(method, int(r["evaluations"][k]), settings.partition)
                new.append(ResultRow(run_seed(base_seed, j, k, runs), mname, "single", names[j],
                                     float(r["best_energy"][k]), int(r["evaluations"][k]), bool(r["converged"][k]),
                                     bs, aa, mm))
            clusters[names[j]] = (r["cluster_of"].tolist(), r["n_clusters"])
        rows += new
        if csv_path:
            _append(csv_path, write_results(new).split("\n", 1)[1])
    return rows, clusters


def gather_rows(rows, rank: int, world: int):
    """Final gather (the only collective): rank 0 receives every rank's rows,
    ordered by (instance, seed)."""
    if world == 1:
        return sorted(rows, key=lambda r: (r.instance, r.seed))
    import torch.distributed as dist

    bucket = [None] * world if rank == 0 else None
    dist.gather_object(rows, bucket, dst=0)
    if rank != 0:
        return None
    return sorted((r for part in bucket for r in part), key=lambda r: (r.instance, r.seed))


def ligands_per_hour(n: int, seconds: float) -> float:
    return n / seconds * 3600.0 if seconds > 0 else math.inf
