"""Python host mirror of the reference operator API (namespace `mdreduce`,
reference proj/include/mdreduce/*.hpp) over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference (errors are
raised before any work with the reference's exception taxonomy), plus
`*_batch` variants that put many independent calls into one launch.  Every
call runs on the GPU through libmdr_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._abi import (
    BASELINE,
    HALF,
    PAIR_FP64_FAST,
    SINGLE,
    TCU,
    TCU_SPLIT,
    Grid,
    Instance,
    LgaSettings,
    LigandParams,
    ReceptorFields,
    LsRecord,
    SizeError,
    SyncStats,
    raise_for,
)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class ScoreResult:
    """ScoreResult docking.hpp:44-49."""

    energy: np.float32
    gradient: np.ndarray  # float32[dim]
    torque: np.ndarray  # float32[3]
    reduce_stats: SyncStats


@dataclass
class LocalSearchResult:
    """LocalSearchResult docking.hpp:86-94."""

    genotype: np.ndarray
    energy: float
    iterations: int
    converged: bool
    stats: SyncStats


@dataclass
class DockResult:
    """DockResult docking.hpp:125-134."""

    best_energy: float
    best_genotype: np.ndarray
    evaluations: int
    converged: bool
    runs: list = field(default_factory=list)  # (best_energy, iterations, converged)
    total_stats: SyncStats = field(default_factory=SyncStats)


class Device:
    """One mdr context on one GPU (one CUDA stream)."""

    def __init__(self, device: int = 0, pair: int = PAIR_FP64_FAST, warps_per_block: int = 2):
        self.lib = _lib.load()
        self.ctx = self.lib.mdr_ctx_create(device)
        if not self.ctx:
            raise RuntimeError(f"mdr_ctx_create({device}) failed: no usable CUDA device")
        self.set_pair_precision(pair)
        self._chk(self.lib.mdr_ctx_set_warps_per_block(self.ctx, warps_per_block))

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mdr_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        if rc:
            raise_for(rc, self.lib.mdr_last_error(self.ctx).decode())

    def set_pair_precision(self, pair: int):
        self._chk(self.lib.mdr_ctx_set_pair_precision(self.ctx, pair))

    def set_exact_torsion(self, on: bool):
        """Analytic-mode torsion gradient: False (default) projects the total
        torque on every torsion axis (score(), docking.cpp:228-231); True
        gives each torsion its own group's torque, the exact gradient of
        score_reference() (docking.cpp:244-268).  See mdr_ctx_set_exact_torsion."""
        self._chk(self.lib.mdr_ctx_set_exact_torsion(self.ctx, 1 if on else 0))

    def set_stream(self, stream_ptr: int | None):
        self._chk(self.lib.mdr_ctx_set_stream(self.ctx, C.c_void_p(stream_ptr or 0)))

    @property
    def launches(self) -> int:
        return int(self.lib.mdr_ctx_launch_count(self.ctx))

    def synchronize(self):
        self._chk(self.lib.mdr_ctx_synchronize(self.ctx))

    # ------------------------------------------------------------ L0
    def f32_to_half(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        out = np.zeros(x.size, np.uint16)
        self._chk(self.lib.mdr_f32_to_half_batch(self.ctx, _p(x), x.size, _p(out)))
        return out

    def half_to_f32(self, h) -> np.ndarray:
        h = np.ascontiguousarray(h, np.uint16).reshape(-1)
        out = np.zeros(h.size, np.float32)
        self._chk(self.lib.mdr_half_to_f32_batch(self.ctx, _p(h), h.size, _p(out)))
        return out

    def mma_batch(self, a, b, c, accum) -> np.ndarray:
        """mma() mma.cpp:41-64 over tiles: a, b uint16 (n,16,16); c float32 (n,16,16)."""
        a = np.ascontiguousarray(a, np.uint16).reshape(-1, 256)
        b = np.ascontiguousarray(b, np.uint16).reshape(-1, 256)
        c = np.ascontiguousarray(c, np.float32).reshape(-1, 256)
        d = np.zeros_like(c)
        self._chk(self.lib.mdr_mma_batch(self.ctx, _p(a), _p(b), _p(c), a.shape[0], accum, _p(d)))
        return d.reshape(-1, 16, 16)

    def mma(self, a, b, c, accum) -> np.ndarray:
        return self.mma_batch(a, b, c, accum)[0]

    # ------------------------------------------------------------ L1
    def reduce4_batch(self, vecs, accum=HALF, method=TCU):
        """reduce4 reduce.cpp:80-111 for vecs (n_red, n, 4)."""
        v = np.ascontiguousarray(vecs, np.float32)
        if v.ndim == 2:
            v = v[None]
        n_red, n = v.shape[0], v.shape[1]
        out = np.zeros((n_red, 4), np.float32)
        st = SyncStats()
        self._chk(self.lib.mdr_reduce4_batch(self.ctx, _p(v), n, n_red, method, accum, _p(out), C.byref(st)))
        return out, st

    def reduce4(self, vecs, accum=HALF, method=TCU):
        v = np.ascontiguousarray(vecs, np.float32).reshape(-1, 4)
        if v.shape[0] == 0:
            raise SizeError("reduce4 requires at least one vector")
        out, st = self.reduce4_batch(v[None], accum, method)
        return out[0], st

    def warp_reduce_batch(self, lanes):
        v = np.ascontiguousarray(lanes, np.float32).reshape(-1, 32)
        out = np.zeros(v.shape[0], np.float32)
        st = SyncStats()
        self._chk(self.lib.mdr_warp_reduce_batch(self.ctx, _p(v), v.shape[0], _p(out), C.byref(st)))
        return out, st

    def warp_reduce(self, lanes):
        v = np.ascontiguousarray(lanes, np.float32).reshape(-1)
        if v.size != 32:
            raise SizeError(f"baseline_warp_reduce expects exactly 32 lanes, got {v.size}")
        out, st = self.warp_reduce_batch(v[None])
        return out[0], st

    def block_reduce_batch(self, values, threads):
        v = np.ascontiguousarray(values, np.float32).reshape(-1, threads) if threads > 0 else values
        out = np.zeros(v.shape[0], np.float32)
        st = SyncStats()
        self._chk(self.lib.mdr_block_reduce_batch(self.ctx, _p(v), threads, v.shape[0], _p(out), C.byref(st)))
        return out, st

    def block_reduce(self, values, threads):
        v = np.ascontiguousarray(values, np.float32).reshape(-1)
        st = SyncStats()
        out = np.zeros(1, np.float32)
        # the threads check (UnsupportedBlockSizeError) precedes the count check (SizeError)
        rc = self.lib.mdr_block_reduce_batch(self.ctx, _p(v), threads, 0, _p(out), C.byref(st))
        self._chk(rc)
        if v.size != threads:
            raise SizeError(f"baseline_block_reduce got {v.size} values for {threads} threads")
        o, st = self.block_reduce_batch(v[None], threads)
        return o[0], st

    def reduce7_batch(self, recs, method=BASELINE, accum=HALF):
        r = np.ascontiguousarray(recs, np.float32)
        if r.ndim == 2:
            r = r[None]
        out = np.zeros((r.shape[0], 7), np.float32)
        st = SyncStats()
        self._chk(self.lib.mdr_reduce7_batch(self.ctx, _p(r), r.shape[1], r.shape[0], method, accum, _p(out),
                                             C.byref(st)))
        return out, st

    def reduce7(self, recs, method=BASELINE, accum=HALF):
        out, st = self.reduce7_batch(np.ascontiguousarray(recs, np.float32).reshape(1, -1, 7), method, accum)
        return out[0], st

    # ------------------------------------------------------------ L2
    def score_batch(self, inst: Instance, genotypes, method=BASELINE, accum=SINGLE, partition=64):
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        n = g.shape[0]
        e = np.zeros(n, np.float32)
        grad = np.zeros((n, inst.dim), np.float32)
        tq = np.zeros((n, 3), np.float32)
        st = SyncStats()
        self._chk(self.lib.mdr_score_batch(self.ctx, C.byref(inst.c()), _p(g), n, method, accum, partition,
                                           _p(e), _p(grad), _p(tq), C.byref(st)))
        return e, grad, tq, st

    def score(self, inst: Instance, g, method=BASELINE, accum=SINGLE, partition=64) -> ScoreResult:
        g = np.asarray(g, np.float64).reshape(-1)
        if g.size != inst.dim:  # check_genotype docking.cpp:138-144
            raise SizeError(f"score: genotype has {g.size - 6} torsions, instance needs {inst.n_rot}")
        e, grad, tq, st = self.score_batch(inst, g[None], method, accum, partition)
        return ScoreResult(e[0], grad[0], tq[0], st)

    def score_reference_batch(self, inst: Instance, genotypes):
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        n = g.shape[0]
        e = np.zeros(n)
        grad = np.zeros((n, inst.dim))
        tq = np.zeros((n, 3))
        self._chk(self.lib.mdr_score_reference_batch(self.ctx, C.byref(inst.c()), _p(g), n, _p(e), _p(grad),
                                                     _p(tq)))
        return e, grad, tq

    def score_reference(self, inst: Instance, g):
        e, grad, tq = self.score_reference_batch(inst, np.asarray(g, np.float64)[None])
        return e[0], grad[0], tq[0]

    # ------------------------------------------------------------ L3
    def adadelta_step_batch(self, sq_g, sq_u, geno, grad, rho=0.95, eps=1e-6):
        sq_g = np.array(sq_g, np.float64, ndmin=2)
        sq_u = np.array(sq_u, np.float64, ndmin=2)
        geno = np.array(geno, np.float64, ndmin=2)
        grad = np.ascontiguousarray(np.array(grad, np.float64, ndmin=2))
        n, dim = geno.shape
        if sq_g.shape != geno.shape or sq_u.shape != geno.shape or grad.shape != geno.shape:
            raise SizeError("adadelta_step: state/gradient dimensions do not match genotype")
        self._chk(self.lib.mdr_adadelta_step_batch(self.ctx, dim, n, rho, eps, _p(sq_g), _p(sq_u), _p(geno),
                                                   _p(grad)))
        return sq_g, sq_u, geno

    def adadelta_step(self, sq_g, sq_u, geno, grad, rho=0.95, eps=1e-6):
        a, b, c = self.adadelta_step_batch(sq_g, sq_u, geno, grad, rho, eps)
        return a[0], b[0], c[0]

    def local_search_batch(self, inst: Instance, starts, max_iters, tol, method=BASELINE, accum=SINGLE,
                           partition=64):
        s = np.ascontiguousarray(starts, np.float64).reshape(-1, inst.dim)
        n = s.shape[0]
        g = np.zeros_like(s)
        e = np.zeros(n)
        it = np.zeros(n, np.int32)
        cv = np.zeros(n, np.int32)
        st = (SyncStats * max(n, 1))()
        self._chk(self.lib.mdr_local_search_batch(self.ctx, C.byref(inst.c()), _p(s), n, max_iters, tol, method,
                                                  accum, partition, _p(g), _p(e), _p(it), _p(cv), st))
        return [LocalSearchResult(g[i], float(e[i]), int(it[i]), bool(cv[i]), st[i]) for i in range(n)]

    def local_search(self, inst, start, max_iters, tol, method=BASELINE, accum=SINGLE, partition=64, rng_seed=0):
        """local_search docking.cpp:310-351 (rng_seed feeds no draws, as in the reference)."""
        return self.local_search_batch(inst, np.asarray(start)[None], max_iters, tol, method, accum, partition)[0]

    def lga_run_batch(self, inst: Instance, method, accum, settings: LgaSettings, seeds):
        seeds = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
        n = seeds.size
        maxr = settings.max_records
        be = np.zeros(n)
        bg = np.zeros((n, inst.dim))
        ev = np.zeros(n, np.int64)
        cv = np.zeros(n, np.int32)
        nr = np.zeros(n, np.int32)
        recs = (LsRecord * (n * maxr))()
        st = (SyncStats * n)()
        self._chk(self.lib.mdr_lga_run_batch(self.ctx, C.byref(inst.c()), method, accum, C.byref(settings),
                                             _p(seeds), n, _p(be), _p(bg), _p(ev), _p(cv), _p(nr), recs, st))
        out = []
        for i in range(n):
            runs = [(recs[i * maxr + k].best_energy, recs[i * maxr + k].iterations, bool(recs[i * maxr + k].converged))
                    for k in range(min(int(nr[i]), maxr))]
            out.append(DockResult(float(be[i]), bg[i], int(ev[i]), bool(cv[i]), runs, st[i]))
        return out

    def lga_run(self, inst, method, accum, settings: LgaSettings, seed: int) -> DockResult:
        return self.lga_run_batch(inst, method, accum, settings, [seed])[0]

    # ------------------------------------------------- clustering (§8 f3)
    def pose_coords(self, inst: Instance, genotypes) -> np.ndarray:
        """World coordinates of poses (evaluate_atoms' transform, docking.cpp:101-106)."""
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        xyz = np.zeros((g.shape[0], inst.n_atoms, 3))
        self._chk(self.lib.mdr_pose_coords_batch(self.ctx, inst.cref(), _p(g), g.shape[0], _p(xyz)))
        return xyz

    def cluster_poses(self, inst: Instance, genotypes, energies, rmsd_tol: float = 2.0):
        """AutoDock clustering of poses: (cluster_of, rmsd_to_seed, n_clusters)."""
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        e = np.ascontiguousarray(energies, np.float64).reshape(-1)
        n = g.shape[0]
        c = np.zeros(n, np.int32)
        r = np.zeros(n)
        nc = np.zeros(1, np.int32)
        self._chk(self.lib.mdr_cluster_poses(self.ctx, inst.cref(), _p(g), _p(e), n, rmsd_tol, _p(c), _p(r), _p(nc)))
        return c, r, int(nc[0])

    # ------------------------------------------------- grid-map mode (§8 f1)
    # include/mdr.h "grid-map scoring mode": partition = CTA threads per pose
    # (>= 6 + n_rot); accum does not apply (fp32 / tf32 reductions).
    def grid_upload(self, grid: Grid) -> DevGrid:
        h = self.lib.mdr_grid_upload(self.ctx, grid.cref())
        if not h:
            raise_for(6, self.lib.mdr_last_error(self.ctx).decode())
        return DevGrid(self, h, grid)

    def grid_build(self, sites: Instance, fields: ReceptorFields, grid: Grid) -> DevGrid:
        h = self.lib.mdr_grid_build(self.ctx, sites.cref(), fields.cref(), grid.cref())
        if not h:
            raise_for(6, self.lib.mdr_last_error(self.ctx).decode())
        return DevGrid(self, h, grid)

    def grid_score_batch(self, dgrid: DevGrid, inst: Instance, params: LigandParams, genotypes, method=BASELINE,
                         partition=64):
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        n = g.shape[0]
        e = np.zeros(n, np.float32)
        grad = np.zeros((n, inst.dim), np.float32)
        tq = np.zeros((n, 3), np.float32)
        self._chk(self.lib.mdr_grid_score_batch(self.ctx, dgrid.h, inst.cref(), params.cref(), _p(g), n, method,
                                                partition, _p(e), _p(grad), _p(tq)))
        return e, grad, tq

    def grid_local_search_batch(self, dgrid: DevGrid, inst: Instance, params: LigandParams, starts, max_iters, tol,
                                method=BASELINE, partition=64):
        s = np.ascontiguousarray(starts, np.float64).reshape(-1, inst.dim)
        n = s.shape[0]
        g = np.zeros((n, inst.dim))
        e = np.zeros(n)
        it = np.zeros(n, np.int32)
        cv = np.zeros(n, np.int32)
        self._chk(self.lib.mdr_grid_local_search_batch(self.ctx, dgrid.h, inst.cref(), params.cref(), _p(s), n,
                                                       max_iters, tol, method, partition, _p(g), _p(e), _p(it),
                                                       _p(cv)))
        return [LocalSearchResult(g[i], float(e[i]), int(it[i]), bool(cv[i]), SyncStats()) for i in range(n)]

    def grid_screen_batch(self, dgrid: DevGrid, ligands, params, runs_per_ligand: int, method,
                          settings: LgaSettings, seeds, rmsd_tol: float = 2.0):
        """Virtual-screen batch (mdr_grid_screen_batch): every ligand docked
        runs_per_ligand times in one launch sequence, then clustered.
        Returns one dict per ligand: best_energy[runs], best_genotype[runs,dim],
        evaluations[runs], converged[runs], cluster_of[runs], rmsd_to_seed[runs],
        n_clusters."""
        from ._abi import CInstance, CLigandParams

        n = len(ligands)
        R = n * runs_per_ligand
        seeds = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
        if seeds.size != R:
            raise ValueError("need one seed per (ligand, run)")
        ci = (CInstance * n)(*[l.c() for l in ligands])
        cp = (CLigandParams * n)(*[p.c() for p in params])
        be = np.zeros(R)
        bg = np.zeros(sum(runs_per_ligand * l.dim for l in ligands))
        ev = np.zeros(R, np.int64)
        cv = np.zeros(R, np.int32)
        cl = np.zeros(R, np.int32)
        rm = np.zeros(R)
        nc = np.zeros(n, np.int32)
        self._chk(self.lib.mdr_grid_screen_batch(self.ctx, dgrid.h, ci, cp, n, runs_per_ligand, method,
                                                 C.byref(settings), _p(seeds), rmsd_tol, _p(be), _p(bg), _p(ev),
                                                 _p(cv), _p(cl), _p(rm), _p(nc)))
        out, o = [], 0
        for j, l in enumerate(ligands):
            sl = slice(j * runs_per_ligand, (j + 1) * runs_per_ligand)
            k = runs_per_ligand * l.dim
            out.append(dict(best_energy=be[sl].copy(), best_genotype=bg[o:o + k].reshape(runs_per_ligand, l.dim),
                            evaluations=ev[sl].copy(), converged=cv[sl].astype(bool), cluster_of=cl[sl].copy(),
                            rmsd_to_seed=rm[sl].copy(), n_clusters=int(nc[j])))
            o += k
        return out

    def grid_lga_run_batch(self, dgrid: DevGrid, inst: Instance, params: LigandParams, method,
                           settings: LgaSettings, seeds):
        seeds = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
        n = seeds.size
        maxr = settings.max_records
        be = np.zeros(n)
        bg = np.zeros((n, inst.dim))
        ev = np.zeros(n, np.int64)
        cv = np.zeros(n, np.int32)
        nr = np.zeros(n, np.int32)
        recs = (LsRecord * (n * maxr))()
        self._chk(self.lib.mdr_grid_lga_run_batch(self.ctx, dgrid.h, inst.cref(), params.cref(), method,
                                                  C.byref(settings), _p(seeds), n, _p(be), _p(bg), _p(ev), _p(cv),
                                                  _p(nr), recs))
        out = []
        for i in range(n):
            runs = [(recs[i * maxr + k].best_energy, recs[i * maxr + k].iterations,
                     bool(recs[i * maxr + k].converged)) for k in range(min(int(nr[i]), maxr))]
            out.append(DockResult(float(be[i]), bg[i], int(ev[i]), bool(cv[i]), runs))
        return out


class DevGrid:
    """A device-resident receptor map set (mdr_dev_grid), shared by every
    ligand docked against it."""

    def __init__(self, dev: "Device", handle, grid: Grid):
        self.dev, self.h, self.grid = dev, handle, grid

    def download(self) -> np.ndarray:
        g = self.grid
        maps = np.zeros((g.n_types + 2,) + tuple(int(v) for v in g.shape[::-1]), np.float32)
        self.dev._chk(self.dev.lib.mdr_grid_download(self.dev.ctx, self.h, _p(maps)))
        return maps

    def free(self):
        if self.h:
            self.dev.lib.mdr_grid_free(self.dev.ctx, self.h)
            self.h = None

    def __del__(self):
        try:
            if self.dev.ctx:
                self.free()
        except Exception:
            pass


def multi_lga_run_batch(devices, inst: Instance, method, accum, settings: LgaSettings, seeds,
                        pair: int = PAIR_FP64_FAST):
    """Native multi-GPU docking (mdr_multi_lga_run_batch): runs sharded
    round-robin over `devices`, one host thread + context per device.
    Returns (best_energy[n], best_genotype[n, dim], evaluations[n], converged[n])."""
    lib = _lib.load()
    dv = np.ascontiguousarray(devices, np.int32)
    seeds = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
    n = seeds.size
    be, bg = np.zeros(n), np.zeros((n, inst.dim))
    ev, cv = np.zeros(n, np.int64), np.zeros(n, np.int32)
    rc = lib.mdr_multi_lga_run_batch(_p(dv), dv.size, inst.cref(), method, accum, pair, C.byref(settings), _p(seeds), n,
                                     _p(be), _p(bg), _p(ev), _p(cv))
    raise_for(rc, lib.mdr_multi_last_error().decode())
    return be, bg, ev, cv.astype(bool)


def multi_screen(devices, sites: Instance, fields: ReceptorFields, grid: Grid, ligands, params, runs_per_ligand: int,
                 method, settings: LgaSettings, seeds, rmsd_tol: float = 2.0, batch_ligands: int = 256):
    """Native multi-GPU virtual screen (mdr_multi_screen): each device builds
    the receptor once and pulls ligand batches from a shared queue.  Returns
    (best_energy[n*R], best_genotype packed, evaluations[n*R],
    cluster_of[n*R], n_clusters[n], device_of_ligand[n])."""
    from ._abi import CInstance, CLigandParams

    lib = _lib.load()
    dv = np.ascontiguousarray(devices, np.int32)
    n, R = len(ligands), runs_per_ligand
    seeds = np.ascontiguousarray(seeds, np.uint64).reshape(-1)
    ci = (CInstance * n)(*[l.c() for l in ligands])
    cp = (CLigandParams * n)(*[p.c() for p in params])
    be = np.zeros(n * R)
    bg = np.zeros(sum(R * l.dim for l in ligands))
    ev = np.zeros(n * R, np.int64)
    cl = np.zeros(n * R, np.int32)
    nc = np.zeros(n, np.int32)
    dol = np.full(n, -1, np.int32)
    rc = lib.mdr_multi_screen(_p(dv), dv.size, sites.cref(), fields.cref(), grid.cref(), ci, cp, n, R, method,
                              C.byref(settings), _p(seeds), rmsd_tol, batch_ligands, _p(be), _p(bg), _p(ev), _p(cl),
                              _p(nc), _p(dol))
    raise_for(rc, lib.mdr_multi_last_error().decode())
    return be, bg, ev, cl, nc, dol


@dataclass
class MethodSummary:
    min: float
    q1: float
    median: float
    q3: float
    max: float
    mean: float
    nonconvergent_fraction: float


def summarize(bests, nonconv: int, n: int) -> MethodSummary:
    """summarize docking.cpp:521-542 (host statistics)."""
    b = sorted(bests)

    def q(p):
        if len(b) == 1:
            return b[0]
        h = p * (len(b) - 1)
        lo = int(h)
        hi = min(lo + 1, len(b) - 1)
        return b[lo] + (h - lo) * (b[hi] - b[lo])

    mean = 0.0
    for x in b:
        mean += x
    return MethodSummary(b[0], q(0.25), q(0.5), q(0.75), b[-1], mean / len(b), nonconv / n)


def validate_pair(dev: Device, inst, ref_method, test_method, accum, n_runs, base_seed, settings):
    """validate_pair docking.cpp:546-580: paired seeds base_seed + i, both
    methods, all runs of a method in one device batch."""
    if n_runs < 1:
        raise SizeError("validate_pair needs at least one run")
    seeds = np.arange(n_runs, dtype=np.uint64) + np.uint64(base_seed)
    a = dev.lga_run_batch(inst, ref_method, accum, settings, seeds)
    b = dev.lga_run_batch(inst, test_method, accum, settings, seeds)
    ref = summarize([r.best_energy for r in a], sum(not r.converged for r in a), n_runs)
    test = summarize([r.best_energy for r in b], sum(not r.converged for r in b), n_runs)
    diff = abs(test.mean - ref.mean)
    rel = float("inf") if ref.mean == 0.0 else diff / abs(ref.mean)
    return dict(ref=ref, test=test, abs_diff_means=diff, relative_error=rel, n_runs=n_runs)


__all__ = ["Device", "ScoreResult", "LocalSearchResult", "DockResult", "validate_pair", "summarize",
           "BASELINE", "TCU", "TCU_SPLIT", "HALF", "SINGLE"]
