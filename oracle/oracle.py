"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over the two CPU checkers:

  * ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement
                               (mdr_oracle.c, each function cites the reference
                               file:line it restates);
  * ``Oracle("reference")`` -> oracle/_ref/libmdr_ref.so, the unmodified
                               reference library compiled in place from
                               /root/reference/proj/src (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may import this.
The product (paper_2410_10447_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2410_10447_b200._abi import (
    BASELINE,
    Grid,
    LgaSettings,
    LsRecord,
    SyncStats,
    dptr,
    fptr,
    raise_for,
    u16ptr,
    u64ptr,
)

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmdr_ref.so")


def build(quiet: bool = True) -> None:
    """Build liboracle.so (always) and _ref/ (when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "reference" else PORT_SO)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = REF_SO if kind == "reference" else PORT_SO
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.p = "ref_" if kind == "reference" else "orc_"
        # functions taking doubles by value need explicit argtypes
        f = self._f("adadelta_step")
        f.argtypes = [C.c_int, C.c_double, C.c_double] + [C.POINTER(C.c_double)] * 4
        f = self._f("local_search")
        f.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_double, C.c_int, C.c_int,
                      C.c_int, C.POINTER(C.c_double), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _err(self) -> str:
        if self.kind == "reference":
            self.lib.ref_last_error.restype = C.c_char_p
            return self.lib.ref_last_error().decode()
        return "oracle error"

    def _chk(self, rc):
        raise_for(rc, self._err())

    # ---- rng / half / mma -------------------------------------------------
    def rng_draws(self, seed: int, label: str, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self._f("rng_draws")(C.c_uint64(seed), label.encode(), C.c_uint64(n), u64ptr(out))
        return out

    def rng_normals(self, seed: int, label: str, n: int) -> np.ndarray:
        out = np.zeros(n, np.float64)
        self._f("rng_normals")(C.c_uint64(seed), label.encode(), C.c_uint64(n), dptr(out))
        return out

    def f32_to_half(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(x.size, np.uint16)
        self._f("f32_to_half")(fptr(x), C.c_size_t(x.size), u16ptr(out))
        return out

    def half_to_f32(self, h) -> np.ndarray:
        h = np.ascontiguousarray(h, np.uint16)
        out = np.zeros(h.size, np.float32)
        self._f("half_to_f32")(u16ptr(h), C.c_size_t(h.size), fptr(out))
        return out

    def mma(self, a, b, c, accum) -> np.ndarray:
        a = np.ascontiguousarray(a, np.uint16).reshape(256)
        b = np.ascontiguousarray(b, np.uint16).reshape(256)
        c = np.ascontiguousarray(c, np.float32).reshape(256)
        d = np.zeros(256, np.float32)
        self._chk(self._f("mma")(u16ptr(a), u16ptr(b), fptr(c), accum, fptr(d)))
        return d.reshape(16, 16)

    # ---- reductions --------------------------------------------------------
    def reduce4(self, vecs, accum):
        v = np.ascontiguousarray(vecs, np.float32).reshape(-1, 4)
        out = np.zeros(4, np.float32)
        st = SyncStats()
        self._chk(self._f("reduce4")(fptr(v), v.shape[0], accum, fptr(out), C.byref(st)))
        return out, st

    def simulate_block4(self, vecs, method, accum):
        v = np.ascontiguousarray(vecs, np.float32).reshape(-1, 4)
        out = np.zeros(4, np.float32)
        st = SyncStats()
        self._chk(self._f("simulate_block4")(fptr(v), v.shape[0], method, accum, fptr(out), C.byref(st)))
        return out, st

    def warp_reduce(self, lanes):
        v = np.ascontiguousarray(lanes, np.float32)
        out = C.c_float()
        st = SyncStats()
        self._chk(self._f("warp_reduce")(fptr(v), v.size, C.byref(out), C.byref(st)))
        return out.value, st

    def block_reduce(self, values, threads):
        v = np.ascontiguousarray(values, np.float32)
        out = C.c_float()
        st = SyncStats()
        self._chk(self._f("block_reduce")(fptr(v), v.size, threads, C.byref(out), C.byref(st)))
        return np.float32(out.value), st

    def reduce7(self, recs, method, accum):
        r = np.ascontiguousarray(recs, np.float32).reshape(-1, 7)
        out = np.zeros(7, np.float32)
        st = SyncStats()
        self._chk(self._f("reduce7")(fptr(r), r.shape[0], method, accum, fptr(out), C.byref(st)))
        return out, st

    # ---- scoring -----------------------------------------------------------
    def score(self, inst, g, method=BASELINE, accum=1, partition=64):
        g = np.ascontiguousarray(g, np.float64)
        e = C.c_float()
        grad = np.zeros(inst.dim, np.float32)
        tq = np.zeros(3, np.float32)
        st = SyncStats()
        self._chk(self._f("score")(inst.cref(), dptr(g), method, accum, partition, C.byref(e),
                                   fptr(grad), fptr(tq), C.byref(st)))
        return np.float32(e.value), grad, tq, st

    def score_many(self, inst, gs, method=BASELINE, accum=1, partition=64):
        """Many poses of one instance (reference-only fast path, else a loop)."""
        gs = np.ascontiguousarray(gs, np.float64).reshape(-1, inst.dim)
        n = gs.shape[0]
        if self.kind == "reference":
            e = np.zeros(n, np.float32)
            grad = np.zeros((n, inst.dim), np.float32)
            tq = np.zeros((n, 3), np.float32)
            self._chk(self.lib.ref_score_many(inst.cref(), dptr(gs), n, method, accum, partition,
                                              fptr(e), fptr(grad), fptr(tq)))
            return e, grad, tq
        res = [self.score(inst, g, method, accum, partition) for g in gs]
        return (np.array([r[0] for r in res], np.float32), np.stack([r[1] for r in res]),
                np.stack([r[2] for r in res]))

    def score_reference(self, inst, g):
        g = np.ascontiguousarray(g, np.float64)
        e = C.c_double()
        grad = np.zeros(inst.dim, np.float64)
        tq = np.zeros(3, np.float64)
        self._chk(self._f("score_reference")(inst.cref(), dptr(g), C.byref(e), dptr(grad), dptr(tq)))
        return e.value, grad, tq

    def torsion_axis(self, k: int) -> np.ndarray:
        out = np.zeros(3)
        if self.kind == "reference":
            self.lib.ref_torsion_axis(k, dptr(out))
        else:
            self.lib.orc_torsion_axis_out(k, dptr(out))
        return out

    # ---- search ------------------------------------------------------------
    def adadelta_step(self, sq_g, sq_u, geno, grad, rho=0.95, eps=1e-6):
        sq_g = np.array(sq_g, np.float64)
        sq_u = np.array(sq_u, np.float64)
        geno = np.array(geno, np.float64)
        grad = np.ascontiguousarray(grad, np.float64)
        self._chk(self._f("adadelta_step")(geno.size, C.c_double(rho), C.c_double(eps), dptr(sq_g),
                                           dptr(sq_u), dptr(geno), dptr(grad)))
        return sq_g, sq_u, geno

    def local_search(self, inst, start, max_iters, tol, method=BASELINE, accum=1, partition=64):
        start = np.ascontiguousarray(start, np.float64)
        g = np.zeros(inst.dim)
        e = C.c_double()
        it = C.c_int32()
        cv = C.c_int32()
        st = SyncStats()
        self._chk(self._f("local_search")(inst.cref(), dptr(start), max_iters, C.c_double(tol), method,
                                          accum, partition, dptr(g), C.byref(e), C.byref(it),
                                          C.byref(cv), C.byref(st)))
        return dict(genotype=g, energy=e.value, iterations=it.value, converged=bool(cv.value), stats=st)

    def lga_run(self, inst, method, accum, settings: LgaSettings, seed: int):
        maxr = settings.max_records
        g = np.zeros(inst.dim)
        be = C.c_double()
        ev = C.c_int64()
        cv = C.c_int32()
        nr = C.c_int32()
        recs = (LsRecord * maxr)()
        st = SyncStats()
        self._chk(self._f("lga_run")(inst.cref(), method, accum, C.byref(settings), C.c_uint64(seed),
                                     C.byref(be), dptr(g), C.byref(ev), C.byref(cv), C.byref(nr),
                                     recs, maxr, C.byref(st)))
        runs = [(recs[i].best_energy, recs[i].iterations, bool(recs[i].converged))
                for i in range(min(nr.value, maxr))]
        return dict(best_energy=be.value, best_genotype=g, evaluations=ev.value,
                    converged=bool(cv.value), runs=runs, total_stats=st)

    # ---- grid mode (port only; no reference counterpart) -------------------
    def grid_build(self, sites_inst, fields, grid: Grid) -> np.ndarray:
        maps = np.zeros((grid.n_types + 2,) + tuple(int(v) for v in grid.shape[::-1]), np.float32)
        shape = grid.c()
        self._chk(self.lib.orc_grid_build(sites_inst.cref(), fields.cref(), C.byref(shape), fptr(maps)))
        return maps

    def grid_score(self, inst, grid: Grid, params, g):
        g = np.ascontiguousarray(g, np.float64)
        e, ei = C.c_double(), C.c_double()
        grad = np.zeros(inst.dim)
        tq = np.zeros(3)
        cg = grid.c()
        self._chk(self.lib.orc_grid_score(inst.cref(), C.byref(cg), params.cref(), dptr(g), C.byref(e),
                                          dptr(grad), dptr(tq), C.byref(ei)))
        return e.value, grad, tq, ei.value

    def grid_local_search(self, inst, grid: Grid, params, start, max_iters, tol):
        f = self.lib.orc_grid_local_search
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_double,
                      C.POINTER(C.c_double), C.c_void_p, C.c_void_p, C.c_void_p]
        start = np.ascontiguousarray(start, np.float64)
        g = np.zeros(inst.dim)
        e, it, cv = C.c_double(), C.c_int32(), C.c_int32()
        cg = grid.c()
        self._chk(f(inst.cref(), C.byref(cg), params.cref(), dptr(start), max_iters, tol, dptr(g), C.byref(e),
                    C.byref(it), C.byref(cv)))
        return dict(genotype=g, energy=e.value, iterations=it.value, converged=bool(cv.value))

    def grid_lga_run(self, inst, grid: Grid, params, settings: LgaSettings, seed: int):
        maxr = settings.max_records
        g = np.zeros(inst.dim)
        be, ev, cv, nr = C.c_double(), C.c_int64(), C.c_int32(), C.c_int32()
        recs = (LsRecord * maxr)()
        cg = grid.c()
        self._chk(self.lib.orc_grid_lga_run(inst.cref(), C.byref(cg), params.cref(), C.byref(settings),
                                            C.c_uint64(seed), C.byref(be), dptr(g), C.byref(ev), C.byref(cv),
                                            C.byref(nr), recs, maxr))
        runs = [(recs[i].best_energy, recs[i].iterations, bool(recs[i].converged))
                for i in range(min(nr.value, maxr))]
        return dict(best_energy=be.value, best_genotype=g, evaluations=ev.value, converged=bool(cv.value),
                    runs=runs)

    # ---- RMSD clustering (port only) ---------------------------------------
    def pose_coords(self, inst, g):
        g = np.ascontiguousarray(g, np.float64)
        xyz = np.zeros((inst.n_atoms, 3))
        self._chk(self.lib.orc_pose_coords(inst.cref(), dptr(g), dptr(xyz)))
        return xyz

    def cluster_poses(self, inst, genotypes, energies, rmsd_tol=2.0):
        f = self.lib.orc_cluster_poses
        f.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int, C.c_double,
                      C.c_void_p, C.POINTER(C.c_double), C.c_void_p]
        g = np.ascontiguousarray(genotypes, np.float64).reshape(-1, inst.dim)
        e = np.ascontiguousarray(energies, np.float64).reshape(-1)
        n = g.shape[0]
        c = np.zeros(n, np.int32)
        r = np.zeros(n)
        nc = C.c_int32()
        self._chk(f(inst.cref(), dptr(g), dptr(e), n, rmsd_tol, c.ctypes.data, dptr(r), C.byref(nc)))
        return c, r, nc.value


def _lga_job(args):
    kind, inst, method, accum, settings, seed = args
    r = Oracle(kind).lga_run(inst, method, accum, settings, int(seed))
    return r["best_energy"], r["evaluations"], r["converged"], np.asarray(r["best_genotype"]).copy()


def lga_runs_parallel(kind, inst, method, accum, settings: LgaSettings, seeds, procs=None):
    """Test infrastructure: CPU LGA runs (one per seed) on a pool of
    `spawn`ed processes (safe after CUDA initialisation in the parent, and
    processes rather than threads: the reference's per-call vectors contend
    on the allocator).  Returns a list of (best_energy,
    evaluations, converged, best_genotype) in seed order."""
    import multiprocessing as mp

    procs = procs or min(len(seeds), os.cpu_count() or 1)
    jobs = [(kind, inst, method, accum, settings, int(s)) for s in seeds]
    with mp.get_context("spawn").Pool(procs) as pool:
        return pool.map(_lga_job, jobs)


_GRID_JOB = {}  # (inst, grid, params, settings) shared with forked workers


def _grid_lga_job(seed):
    inst, grid, params, settings = _GRID_JOB["case"]
    r = Oracle("port").grid_lga_run(inst, grid, params, settings, int(seed))
    return r["best_energy"], r["evaluations"], r["converged"], np.asarray(r["best_genotype"]).copy()


def grid_lga_runs_parallel(inst, grid, params, settings: LgaSettings, seeds, procs=None):
    """Test infrastructure: oracle grid-mode LGA runs (orc_grid_lga_run), one
    per seed, on `fork`ed worker processes that inherit the maps (tens of MB)
    instead of receiving them pickled; the workers only call the C oracle.
    Returns (best_energy, evaluations, converged, best_genotype) per seed."""
    import multiprocessing as mp

    _GRID_JOB["case"] = (inst, grid, params, settings)
    procs = procs or min(len(seeds), os.cpu_count() or 1)
    try:
        with mp.get_context("fork").Pool(procs) as pool:
            return pool.map(_grid_lga_job, [int(s) for s in seeds])
    finally:
        _GRID_JOB.clear()


def cr_values(i0: int, n: int) -> np.ndarray:
    """crmath.h's correctly rounded sin a, cos a, log u1, cos z on the
    device crmath probe's inputs (see orc_cr_values); shape (n, 4)."""
    lib = Oracle("port").lib
    out = np.zeros((n, 4))
    lib.orc_cr_values.argtypes = [C.c_int64, C.c_int, C.c_void_p]
    lib.orc_cr_values(i0, n, out.ctypes.data)
    return out
