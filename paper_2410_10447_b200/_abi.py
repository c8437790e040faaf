"""ctypes mirror of the plain-data structs in include/mdr.h, plus the host-side
ligand container.  Shared by the product binding (`_lib.py`) and, read-only, by
the test-only oracle wrapper (`oracle/oracle.py`).

The MDRI text parser here is host I/O (SURVEY §2 row 7 is out of the hot path);
it follows parse_instance (reference proj/src/instance_io.cpp:137-253): magic
line first, `nrot` exactly once, `atom x y z w tors|-`, `site x y z depth d0`,
'#' comments, line-numbered errors.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

# status codes / enums (mdr.h)
OK, ERR_SIZE, ERR_BLOCK_SIZE, ERR_NUMERIC_DOMAIN, ERR_PARSE, ERR_CUDA, ERR_INVALID = range(7)
BASELINE, TCU, TCU_SPLIT = 0, 1, 2
HALF, SINGLE = 0, 1
PAIR_FP64, PAIR_FP32, PAIR_FP64_FAST = 0, 1, 2


class SizeError(ValueError):
    """reference errors.hpp:10-13"""


class UnsupportedBlockSizeError(ValueError):
    """reference errors.hpp:16-20"""


class NumericDomainError(ArithmeticError):
    """reference errors.hpp:23-26"""


class ParseError(RuntimeError):
    """reference errors.hpp:29-42 (carries the 1-based line, 0 = none)"""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}" if line > 0 else what)
        self.line = line


class DeviceError(RuntimeError):
    """CUDA / driver failure (no reference counterpart)."""


_EXC = {
    ERR_SIZE: SizeError,
    ERR_BLOCK_SIZE: UnsupportedBlockSizeError,
    ERR_NUMERIC_DOMAIN: NumericDomainError,
    ERR_CUDA: DeviceError,
    ERR_INVALID: ValueError,
}


def raise_for(status: int, msg: str) -> None:
    if status == OK:
        return
    if status == ERR_PARSE:
        raise ParseError(0, msg)
    raise _EXC.get(status, RuntimeError)(msg)


class SyncStats(C.Structure):
    """SyncStats reference include/mdreduce/reduce.hpp:33-54."""

    _fields_ = [
        ("block_syncs", C.c_uint64),
        ("warp_shuffles", C.c_uint64),
        ("atomic_adds", C.c_uint64),
        ("memory_fences", C.c_uint64),
        ("mma_ops", C.c_uint64),
        ("shared_mem_bytes", C.c_uint64),
        ("precision_conversions", C.c_uint64),
    ]

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_)

    def __eq__(self, other):
        return isinstance(other, SyncStats) and self.as_tuple() == other.as_tuple()

    def __repr__(self):
        return "SyncStats(" + ", ".join(f"{f}={getattr(self, f)}" for f, _ in self._fields_) + ")"


class CInstance(C.Structure):
    _fields_ = [
        ("n_atoms", C.c_int32),
        ("n_sites", C.c_int32),
        ("n_rot", C.c_int32),
        ("reserved", C.c_int32),
        ("atom_xyzw", C.POINTER(C.c_double)),
        ("atom_torsion", C.POINTER(C.c_int32)),
        ("site_xyzdd", C.POINTER(C.c_double)),
    ]


class LgaSettings(C.Structure):
    """LgaSettings reference include/mdreduce/docking.hpp:106-115 (defaults)."""

    _fields_ = [
        ("population_size", C.c_int32),
        ("generations", C.c_int32),
        ("max_evaluations", C.c_int64),
        ("ls_fraction", C.c_double),
        ("ls_max_iters", C.c_int32),
        ("partition", C.c_int32),
        ("ls_convergence_tol", C.c_double),
        ("mutation_sigma", C.c_double),
    ]

    def __init__(self, **kw):
        super().__init__()
        self.population_size = 36
        self.generations = 20
        self.max_evaluations = 100000
        self.ls_fraction = 0.25
        self.ls_max_iters = 150
        self.partition = 64
        self.ls_convergence_tol = 1e-4
        self.mutation_sigma = 0.3
        for k, v in kw.items():
            setattr(self, k, v)

    @property
    def ls_count(self) -> int:
        off = self.population_size - 1
        return min(max(int(math.ceil(self.ls_fraction * off)), 0), off)

    @property
    def max_records(self) -> int:
        return self.generations * self.ls_count + 1


class LsRecord(C.Structure):
    _fields_ = [("best_energy", C.c_double), ("iterations", C.c_int32), ("converged", C.c_int32)]


def dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def i32ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def i64ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def u64ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def u16ptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint16))


@dataclass
class Instance:
    """LigandInstance (reference include/mdreduce/instance_io.hpp:13-30)."""

    atoms: np.ndarray  # (n_atoms, 4) float64: x, y, z, weight
    torsion: np.ndarray  # (n_atoms,) int32, -1 rigid
    sites: np.ndarray  # (n_sites, 5) float64: x, y, z, depth, d0
    n_rot: int
    name: str = ""
    _c: CInstance | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.atoms = np.ascontiguousarray(self.atoms, dtype=np.float64).reshape(-1, 4)
        self.torsion = np.ascontiguousarray(self.torsion, dtype=np.int32).reshape(-1)
        self.sites = np.ascontiguousarray(self.sites, dtype=np.float64).reshape(-1, 5)
        self.n_rot = int(self.n_rot)

    @property
    def n_atoms(self) -> int:
        return int(self.atoms.shape[0])

    @property
    def n_sites(self) -> int:
        return int(self.sites.shape[0])

    @property
    def dim(self) -> int:
        return 6 + self.n_rot

    def c(self) -> CInstance:
        if self._c is None:
            ci = CInstance()
            ci.n_atoms, ci.n_sites, ci.n_rot, ci.reserved = self.n_atoms, self.n_sites, self.n_rot, 0
            ci.atom_xyzw = dptr(self.atoms)
            ci.atom_torsion = i32ptr(self.torsion)
            ci.site_xyzdd = dptr(self.sites)
            self._c = ci
        return self._c

    def cref(self):
        return C.byref(self.c())


def parse_instance(text: str) -> Instance:
    """parse_instance (reference proj/src/instance_io.cpp:137-253)."""
    saw_magic = False
    n_rot = None
    atoms, tors, sites, atom_lines = [], [], [], []
    lines = text.split("\n")
    line_no = 0

    def num(tok, ln, what):
        try:
            v = float(tok)
        except ValueError:
            raise ParseError(ln, f"invalid number for {what}: '{tok}'") from None
        if not math.isfinite(v):
            raise ParseError(ln, f"non-finite value for {what}")
        return v

    def integer(tok, ln, what):
        try:
            return int(tok)
        except ValueError:
            raise ParseError(ln, f"invalid integer for {what}: '{tok}'") from None

    for raw in lines:
        line_no += 1
        line = raw.split("#", 1)[0]
        toks = line.split()
        if not saw_magic:
            if not toks:
                if line_no == 1:
                    raise ParseError(1, "missing magic line 'MDRI 1'")
                continue
            if toks != ["MDRI", "1"]:
                raise ParseError(line_no, "missing magic line 'MDRI 1'")
            saw_magic = True
            continue
        if not toks:
            continue
        if toks[0] == "nrot":
            if n_rot is not None:
                raise ParseError(line_no, "duplicate nrot line")
            if len(toks) != 2:
                raise ParseError(line_no, "nrot expects one integer")
            n = integer(toks[1], line_no, "nrot")
            if n < 0:
                raise ParseError(line_no, "nrot must be non-negative")
            n_rot = n
        elif toks[0] == "atom":
            if len(toks) != 6:
                raise ParseError(line_no, "atom expects <x> <y> <z> <weight> <torsion|->")
            xyz = [num(t, line_no, "atom coordinate") for t in toks[1:4]]
            w = num(toks[4], line_no, "atom weight")
            if w <= 0.0:
                raise ParseError(line_no, "atom weight must be positive")
            if toks[5] == "-":
                t = -1
            else:
                t = integer(toks[5], line_no, "torsion index")
                if t < 0:
                    raise ParseError(line_no, "torsion index must be non-negative or '-'")
            atoms.append(xyz + [w])
            tors.append(t)
            atom_lines.append(line_no)
        elif toks[0] == "site":
            if len(toks) != 6:
                raise ParseError(line_no, "site expects <x> <y> <z> <depth> <d0>")
            vals = [num(t, line_no, "site value") for t in toks[1:6]]
            if vals[3] <= 0.0:
                raise ParseError(line_no, "site depth must be positive")
            if vals[4] <= 0.0:
                raise ParseError(line_no, "site d0 must be positive")
            sites.append(vals)
        else:
            raise ParseError(line_no, f"unknown directive '{toks[0]}'")
    if not saw_magic:
        raise ParseError(1, "missing magic line 'MDRI 1'")
    if n_rot is None:
        raise ParseError(line_no, "missing nrot line")
    for t, ln in zip(tors, atom_lines):
        if t >= n_rot:
            raise ParseError(ln, f"atom references torsion {t} but nrot is {n_rot}")
    if not atoms:
        raise ParseError(line_no, "instance needs at least one atom")
    if not sites:
        raise ParseError(line_no, "instance needs at least one site")
    return Instance(np.array(atoms), np.array(tors), np.array(sites), n_rot)


def serialize_instance(inst: Instance) -> str:
    out = ["MDRI 1", f"nrot {inst.n_rot}"]
    for a, t in zip(inst.atoms, inst.torsion):
        out.append("atom " + " ".join(repr(float(v)) for v in a) + " " + ("-" if t < 0 else str(int(t))))
    for s in inst.sites:
        out.append("site " + " ".join(repr(float(v)) for v in s))
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------ RNG
# RngStream (reference proj/src/rng.cpp:9-56) — pure uint64 arithmetic, used by
# the host to build synthetic instances (bench configs C3/C4/C5) exactly like
# the reference's random_instance recipe (tests/test_docking.cpp:39-59).
_M64 = (1 << 64) - 1


def _mix64(z: int) -> int:
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for b in s.encode():
        h = ((h ^ b) * 0x100000001B3) & _M64
    return h


class RngStream:
    def __init__(self, seed: int, label: str):
        self.key = _mix64((seed & _M64) ^ _mix64(_fnv1a64(label)))
        self.counter = 0

    def next_u64(self) -> int:
        self.counter += 1
        return _mix64((self.key + self.counter * 0x9E3779B97F4A7C15) & _M64)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0**-53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def next_index(self, n: int) -> int:
        return 0 if n == 0 else self.next_u64() % n


def derive_rng(seed: int, label: str) -> RngStream:
    return RngStream(seed, label)


def random_instance(rng: RngStream, nrot: int, natoms: int, nsites: int) -> Instance:
    """random_instance recipe (reference tests/test_docking.cpp:39-59)."""
    atoms, tors, sites = [], [], []
    for i in range(natoms):
        pos = [rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5)]
        w = rng.uniform(0.5, 1.5)
        t = rng.next_index(nrot) if (nrot > 0 and i % 2 == 0) else -1
        atoms.append(pos + [w])
        tors.append(t)
    for _ in range(nsites):
        pos = [rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0)]
        depth = rng.uniform(0.8, 1.6)
        d0 = rng.uniform(1.0, 2.0)
        sites.append(pos + [depth, d0])
    return Instance(np.array(atoms), np.array(tors), np.array(sites), nrot)


def random_pose(rng: RngStream, nrot: int, spread: float) -> np.ndarray:
    """random_pose recipe (reference tests/test_docking.cpp:61-73)."""
    g = [rng.uniform(-spread, spread) for _ in range(3)]
    g += [rng.uniform(-3.1, 3.1) for _ in range(3)]
    g += [rng.uniform(-3.1, 3.1) for _ in range(nrot)]
    return np.array(g)


# ----------------------------------------------------------------- grid mode
# mdr.h "grid-map scoring mode".
GRID_OUTSIDE_K = 10.0  # MDR_GRID_OUTSIDE_K


class CGrid(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("n_types", C.c_int32),
        ("origin", C.c_double * 3), ("spacing", C.c_double),
        ("maps", C.POINTER(C.c_float)),
    ]


class CLigandParams(C.Structure):
    _fields_ = [
        ("atom_type", C.POINTER(C.c_int32)), ("atom_charge", C.POINTER(C.c_double)),
        ("atom_radius", C.POINTER(C.c_double)), ("atom_epsilon", C.POINTER(C.c_double)),
        ("elec_scale", C.c_double), ("intra", C.c_int32), ("reserved", C.c_int32),
    ]


class CReceptorFields(C.Structure):
    _fields_ = [
        ("site_charge", C.POINTER(C.c_double)), ("site_volume", C.POINTER(C.c_double)),
        ("type_depth_scale", C.POINTER(C.c_double)), ("type_dist_scale", C.POINTER(C.c_double)),
        ("elec_scale", C.c_double), ("desolv_sigma", C.c_double),
    ]


@dataclass
class Grid:
    """Receptor maps: (n_types + 2, nz, ny, nx) float32 (types, elec, desolv)."""

    shape: tuple  # (nx, ny, nz)
    n_types: int
    origin: tuple
    spacing: float
    maps: np.ndarray | None = None
    _c: CGrid | None = field(default=None, repr=False, compare=False)

    def c(self) -> CGrid:
        g = CGrid()
        g.nx, g.ny, g.nz = (int(v) for v in self.shape)
        g.n_types = int(self.n_types)
        g.origin = (C.c_double * 3)(*[float(v) for v in self.origin])
        g.spacing = float(self.spacing)
        if self.maps is not None:
            self.maps = np.ascontiguousarray(self.maps, np.float32)
            g.maps = fptr(self.maps)
        self._c = g
        return g

    def cref(self):
        return C.byref(self.c())

    @property
    def n_points(self) -> int:
        nx, ny, nz = self.shape
        return int(nx) * int(ny) * int(nz)


@dataclass
class LigandParams:
    """Per-atom chemistry for grid mode (mdr_ligand_params)."""

    atom_type: np.ndarray
    charge: np.ndarray
    radius: np.ndarray
    epsilon: np.ndarray
    elec_scale: float = 83.0
    intra: bool = True
    _c: CLigandParams | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.atom_type = np.ascontiguousarray(self.atom_type, np.int32)
        self.charge = np.ascontiguousarray(self.charge, np.float64)
        self.radius = np.ascontiguousarray(self.radius, np.float64)
        self.epsilon = np.ascontiguousarray(self.epsilon, np.float64)

    def c(self) -> CLigandParams:
        p = CLigandParams()
        p.atom_type = i32ptr(self.atom_type)
        p.atom_charge = dptr(self.charge)
        p.atom_radius = dptr(self.radius)
        p.atom_epsilon = dptr(self.epsilon)
        p.elec_scale = float(self.elec_scale)
        p.intra = 1 if self.intra else 0
        self._c = p
        return p

    def cref(self):
        return C.byref(self.c())


@dataclass
class ReceptorFields:
    """Inputs of the synthetic map builder (mdr_receptor_fields)."""

    site_charge: np.ndarray
    site_volume: np.ndarray
    type_depth_scale: np.ndarray
    type_dist_scale: np.ndarray
    elec_scale: float = 83.0
    desolv_sigma: float = 3.6
    _c: CReceptorFields | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        for k in ("site_charge", "site_volume", "type_depth_scale", "type_dist_scale"):
            setattr(self, k, np.ascontiguousarray(getattr(self, k), np.float64))

    @property
    def n_types(self) -> int:
        return int(self.type_depth_scale.size)

    def c(self) -> CReceptorFields:
        f = CReceptorFields()
        f.site_charge = dptr(self.site_charge)
        f.site_volume = dptr(self.site_volume)
        f.type_depth_scale = dptr(self.type_depth_scale)
        f.type_dist_scale = dptr(self.type_dist_scale)
        f.elec_scale = float(self.elec_scale)
        f.desolv_sigma = float(self.desolv_sigma)
        self._c = f
        return f

    def cref(self):
        return C.byref(self.c())


def random_ligand_params(rng: RngStream, n_atoms: int, n_types: int) -> LigandParams:
    """Synthetic ligand chemistry: per atom, in this draw order,
    type = next_index(n_types), charge U(-0.4, 0.4), radius U(0.35, 0.55),
    epsilon U(0.02, 0.1)."""
    t, q, r, e = [], [], [], []
    for _ in range(n_atoms):
        t.append(rng.next_index(n_types))
        q.append(rng.uniform(-0.4, 0.4))
        r.append(rng.uniform(0.35, 0.55))
        e.append(rng.uniform(0.02, 0.1))
    return LigandParams(np.array(t), np.array(q), np.array(r), np.array(e))


def random_receptor_fields(rng: RngStream, n_sites: int, n_types: int) -> ReceptorFields:
    """Synthetic receptor chemistry: per site charge U(-0.5, 0.5) and volume
    U(0.5, 1.5); type 0 has scales (1, 1) (== the reference's analytic well),
    type t > 0 depth scale U(0.5, 1.5) and distance scale U(0.8, 1.2)."""
    q = [rng.uniform(-0.5, 0.5) for _ in range(n_sites)]
    v = [rng.uniform(0.5, 1.5) for _ in range(n_sites)]
    ds, dd = [1.0], [1.0]
    for _ in range(1, n_types):
        ds.append(rng.uniform(0.5, 1.5))
        dd.append(rng.uniform(0.8, 1.2))
    return ReceptorFields(np.array(q), np.array(v), np.array(ds), np.array(dd))


def centered_grid(n: int, spacing: float, n_types: int, center=(0.0, 0.0, 0.0)) -> Grid:
    """An n^3 lattice centred on `center` (C4: n=126, spacing 0.375)."""
    half = 0.5 * (n - 1) * spacing
    return Grid((n, n, n), n_types, tuple(c - half for c in center), spacing)
