"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module draws graphs and internal opinions only; it holds none of the
Friedkin–Johnsen arithmetic.  The C side
(`fjgen.c`, OpenMP) is built by `__graft_entry__.build()` into
`fjgen/libfjgen.so`.

Every builder returns a :class:`Problem` whose graph is the C-ABI's in-CSR
(row v lists the u with an arc u→v, i.e. u listens to v).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _CSR(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64),
                ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("col", ctypes.POINTER(ctypes.c_int32))]


def build_lib(force: bool = False) -> str:
    so = os.path.join(_HERE, "libfjgen.so")
    src = os.path.join(_HERE, "fjgen.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        cmd = f"gcc -O2 -fopenmp -fPIC -shared -o {so} {src} -lm"
        if os.system(cmd) != 0:
            raise RuntimeError("building libfjgen.so failed: " + cmd)
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build_lib())
        i64, u64, d, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        P = ctypes.c_void_p
        L.fjgen_er.argtypes = [i64, d, u64, ctypes.POINTER(_CSR)]
        L.fjgen_rmat.argtypes = [i32, i64, d, d, d, u64, ctypes.POINTER(_CSR)]
        L.fjgen_chunglu.argtypes = [i64, d, d, d, u64, ctypes.POINTER(_CSR), P]
        L.fjgen_lattice.argtypes = [i64, d, u64, ctypes.POINTER(_CSR)]
        for f in (L.fjgen_er, L.fjgen_rmat, L.fjgen_chunglu, L.fjgen_lattice):
            f.restype = i32
        L.fjgen_weights.argtypes = [i64, P, P, u64, P]
        L.fjgen_opinions.argtypes = [i64, i32, d, d, u64, P]
        L.fjgen_zero_mask.argtypes = [i64, i64, u64, P]
        L.fjgen_free.argtypes = [P]
        L.fjgen_u01.argtypes = [u64, u64, u64]
        L.fjgen_u01.restype = d
        L.fjgen_num_threads.restype = i32
        _LIB = L
    return _LIB


def _take(csr: _CSR):
    n, m = csr.n, csr.m
    rp = np.ctypeslib.as_array(csr.row_ptr, shape=(n + 1,)).copy()
    col = np.ctypeslib.as_array(csr.col, shape=(max(m, 1),))[:m].copy()
    lib().fjgen_free(ctypes.cast(csr.row_ptr, ctypes.c_void_p))
    lib().fjgen_free(ctypes.cast(csr.col, ctypes.c_void_p))
    return rp, col


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Problem:
    """One FJ instance: in-CSR graph (+optional fp32 weights) and fp32 s."""
    name: str
    n: int
    row_ptr: np.ndarray          # int64[n+1]
    col: np.ndarray              # int32[m]
    w: np.ndarray | None         # float32[m] or None (unit weights)
    s: np.ndarray                # float32[n]
    directed: bool
    meta: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.row_ptr[-1])


# ------------------------------------------------------------------ graphs
def er_graph(n: int, avg_deg: float, seed: int):
    c = _CSR()
    p = avg_deg / (n - 1)
    if lib().fjgen_er(n, p, seed, ctypes.byref(c)) != 0:
        raise MemoryError("fjgen_er")
    return _take(c)


def rmat_graph(scale: int, edge_factor: int, seed: int, abcd=(0.57, 0.19, 0.19, 0.05)):
    c = _CSR()
    a, b, cc, _ = abcd
    if lib().fjgen_rmat(scale, edge_factor, a, b, cc, seed, ctypes.byref(c)) != 0:
        raise MemoryError("fjgen_rmat")
    return _take(c)


def chunglu_graph(n: int, gamma: float, avg_deg: float, seed: int, wmax: float | None = None):
    c = _CSR()
    wmax = float(np.sqrt(n * avg_deg)) if wmax is None else wmax
    if lib().fjgen_chunglu(n, gamma, avg_deg, wmax, seed, ctypes.byref(c), None) != 0:
        raise MemoryError("fjgen_chunglu")
    return _take(c)


def chunglu_expected_degrees(n: int, gamma: float, avg_deg: float, wmax: float | None = None):
    """Expected degrees w_i of the Chung–Lu model (tests the generator only)."""
    wmax = float(np.sqrt(n * avg_deg)) if wmax is None else wmax
    c = _CSR()
    w = np.empty(n, np.float64)
    # tiny run with a large seed; the degrees do not depend on the seed
    lib().fjgen_chunglu(n, gamma, avg_deg, wmax, 0, ctypes.byref(c), _ptr(w))
    _take(c)
    return w


def lattice_graph(N: int, frac: float, seed: int):
    c = _CSR()
    if lib().fjgen_lattice(N, frac, seed, ctypes.byref(c)) != 0:
        raise MemoryError("fjgen_lattice")
    return _take(c)


def arc_weights(row_ptr, col, seed: int) -> np.ndarray:
    n = len(row_ptr) - 1
    w = np.empty(len(col), np.float32)
    lib().fjgen_weights(n, _ptr(row_ptr), _ptr(col), seed, _ptr(w))
    return w


# ---------------------------------------------------------------- opinions
def uniform(n, seed, lo=0.0, hi=1.0):
    s = np.empty(n, np.float32)
    lib().fjgen_opinions(n, 0, lo, hi, seed, _ptr(s))
    return s


def beta25(n, seed):
    s = np.empty(n, np.float32)
    lib().fjgen_opinions(n, 1, 0.0, 0.0, seed, _ptr(s))
    return s


def step_noise(N, seed, sd=0.1):
    s = np.empty(N * N, np.float32)
    lib().fjgen_opinions(N * N, 2, float(N), sd, seed, _ptr(s))
    return s


def exponential(n, seed, x_min=1.0):
    s = np.empty(n, np.float32)
    lib().fjgen_opinions(n, 3, x_min, 0.0, seed, _ptr(s))
    return s


def pareto(n, seed, alpha=2.5, x_min=1.0):
    s = np.empty(n, np.float32)
    lib().fjgen_opinions(n, 4, x_min, alpha, seed, _ptr(s))
    return s


def zero_mask(s, count, seed):
    lib().fjgen_zero_mask(len(s), count, seed, _ptr(s))
    return s


# ----------------------------------------------------------------- configs
CONFIG_SEEDS = {1: 101, 2: 202, 3: 303, 4: 404, 5: 505}

#: solve parameters per config (BASELINE.json configs).  `tuned`
#: is reading R10's tuned ω: the paper's fewest-updates heuristic run by
#: the ORACLE (tests/harness/omega_tune.py → profiles/r02_oracle_omega_tune.jsonl;
#: values copied from there, no arithmetic here).  C4's ω list is BASELINE's own.
CONFIG_SOLVE = {
    1: dict(eps=1e-6, omegas=[1.0, 1.5], tuned=1.5),
    2: dict(eps=1e-6, omegas=[1.0, 1.55], tuned=1.55),
    3: dict(eps=1e-6, omegas=[1.0, 1.6], tuned=1.6),
    4: dict(eps=1e-6, omegas=[1.0, 1.2, 1.4, 1.6, 1.8], tuned=None),
    5: dict(eps=1e-6, omegas=[1.0, 1.25, 1.3], tuned=1.3),
}


def config(cid: int, shrink: int = 0) -> Problem:
    """BASELINE.json config `cid` (1-based).  `shrink` > 0 builds the same
    recipe at a smaller size (scale − shrink, n / 4**shrink, N / 2**shrink) for
    oracle-sized parity cases."""
    seed = CONFIG_SEEDS[cid]
    if cid == 1:
        n = max(16, 10_000 >> (2 * shrink))
        rp, col = er_graph(n, 10.0, seed)
        s = uniform(n, seed)
        return Problem(f"C1-ER(n={n})", n, rp, col, None, s, False,
                       dict(seed=seed, kind="er", avg_deg=10))
    if cid == 2:
        scale = 20 - 2 * shrink
        rp, col = rmat_graph(scale, 16, seed)
        n = 1 << scale
        s = uniform(n, seed)
        return Problem(f"C2-RMAT{scale}", n, rp, col, None, s, True,
                       dict(seed=seed, kind="rmat", scale=scale))
    if cid == 3:
        n = 1 << (22 - 2 * shrink)
        rp, col = chunglu_graph(n, 2.1, 20.0, seed)
        s = uniform(n, seed, -1.0, 1.0)
        zero_mask(s, n // 2, seed)
        return Problem(f"C3-ChungLu(n={n})", n, rp, col, None, s, False,
                       dict(seed=seed, kind="chunglu", gamma=2.1, avg_deg=20))
    if cid == 4:
        scale = 24 - 2 * shrink
        rp, col = rmat_graph(scale, 16, seed)
        n = 1 << scale
        w = arc_weights(rp, col, seed)
        s = beta25(n, seed)
        return Problem(f"C4-RMAT{scale}w", n, rp, col, w, s, True,
                       dict(seed=seed, kind="rmat", scale=scale, weighted=True))
    if cid == 5:
        N = 4096 >> shrink
        rp, col = lattice_graph(N, 0.01, seed)
        s = step_noise(N, seed, 0.1)
        return Problem(f"C5-lattice({N}x{N})", N * N, rp, col, None, s, False,
                       dict(seed=seed, kind="lattice", N=N, shortcut_frac=0.01, noise_sd=0.1))
    raise ValueError(cid)


def num_threads() -> int:
    return lib().fjgen_num_threads()


# --------------------------------------------------- sharded inputs (row f4)
def to_out_csr(row_ptr, col, w=None):
    """Transpose an in-CSR (row v lists the u with u→v) into the out-CSR
    (row u lists the v with u→v, ascending): index shuffling only."""
    row_ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col, np.int32)
    n = len(row_ptr) - 1
    v = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    order = np.lexsort((v, col.astype(np.int64)))
    orp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(col, minlength=n), out=orp[1:])
    ocol = v[order].astype(np.int32)
    ow = None if w is None else np.asarray(w, np.float32)[order]
    return orp, ocol, ow


def shard_rows(out_rp, out_col, out_w, begin, rank: int):
    """Rank `rank`'s rows [begin[rank], begin[rank+1]) of an out-CSR, row_ptr
    rebased to 0, columns kept global."""
    a, b = int(begin[rank]), int(begin[rank + 1])
    k0, k1 = int(out_rp[a]), int(out_rp[b])
    rp = (np.asarray(out_rp[a:b + 1], np.int64) - k0).copy()
    col = np.ascontiguousarray(out_col[k0:k1], np.int32)
    w = None if out_w is None else np.ascontiguousarray(out_w[k0:k1], np.float32)
    return rp, col, w
