"""Python binding of libfj (include/fj.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module
converts arrays to pointers and C structs to Python values.  It never computes
on the host and has no fallback: if ``libfj.so`` is missing or fails to load,
every entry point raises.

Arrays may be numpy arrays (host memory) or torch tensors (host or CUDA); the
library detects the memory space of each pointer (fj.h "Memory").
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FJ_LIB_PATH") or os.path.join(_HERE, "libfj.so")
_LIB = None

FJ_OK, FJ_ERR_INVALID, FJ_ERR_NUMERIC, FJ_ERR_CUDA = 0, 2, 3, 4
METHODS = {"auto": 0, "async": 1, "colored": 2, "push": 3}

#: every symbol include/fj.h declares
EXPORTS = ("fj_graph_create", "fj_graph_destroy", "fj_graph_get_info", "fj_solve", "fj_solve_ex",
           "fj_measures", "fj_measures_ex", "fj_opts_default", "fj_last_error",
           "fj_abi_version", "fj_kernel_launches", "fj_omega_opt", "fj_omega_sweep",
           "fj_solve_batch", "fj_solve_batch_omega", "fj_shard_plan", "fj_comm_unique_id", "fj_comm_create",
           "fj_comm_create_local", "fj_comm_create_loopback", "fj_comm_destroy", "fj_shard_create",
           "fj_shard_connect",
           "fj_shard_solve", "fj_shard_measures", "fj_shard_destroy", "fj_shard_info", "fj_gather_probe")


class FJError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[fj status {status}] {msg}")
        self.status = status


class _Opts(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double), ("c", ctypes.c_double), ("method", ctypes.c_int),
                ("max_sweeps", ctypes.c_int), ("cert_rounds", ctypes.c_int),
                ("certify", ctypes.c_int), ("zprime_out", ctypes.c_void_p),
                ("z_init", ctypes.c_void_p), ("tail_frac", ctypes.c_double),
                ("coloring", ctypes.c_int), ("push_compact", ctypes.c_int),
                ("push_sparse_div", ctypes.c_int), ("shadow", ctypes.c_int),
                ("slices", ctypes.c_int), ("frontier", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("phases", ctypes.c_int64),
                ("relaxations", ctypes.c_int64), ("edge_updates", ctypes.c_int64),
                ("rows_read", ctypes.c_int64), ("arcs_read", ctypes.c_int64),
                ("cert_rounds", ctypes.c_int64), ("cert_ratio", ctypes.c_double),
                ("c", ctypes.c_double), ("eps_prime", ctypes.c_double),
                ("colors", ctypes.c_int), ("status", ctypes.c_int), ("reason", ctypes.c_int),
                ("solve_ms", ctypes.c_double), ("sweep_ms", ctypes.c_double),
                ("cert_ms", ctypes.c_double), ("shadow_sweeps", ctypes.c_int64),
                ("shadow_ms", ctypes.c_double), ("frontier_rounds", ctypes.c_int64),
                ("frontier_pushes", ctypes.c_int64), ("frontier_ms", ctypes.c_double)]


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("directed", ctypes.c_int),
                ("weighted", ctypes.c_int), ("max_out_degree", ctypes.c_int64),
                ("empty_rows", ctypes.c_int64), ("tasks", ctypes.c_int64),
                ("colors", ctypes.c_int), ("num_sms", ctypes.c_int)]


class _Measures(ctypes.Structure):
    _fields_ = [("polarization", ctypes.c_double), ("disagreement", ctypes.c_double),
                ("internal_conflict", ctypes.c_double), ("controversy", ctypes.c_double)]


def lib():
    """Load libfj.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, d, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.fj_graph_create.argtypes = [i64, i64, P, P, P, i, P, ctypes.POINTER(P)]
        L.fj_graph_destroy.argtypes = [P]
        L.fj_graph_get_info.argtypes = [P, ctypes.POINTER(_Info)]
        L.fj_solve.argtypes = [P, P, d, d, P]
        L.fj_solve_ex.argtypes = [P, P, d, d, ctypes.POINTER(_Opts), P, ctypes.POINTER(_Stats)]
        L.fj_measures.argtypes = [P, P, ctypes.POINTER(d), ctypes.POINTER(d)]
        L.fj_measures_ex.argtypes = [P, P, P, ctypes.POINTER(_Measures)]
        L.fj_opts_default.argtypes = [ctypes.POINTER(_Opts)]
        L.fj_opts_default.restype = None
        L.fj_last_error.restype = ctypes.c_char_p
        L.fj_kernel_launches.restype = ctypes.c_int64
        L.fj_solve_batch.argtypes = [P, P, i, d, d, ctypes.POINTER(_Opts), P,
                                     ctypes.POINTER(_Stats)]
        L.fj_omega_opt.argtypes = [P, i, d, ctypes.POINTER(d), ctypes.POINTER(d)]
        L.fj_omega_sweep.argtypes = [P, P, d, d, d, d, i, ctypes.POINTER(d), P,
                                     ctypes.POINTER(i)]
        L.fj_solve_batch_omega.argtypes = [P, P, i, P, d, ctypes.POINTER(_Opts), P,
                                           ctypes.POINTER(_Stats), P, P]
        PP = ctypes.POINTER(P)
        L.fj_shard_plan.argtypes = [i64, P, i, P]
        L.fj_comm_unique_id.argtypes = [P]
        L.fj_comm_create.argtypes = [P, i, i, PP]
        L.fj_comm_create_local.argtypes = [i, PP]
        L.fj_comm_create_loopback.argtypes = [i, PP]
        L.fj_comm_destroy.argtypes = [P]
        L.fj_shard_create.argtypes = [P, i, i64, P, P, P, P, i, PP]
        L.fj_shard_connect.argtypes = [PP, i]
        L.fj_shard_solve.argtypes = [PP, i, PP, d, d, ctypes.POINTER(_Opts), PP, PP,
                                     ctypes.POINTER(_Stats)]
        L.fj_shard_measures.argtypes = [PP, i, PP, PP, ctypes.POINTER(_Measures)]
        L.fj_shard_destroy.argtypes = [P]
        L.fj_gather_probe.argtypes = [P, i, ctypes.POINTER(d)]
        L.fj_shard_info.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        for f in ("fj_graph_create", "fj_graph_destroy", "fj_graph_get_info", "fj_solve",
                  "fj_solve_ex", "fj_measures", "fj_measures_ex", "fj_omega_opt",
                  "fj_omega_sweep", "fj_solve_batch", "fj_solve_batch_omega", "fj_shard_plan",
                  "fj_comm_unique_id",
                  "fj_comm_create", "fj_comm_create_local", "fj_comm_create_loopback",
                  "fj_comm_destroy",
                  "fj_shard_create", "fj_shard_connect", "fj_shard_solve",
                  "fj_shard_measures", "fj_shard_destroy", "fj_gather_probe", "fj_shard_info"):
            getattr(L, f).restype = i
        _LIB = L
    return _LIB


def _check(st: int):
    if st != FJ_OK:
        raise FJError(st, lib().fj_last_error().decode(errors="replace"))


def _ptr(a):
    """Pointer of a numpy array or torch tensor (None → NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def _dtype_ok(a, name: str, kind: str, numel: int | None = None):
    """dtype check, and (``numel``) the element count the library will read or
    write through the pointer: a short buffer would be overrun on the device
    or, for host outputs, by the device→host copy."""
    if a is None:
        return
    dt = str(a.dtype)
    if kind not in dt:
        raise TypeError(f"{name} must be {kind}, got {dt}")
    if numel is not None:
        got = int(a.numel()) if hasattr(a, "numel") else int(a.size)
        if got < numel:
            raise ValueError(f"{name} has {got} elements, the call needs {numel}")
        if hasattr(a, "is_contiguous") and not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if hasattr(a, "flags") and not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")


def _stream_of(*arrays):
    for a in arrays:
        if a is not None and getattr(a, "is_cuda", False):
            import torch
            return ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
    return None


@dataclass
class SolveStats:
    sweeps: int
    phases: int
    relaxations: int
    edge_updates: int
    rows_read: int
    arcs_read: int
    cert_rounds: int
    cert_ratio: float
    c: float
    eps_prime: float
    colors: int
    status: int
    reason: int
    solve_ms: float
    sweep_ms: float
    cert_ms: float
    shadow_sweeps: int = 0
    shadow_ms: float = 0.0
    frontier_rounds: int = 0
    frontier_pushes: int = 0
    frontier_ms: float = 0.0


class Graph:
    """Owning handle of an ``fj_graph_t`` (§8 row a1).

    ``row_ptr`` int64[n+1], ``col`` int32[m], ``w`` float32[m] or None: the
    in-CSR (row v lists the u with an arc u→v, u listens to v)."""

    def __init__(self, n, row_ptr, col, w=None, directed=True, stream=None):
        _dtype_ok(row_ptr, "row_ptr", "int64", int(n) + 1)
        nnz = int(row_ptr[int(n)])
        _dtype_ok(col, "col", "int32", nnz)
        _dtype_ok(w, "w", "float32", nnz)
        self._h = ctypes.c_void_p()
        st = stream if stream is not None else _stream_of(row_ptr, col, w)
        _check(lib().fj_graph_create(int(n), nnz, _ptr(row_ptr), _ptr(col), _ptr(w),
                                     1 if directed else 0, st, ctypes.byref(self._h)))
        self.n = int(n)
        self.directed = bool(directed)

    def info(self) -> dict:
        i = _Info()
        _check(lib().fj_graph_get_info(self._h, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in _Info._fields_}

    def close(self):
        if self._h:
            lib().fj_graph_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def solve(g: Graph, s, z_out, eps: float, omega: float = 1.0, method: str = "auto",
          sigma: float = 1e-5, c: float = 0.0, max_sweeps: int = 0, cert_rounds: int = -1,
          certify: bool = True, zprime_out=None, raise_on_numeric: bool = True,
          z_init=None, tail_frac: float = -1.0, coloring: str = "spec",
          push_compact: bool = False, push_sparse_div: int = 8,
          shadow: int = -1, slices: int = -1, frontier: int = -1) -> SolveStats:
    """fj_solve_ex: writes z into ``z_out`` (float32[n]); returns the stats.
    ``shadow``: fj_opts.shadow (1 = shadow sweeps, 0 = fp64 only, −1 = library default).
    ``slices``: fj_opts.slices (nonzero = short rows as row slices, 0 = as warp tiles).
    ``frontier``: fj_opts.frontier (0 = off, > 0 = thin-sweep threshold in rows, −1 = default).
    ``z_init`` (float64[n], optional): warm start / resume from an earlier z.
    Schedule options (fj_opts): ``tail_frac`` (COLORED tail merge, R23; 0 =
    exact multicolor SOR), ``coloring`` ("spec" or "jp"), ``push_compact`` /
    ``push_sparse_div`` (PUSH frontier)."""
    _dtype_ok(s, "s", "float32", g.n)
    _dtype_ok(z_out, "z_out", "float32", g.n)
    _dtype_ok(zprime_out, "zprime_out", "float64", g.n)
    o = _Opts()
    lib().fj_opts_default(ctypes.byref(o))
    o.sigma, o.c, o.method = sigma, c, METHODS[method]
    o.max_sweeps, o.cert_rounds, o.certify = max_sweeps, cert_rounds, int(certify)
    o.tail_frac, o.coloring = float(tail_frac), {"spec": 0, "jp": 1}[coloring]
    o.push_compact, o.push_sparse_div = int(bool(push_compact)), int(push_sparse_div)
    o.shadow = int(shadow)
    o.slices = int(slices)
    o.frontier = int(frontier)
    zp = _ptr(zprime_out)
    o.zprime_out = zp.value if zp is not None else None
    _dtype_ok(z_init, "z_init", "float64", g.n)
    zi = _ptr(z_init)
    o.z_init = zi.value if zi is not None else None
    st = _Stats()
    rc = lib().fj_solve_ex(g._h, _ptr(s), float(eps), float(omega), ctypes.byref(o),
                           _ptr(z_out), ctypes.byref(st))
    stats = SolveStats(**{k: getattr(st, k) for k, _ in _Stats._fields_})
    if rc == FJ_ERR_NUMERIC and not raise_on_numeric:
        return stats
    _check(rc)
    return stats


def solve_batch(g: Graph, S, Z_out, k: int, eps: float, omega: float = 1.0,
                sigma: float = 1e-5, max_sweeps: int = 0, raise_on_numeric: bool = True,
                method: str = "auto", tail_frac: float = -1.0, frontier: int = -1) -> SolveStats:
    """fj_solve_batch: k ≤ 8 opinion vectors (node-major fp32[n*k]) in one
    solve; AUTO runs ASYNC at ω = 1 or on directed graphs, else COLORED."""
    _dtype_ok(S, "S", "float32", g.n * int(k))
    _dtype_ok(Z_out, "Z_out", "float32", g.n * int(k))
    o = _Opts()
    lib().fj_opts_default(ctypes.byref(o))
    o.sigma, o.max_sweeps = sigma, max_sweeps
    o.method, o.tail_frac = METHODS[method], float(tail_frac)
    o.frontier = int(frontier)
    st = _Stats()
    rc = lib().fj_solve_batch(g._h, _ptr(S), int(k), float(eps), float(omega), ctypes.byref(o),
                              _ptr(Z_out), ctypes.byref(st))
    stats = SolveStats(**{kk: getattr(st, kk) for kk, _ in _Stats._fields_})
    if rc == FJ_ERR_NUMERIC and not raise_on_numeric:
        return stats
    _check(rc)
    return stats


def solve_batch_omega(g: Graph, s, Z_out, omegas, eps: float, sigma: float = 1e-5,
                      max_sweeps: int = 0, method: str = "auto", tail_frac: float = -1.0):
    """fj_solve_batch_omega: one opinion vector at k ≤ 8 values of ω in one
    solve.  Returns (stats, relaxations per ω, status per ω)."""
    k = len(omegas)
    _dtype_ok(s, "s", "float32", g.n)
    _dtype_ok(Z_out, "Z_out", "float32", g.n * k)
    o = _Opts()
    lib().fj_opts_default(ctypes.byref(o))
    o.sigma, o.max_sweeps = sigma, max_sweeps
    o.method, o.tail_frac = METHODS[method], float(tail_frac)
    om = (ctypes.c_double * k)(*[float(x) for x in omegas])
    rel = (ctypes.c_int64 * k)()
    sts = (ctypes.c_int * k)()
    st = _Stats()
    rc = lib().fj_solve_batch_omega(g._h, _ptr(s), k, om, float(eps), ctypes.byref(o),
                                    _ptr(Z_out), ctypes.byref(st), rel, sts)
    if rc != FJ_ERR_NUMERIC:
        _check(rc)
    stats = SolveStats(**{kk: getattr(st, kk) for kk, _ in _Stats._fields_})
    return stats, list(rel), list(sts)


def solve_simple(g: Graph, s, z_out, eps: float, omega: float = 1.0):
    """The plain ABI call fj_solve(graph, s, eps, omega, z_out)."""
    _check(lib().fj_solve(g._h, _ptr(s), float(eps), float(omega), _ptr(z_out)))


def measures(g: Graph, z, s=None) -> dict:
    """fj_measures_ex: P, D (and I, C) of Table tab:measures."""
    _dtype_ok(z, "z", "float32", g.n)
    _dtype_ok(s, "s", "float32", g.n)
    m = _Measures()
    _check(lib().fj_measures_ex(g._h, _ptr(z), _ptr(s), ctypes.byref(m)))
    return dict(P=m.polarization, D=m.disagreement, I=m.internal_conflict, C=m.controversy)


def measures_pd(g: Graph, z):
    """The plain ABI call fj_measures(graph, z, &P, &D)."""
    _dtype_ok(z, "z", "float32", g.n)
    P, D = ctypes.c_double(), ctypes.c_double()
    _check(lib().fj_measures(g._h, _ptr(z), ctypes.byref(P), ctypes.byref(D)))
    return P.value, D.value


def gather_probe(g: Graph, reps: int = 10) -> float:
    """fj_gather_probe: ms per pass of the sweep's memory pattern (stream every
    arc, gather one fp64 per arc) — the practical ceiling of a sweep."""
    ms = ctypes.c_double()
    _check(lib().fj_gather_probe(g._h, int(reps), ctypes.byref(ms)))
    return ms.value


def omega_opt(g: Graph, max_iters: int = 2000, tol: float = 1e-9):
    """fj_omega_opt: (μ, ω_opt) — Eq. optimal-omega, μ by power iteration."""
    mu, om = ctypes.c_double(), ctypes.c_double()
    _check(lib().fj_omega_opt(g._h, int(max_iters), float(tol), ctypes.byref(mu),
                              ctypes.byref(om)))
    return mu.value, om.value


def omega_sweep(g: Graph, s, eps: float, lo: float = 1.0, hi: float = 1.95, step: float = 0.05,
                method: str = "auto"):
    """fj_omega_sweep: the paper's fewest-updates heuristic.
    Returns (best ω, [(ω, relaxations, status), ...])."""
    cap = int(round((hi - lo) / step)) + 2
    table = (ctypes.c_double * (3 * cap))()
    n = ctypes.c_int(cap)
    best = ctypes.c_double()
    _check(lib().fj_omega_sweep(g._h, _ptr(s), float(eps), float(lo), float(hi), float(step),
                                METHODS[method], ctypes.byref(best), table, ctypes.byref(n)))
    rows = [(table[3 * i], int(table[3 * i + 1]), int(table[3 * i + 2])) for i in range(n.value)]
    return best.value, rows


# ----------------------------------------------------------------- sharded (f4)
def shard_plan(row_ptr, world: int):
    """fj_shard_plan: arc-balanced 1-D partition of the out-CSR row_ptr (host
    int64[n+1], contiguous); returns begin as a list of world+1 ints."""
    _dtype_ok(row_ptr, "row_ptr", "int64")
    begin = (ctypes.c_int64 * (world + 1))()
    _check(lib().fj_shard_plan(len(row_ptr) - 1, _ptr(row_ptr), int(world), begin))
    return list(begin)


def comm_unique_id() -> bytes:
    """fj_comm_unique_id: the 128-byte NCCL id (create on one rank, broadcast)."""
    buf = (ctypes.c_char * 128)()
    _check(lib().fj_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """Owning handle of an ``fj_comm_t``: ``Comm.in_process(world)`` (all
    shards in this process, current device) or ``Comm.nccl(uid, rank, world)``."""

    def __init__(self, h, world: int, rank: int, in_process: bool):
        self._h, self.world, self.rank, self.in_process_ = h, world, rank, in_process

    @classmethod
    def in_process(cls, world: int, loopback: bool = False) -> "Comm":
        """All shards in this process.  ``loopback``: run the NCCL path's send
        lists and pack kernel with device copies in place of NCCL (tests)."""
        h = ctypes.c_void_p()
        fn = lib().fj_comm_create_loopback if loopback else lib().fj_comm_create_local
        _check(fn(int(world), ctypes.byref(h)))
        return cls(h, int(world), 0, True)

    @classmethod
    def nccl(cls, uid: bytes, rank: int, world: int) -> "Comm":
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        h = ctypes.c_void_p()
        buf = (ctypes.c_char * 128).from_buffer_copy(uid)
        _check(lib().fj_comm_create(buf, int(rank), int(world), ctypes.byref(h)))
        return cls(h, int(world), int(rank), False)

    def close(self):
        if self._h:
            lib().fj_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Shard:
    """Owning handle of an ``fj_shard_t``: rank ``rank``'s OUT-rows
    (``row_ptr`` int64[n_local+1], ``col`` int32 GLOBAL ids, ``w`` float32 or
    None) of an n-node graph partitioned by ``begin``."""

    def __init__(self, comm: Comm, rank: int, n: int, begin, row_ptr, col, w=None,
                 directed=True):
        _dtype_ok(row_ptr, "row_ptr", "int64")
        _dtype_ok(col, "col", "int32")
        _dtype_ok(w, "w", "float32")
        self._b = (ctypes.c_int64 * len(begin))(*[int(x) for x in begin])
        self._h = ctypes.c_void_p()
        _check(lib().fj_shard_create(comm._h, int(rank), int(n), self._b, _ptr(row_ptr),
                                     _ptr(col), _ptr(w), 1 if directed else 0,
                                     ctypes.byref(self._h)))
        self.comm, self.rank, self.n = comm, int(rank), int(n)
        self.n_local = int(self._b[rank + 1] - self._b[rank])

    def info(self):
        """(n_local, halo): owned rows and, after connect, the remote values
        received per sweep."""
        nl, h = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().fj_shard_info(self._h, ctypes.byref(nl), ctypes.byref(h)))
        return nl.value, h.value

    def close(self):
        if self._h:
            lib().fj_shard_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _handles(shards):
    return (ctypes.c_void_p * len(shards))(*[sh._h.value for sh in shards])


def _ptrs(arrs):
    if arrs is None:
        return None
    return (ctypes.c_void_p * len(arrs))(*[(_ptr(a).value if a is not None else None)
                                           for a in arrs])


def shard_connect(shards):
    """fj_shard_connect (collective over this process's shards, rank order)."""
    _check(lib().fj_shard_connect(_handles(shards), len(shards)))


def shard_solve(shards, s_list, z_list, eps: float, omega: float = 1.0, sigma: float = 1e-5,
                max_sweeps: int = 0, cert_rounds: int = -1, certify: bool = True,
                zprime_list=None, raise_on_numeric: bool = True) -> SolveStats:
    """fj_shard_solve: per-shard float32 slices in, float32 (and optional fp64
    ẑ') slices out; stats aggregated over ranks."""
    for a in s_list:
        _dtype_ok(a, "s", "float32")
    for a in z_list:
        _dtype_ok(a, "z_out", "float32")
    o = _Opts()
    lib().fj_opts_default(ctypes.byref(o))
    o.sigma, o.max_sweeps, o.cert_rounds, o.certify = sigma, max_sweeps, cert_rounds, int(certify)
    st = _Stats()
    rc = lib().fj_shard_solve(_handles(shards), len(shards), _ptrs(s_list), float(eps),
                              float(omega), ctypes.byref(o), _ptrs(z_list), _ptrs(zprime_list),
                              ctypes.byref(st))
    stats = SolveStats(**{k: getattr(st, k) for k, _ in _Stats._fields_})
    if rc == FJ_ERR_NUMERIC and not raise_on_numeric:
        return stats
    _check(rc)
    return stats


def shard_measures(shards, z_list, s_list=None) -> dict:
    """fj_shard_measures: P, D, I, C of a sharded z."""
    m = _Measures()
    _check(lib().fj_shard_measures(_handles(shards), len(shards), _ptrs(z_list), _ptrs(s_list),
                                   ctypes.byref(m)))
    return dict(P=m.polarization, D=m.disagreement, I=m.internal_conflict, C=m.controversy)
