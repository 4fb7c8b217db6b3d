"""CPU oracle of the FJ hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path (``paper_2507_14864_b200``) and never
imports it.

Layers:

* plain definition — :func:`dense_solve`: z = (I+L)^{-1} s (Lemma 1)
  by LAPACK Gaussian elimination with partial pivoting in fp64 (n ≤ ~3000);
* the algorithm — :func:`solve`: ImprovedBLI / ImprovedBLISOR (Alg. 2 around
  Alg. 1 / Alg. 3) verbatim with a FIFO queue
  in fp64, single thread, in ``oracle.c``;
* the residual certificate — :func:`certificate` (Lemma 3, Lemma 6
  P:474);
* the measures — :func:`measures` (Table ``tab:measures`` P:96–110).

Pinned by ``tests/test_oracle_pins.py`` (closed forms, dense GE, Lemma 3/4/6
invariants, golden fixtures).  Every function is pinned; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SIGMA = 1e-5  # σ = c = 1e-5 (§6 "Experiment Settings")


class _Stats(ctypes.Structure):
    _fields_ = [("pushes", ctypes.c_int64), ("touched", ctypes.c_int64),
                ("cert_rounds", ctypes.c_int64), ("cert_ratio", ctypes.c_double),
                ("c", ctypes.c_double), ("eps_prime", ctypes.c_double),
                ("seconds", ctypes.c_double), ("status", ctypes.c_int)]


def build_lib(force: bool = False) -> str:
    so = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        cmd = (f"gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared "
               f"-o {so} {src} -lm")
        if os.system(cmd) != 0:
            raise RuntimeError("building liboracle.so failed: " + cmd)
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build_lib())
        P, i64, d, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.or_degrees.argtypes = [i64, P, P, P, P]
        L.or_thresholds.argtypes = [i64, P, d, d, d, P, P, P, P]
        L.or_improved.argtypes = [i64, P, P, P, P, d, d, d, d, i32, i64, i32, P, P, P,
                                  ctypes.POINTER(_Stats)]
        L.or_improved.restype = i32
        L.or_bound_local_iter.argtypes = [i64, P, P, P, P, P, P, P, P, i64, i64,
                                          ctypes.POINTER(_Stats)]
        L.or_bound_local_iter.restype = i32
        L.or_certificate.argtypes = [i64, P, P, P, P, P, P, P, P]
        L.or_certificate.restype = d
        L.or_measures.argtypes = [i64, P, P, P, P, P, i32, P]
        L.or_fj_iterate.argtypes = [i64, P, P, P, P, i64, P]
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _graph(rp, col, w):
    rp = np.ascontiguousarray(rp, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    w = None if w is None else np.ascontiguousarray(w, np.float32)
    return rp, col, w


@dataclass
class Result:
    z: np.ndarray          # fp64, unshifted ẑ
    zprime: np.ndarray     # fp64 ẑ' = ẑ + c
    r: np.ndarray          # final tracked residual (shifted system)
    pushes: int
    touched: int           # edge updates
    cert_rounds: int
    cert_ratio: float
    c: float
    eps_prime: float
    seconds: float
    status: int


def solve(rp, col, w, s, eps, omega=1.0, sigma=SIGMA, c=None, alg=None,
          max_pushes=-1, max_cert_rounds=3) -> Result:
    """ImprovedBLI (alg=1; ω must be 1) or ImprovedBLISOR (alg=3), fp64 FIFO.

    ``alg`` defaults to 1 at ω = 1 and 3 otherwise.  ``c`` overrides the shift
    (default σ + max(0, −min s), reading R5)."""
    rp, col, w = _graph(rp, col, w)
    s = np.ascontiguousarray(s, np.float32)
    n = len(rp) - 1
    if alg is None:
        alg = 1 if omega == 1.0 else 3
    if alg == 1 and omega != 1.0:
        raise ValueError("Algorithm 1 has no ω")
    z = np.empty(n); zp = np.empty(n); r = np.empty(n)
    st = _Stats()
    lib().or_improved(n, _p(rp), _p(col), _p(w), _p(s), eps, sigma,
                      -1.0 if c is None else float(c), float(omega), int(alg),
                      int(max_pushes), int(max_cert_rounds), _p(z), _p(zp), _p(r),
                      ctypes.byref(st))
    return Result(z, zp, r, st.pushes, st.touched, st.cert_rounds, st.cert_ratio, st.c,
                  st.eps_prime, st.seconds, st.status)


def degrees(rp, col, w):
    """d_u = Σ_v a_uv, from the in-CSR."""
    rp, col, w = _graph(rp, col, w)
    n = len(rp) - 1
    d = np.empty(n)
    lib().or_degrees(n, _p(rp), _p(col), _p(w), _p(d))
    return d


def thresholds(s, eps, sigma=SIGMA, c=None):
    """(s', h, c, ε') of Alg. 2 with reading R5."""
    s = np.ascontiguousarray(s, np.float32)
    n = len(s)
    sp = np.empty(n); h = np.empty(n)
    cc = ctypes.c_double(); ep = ctypes.c_double()
    lib().or_thresholds(n, _p(s), eps, sigma, -1.0 if c is None else float(c), _p(sp), _p(h),
                        ctypes.byref(cc), ctypes.byref(ep))
    return sp, h, cc.value, ep.value


def certificate(rp, col, w, s, zprime, eps, sigma=SIGMA, c=None):
    """max_v |R_v|/h_v with R = s' − (I+L)ẑ' (compensated fp64) and R itself.

    This is the harness tool that certifies a GPU ẑ' independently: ratio ≤ 1
    ⇒ |z − ẑ| ≤ ε·max(|z|, σ) for every v (Lemma 6 P:474–478 + reading R5)."""
    rp, col, w = _graph(rp, col, w)
    n = len(rp) - 1
    d = degrees(rp, col, w)
    sp, h, _, _ = thresholds(s, eps, sigma, c)
    zp = np.ascontiguousarray(zprime, np.float64)
    R = np.empty(n)
    ratio = lib().or_certificate(n, _p(rp), _p(col), _p(w), _p(d), _p(sp), _p(zp), _p(h),
                                 _p(R))
    return ratio, R


def measures(rp, col, w, z, s=None, directed=False):
    """(P, D, I, C) of Table `tab:measures`, compensated fp64."""
    rp, col, w = _graph(rp, col, w)
    n = len(rp) - 1
    z = np.ascontiguousarray(z, np.float64)
    s = None if s is None else np.ascontiguousarray(s, np.float32)
    out = np.empty(4)
    lib().or_measures(n, _p(rp), _p(col), _p(w), _p(z), _p(s), int(bool(directed)), _p(out))
    return dict(P=out[0], D=out[1], I=out[2], C=out[3])


def fj_iterate(rp, col, w, s, iters):
    """Synchronous FJ update Eq. (1), `iters` steps from z = s."""
    rp, col, w = _graph(rp, col, w)
    n = len(rp) - 1
    s = np.ascontiguousarray(s, np.float32)
    z = np.empty(n)
    lib().or_fj_iterate(n, _p(rp), _p(col), _p(w), _p(s), int(iters), _p(z))
    return z


# ------------------------------------------------------------ dense layer
def dense_system(rp, col, w):
    """I + L = I + D − A with A[u, v] = a_uv for the in-CSR (R1)."""
    n = len(rp) - 1
    A = np.zeros((n, n))
    for v in range(n):
        for e in range(rp[v], rp[v + 1]):
            A[col[e], v] = 1.0 if w is None else float(w[e])
    return np.eye(n) + np.diag(A.sum(axis=1)) - A


def dense_solve(rp, col, w, s):
    """z = (I+L)^{-1} s (Lemma 1) by LU with partial pivoting (fp64)."""
    M = dense_system(rp, col, w)
    return np.linalg.solve(M, np.asarray(s, np.float64))


def omega_opt(mu: float) -> float:
    """ω_opt = 1 + (μ/(1+√(1−μ²)))² (Eq. optimal-omega)."""
    return 1.0 + (mu / (1.0 + np.sqrt(1.0 - mu * mu))) ** 2


def omega_grid(lo=1.0, hi=1.95, step=0.05):
    """The ω grid of the heuristic, visited from ω → 2⁻ down to 1;
    step 0.05 per reading R10 (P:625's 'step size of 0.5' read as garbled)."""
    k = int(round((hi - lo) / step))
    return [round(hi - i * step, 10) for i in range(k + 1)]


def omega_sweep(rp, col, w, s, eps, lo=1.0, hi=1.95, step=0.05, sigma=SIGMA, prune=True):
    """The paper's ω heuristic, verbatim on the oracle: "begin with
    ω → 2⁻ and iteratively reduce ω by a fixed step size until it reaches 1;
    the ω that achieves the minimum number of updates" — updates = pops of Q
    of ImprovedBLISOR (Alg. 2 + Alg. 3, FIFO, fp64).  Reading R10: grid
    1.95:−0.05:1.00, a diverging or unterminated ω costs +∞, ties go to the
    smaller ω (the later point of the downward walk).

    With ``prune`` a run is stopped once it exceeds the best count so far (it
    can no longer win; its cost is recorded as +∞ with status "pruned").
    Returns (best_omega, table) with table rows (ω, pushes or inf, status)."""
    best, best_cost, table = None, None, []
    for om in omega_grid(lo, hi, step):
        cap = best_cost if (prune and best_cost is not None) else -1
        res = solve(rp, col, w, s, eps, om, sigma=sigma, alg=3, max_pushes=cap)
        if res.status == 0 and res.cert_ratio <= 1.0:
            cost, status = res.pushes, "ok"
        else:
            cost = float("inf")
            status = "pruned" if (cap >= 0 and res.pushes >= cap) else "diverged"
        table.append((om, cost, status))
        if cost != float("inf") and (best_cost is None or cost <= best_cost):
            best, best_cost = om, cost           # ≤: ties go to the smaller ω
    return best, table


def jacobi_mu_dense(rp, col, w):
    """μ = ρ((I+D)^{-1}A) by dense eigenvalues (small n only)."""
    M = dense_system(rp, col, w)
    n = M.shape[0]
    diag = np.diag(M).copy()
    A = np.diag(diag) - M   # = A (off-diagonal part), since I+D = diag(M)
    J = A / diag[:, None]
    return float(np.max(np.abs(np.linalg.eigvals(J)))) if n else 0.0
