"""Closed-form equilibria z = (I+L)^{-1} s for special graphs — TEST
INFRASTRUCTURE ONLY (same import rule as the rest of ``oracle/``).

These are the plain definition (Lemma 1) written out for graphs whose
Laplacian is diagonalised or reduced by hand; they pin both the oracle (at small
n) and the GPU path at full size (the 4096² lattice of config 5).
"""
from __future__ import annotations

import numpy as np


def path_eigen(N: int, k: int):
    """Eigenpair of the path Laplacian on N nodes (Neumann ends):
    L_path cos(πk(x+½)/N) = λ_k cos(πk(x+½)/N), λ_k = 2 − 2cos(πk/N)."""
    x = np.arange(N)
    return np.cos(np.pi * k * (x + 0.5) / N), 2.0 - 2.0 * np.cos(np.pi * k / N)


def grid_mode(N: int, k: int, l: int, base: float = 0.5, amp: float = 0.4):
    """On the N×N 4-neighbour grid (id = y·N + x) with
    s = base + amp·φ_k(x)·φ_l(y), the equilibrium is
    z = base + amp·φ_k(x)φ_l(y)/(1 + λ_k + λ_l)  (L = L_path⊗I + I⊗L_path;
    constants are preserved since (I+L)^{-1} is row-stochastic).
    Returns (s, z) as fp64 arrays of length N²."""
    fx, lk = path_eigen(N, k)
    fy, ll = path_eigen(N, l)
    mode = np.outer(fy, fx).ravel()
    s = base + amp * mode
    z = base + amp * mode / (1.0 + lk + ll)
    return s, z


def thomas(a, b, c, f):
    """Tridiagonal solve (sub a, diag b, super c) by the Thomas algorithm."""
    n = len(b)
    cp = np.zeros(n); fp = np.zeros(n)
    cp[0] = c[0] / b[0]; fp[0] = f[0] / b[0]
    for i in range(1, n):
        den = b[i] - a[i] * cp[i - 1]
        cp[i] = c[i] / den if i < n - 1 else 0.0
        fp[i] = (f[i] - a[i] * fp[i - 1]) / den
    x = np.zeros(n)
    x[-1] = fp[-1]
    for i in range(n - 2, -1, -1):
        x[i] = fp[i] - cp[i] * x[i + 1]
    return x


def grid_rows_constant(N: int, f):
    """If s on the N×N grid depends only on x (s = f(x)), then z does too and
    solves the 1-D system (I + L_path) g = f (the y-couplings cancel).
    Returns z as an fp64 array of length N²."""
    f = np.asarray(f, np.float64)
    a = -np.ones(N); c = -np.ones(N)
    b = np.full(N, 3.0); b[0] = 2.0; b[-1] = 2.0
    if N == 1:
        b[0] = 1.0
    a[0] = 0.0; c[-1] = 0.0
    g = thomas(a, b, c, f)
    return np.tile(g, N)


def complete_graph(s):
    """K_k: (I+L) = (1+k)I − J  ⇒  z = mean(s)·1 + (s − mean(s)1)/(k+1)."""
    s = np.asarray(s, np.float64)
    k = len(s)
    m = s.mean()
    return m + (s - m) / (k + 1.0)


def weighted_pair(w: float, s0: float = 1.0, s1: float = 0.0):
    """Two nodes joined by an undirected edge of weight w:
    [[1+w, −w], [−w, 1+w]] z = s  ⇒  z = ((1+w)s0 + w s1, w s0 + (1+w)s1)/(1+2w)."""
    den = 1.0 + 2.0 * w
    return np.array([((1 + w) * s0 + w * s1) / den, (w * s0 + (1 + w) * s1) / den])


def directed_arc(s0: float, s1: float, w: float = 1.0):
    """Arc 0→1 (0 listens to 1, weight w): z1 = s1, z0 = (s0 + w s1)/(1 + w)."""
    return np.array([(s0 + w * s1) / (1.0 + w), s1])
