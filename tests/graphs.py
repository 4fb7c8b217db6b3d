"""Small-graph helpers for the tests: edge lists → the C-ABI in-CSR.

Pure data plumbing (no FJ arithmetic); shared by oracle and GPU tests.
"""
from __future__ import annotations

import numpy as np


def in_csr_from_arcs(n, arcs, weights=None):
    """arcs: iterable of (u, v) meaning u→v (u listens to v).  Row v of the
    in-CSR lists u (ascending) with weight a_uv."""
    arcs = [(int(u), int(v)) for u, v in arcs]
    w = None if weights is None else [float(x) for x in weights]
    order = sorted(range(len(arcs)), key=lambda i: (arcs[i][1], arcs[i][0]))
    rp = np.zeros(n + 1, np.int64)
    col = np.zeros(len(arcs), np.int32)
    ww = None if w is None else np.zeros(len(arcs), np.float32)
    for k, i in enumerate(order):
        u, v = arcs[i]
        rp[v + 1] += 1
        col[k] = u
        if ww is not None:
            ww[k] = w[i]
    rp = np.cumsum(rp).astype(np.int64)
    return rp, col, ww


def in_csr_from_edges(n, edges, weights=None):
    """Undirected edges (i, j): both arcs, equal weights."""
    arcs, ws = [], []
    for k, (i, j) in enumerate(edges):
        arcs += [(i, j), (j, i)]
        if weights is not None:
            ws += [weights[k], weights[k]]
    return in_csr_from_arcs(n, arcs, ws if weights is not None else None)


def random_undirected(n, p, seed, weighted=False):
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < p
    edges = list(zip(iu[0][keep], iu[1][keep]))
    w = list(rng.uniform(0.1, 1.0, len(edges))) if weighted else None
    return in_csr_from_edges(n, edges, w)


def random_directed(n, p, seed, weighted=False):
    rng = np.random.default_rng(seed)
    A = rng.random((n, n)) < p
    np.fill_diagonal(A, False)
    arcs = list(zip(*np.nonzero(A)))
    w = list(rng.uniform(0.1, 1.0, len(arcs))) if weighted else None
    return in_csr_from_arcs(n, arcs, w)


def grid_edges(N):
    e = []
    for y in range(N):
        for x in range(N):
            i = y * N + x
            if x + 1 < N:
                e.append((i, i + 1))
            if y + 1 < N:
                e.append((i, i + N))
    return e


def out_degree_unweighted(rp, col):
    n = len(rp) - 1
    return np.bincount(col, minlength=n)
