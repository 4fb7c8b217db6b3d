"""Generator checks (the input recipe of DESIGN.md; no FJ arithmetic here)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import fjgen


def _canonical(rp, col, n):
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0)
    assert col.min(initial=0) >= 0 and col.max(initial=0) < n
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert not np.any(rows == col), "self-loop"
    # strictly ascending within each row ⇒ no duplicates
    same = rows[1:] == rows[:-1]
    assert np.all(col[1:][same] > col[:-1][same])
    return rows


def _symmetric(rp, col, n):
    rows = np.repeat(np.arange(n), np.diff(rp))
    a = set(zip(rows.tolist(), col.tolist()))
    assert all((c, r) in a for r, c in a)


def test_er_stats_and_determinism():
    rp, col = fjgen.er_graph(4000, 10.0, 101)
    rp2, col2 = fjgen.er_graph(4000, 10.0, 101)
    assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
    _canonical(rp, col, 4000)
    _symmetric(rp, col, 4000)
    mean_deg = rp[-1] / 4000
    assert abs(mean_deg - 10.0) < 0.3  # 3σ of the edge count ≈ 0.13
    rp3, _ = fjgen.er_graph(4000, 10.0, 102)
    assert not np.array_equal(rp, rp3)


def test_rmat_orientation_and_skew():
    rp, col = fjgen.rmat_graph(12, 16, 202)
    n = 1 << 12
    _canonical(rp, col, n)
    m = rp[-1]
    assert 0.6 * 16 * n < m <= 16 * n
    indeg = np.diff(rp)
    outdeg = np.bincount(col, minlength=n)
    # a + c = 0.76 of draws keep the dst bit 0 at each level: low ids are hubs
    assert indeg[: n // 2].sum() > 2.5 * indeg[n // 2:].sum()
    assert outdeg.sum() == m and (outdeg == 0).mean() > 0.1


def test_chunglu_degrees():
    n = 1 << 14
    w = fjgen.chunglu_expected_degrees(n, 2.1, 20.0)
    assert w[0] == pytest.approx(np.sqrt(20.0 * n), rel=1e-9)
    assert w.mean() == pytest.approx(20.0, rel=1e-6)
    assert np.all(np.diff(w) <= 0)
    rp, col = fjgen.chunglu_graph(n, 2.1, 20.0, 303)
    _canonical(rp, col, n)
    _symmetric(rp, col, n)
    assert 14.0 < rp[-1] / n < 21.0  # capping at p = 1 trims a little


def test_lattice_counts():
    N = 64
    rp, col = fjgen.lattice_graph(N, 0.01, 505)
    n = N * N
    _canonical(rp, col, n)
    _symmetric(rp, col, n)
    k = int(0.01 * n)
    assert rp[-1] == 4 * N * (N - 1) + 2 * k
    deg = np.diff(rp)
    assert deg.max() <= 4 + 4  # a node can receive several shortcuts, rarely


def test_opinion_distributions():
    n = 200_000
    u = fjgen.uniform(n, 1)
    assert u.dtype == np.float32 and 0 <= u.min() and u.max() < 1
    assert abs(u.mean() - 0.5) < 3 / np.sqrt(12 * n)
    b = fjgen.beta25(n, 4)
    assert abs(b.mean() - 2 / 7) < 0.002  # Beta(2,5) mean
    assert abs(b.var() - 10 / (49 * 8)) < 0.001
    s = fjgen.uniform(1000, 3, -1.0, 1.0)
    fjgen.zero_mask(s, 500, 3)
    assert (s == 0).sum() == 500
    st = fjgen.step_noise(128, 5, 0.1)
    x = np.tile(np.arange(128), 128)
    assert abs(st[x < 64].mean() - 1) < 0.01 and abs(st[x >= 64].mean()) < 0.01
    assert abs(st[x >= 64].std() - 0.1) < 0.005


def test_weights_hash_of_arc():
    rp, col = fjgen.rmat_graph(10, 8, 404)
    w = fjgen.arc_weights(rp, col, 404)
    assert w.min() > 0 and w.max() <= 1
    assert abs(w.mean() - 0.5) < 0.01


def test_thread_count_independent():
    code = ("import fjgen,hashlib;rp,c=fjgen.rmat_graph(11,8,7);"
            "s=fjgen.beta25(5000,7);"
            "print(hashlib.sha1(rp.tobytes()+c.tobytes()+s.tobytes()).hexdigest())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = set()
    for t in ("1", "3"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=root)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=root).strip())
    assert len(outs) == 1


@pytest.mark.parametrize("cid", [1, 2, 3, 4, 5])
def test_configs_small(cid):
    p = fjgen.config(cid, shrink=3 if cid in (2, 3, 4) else 2)
    _canonical(p.row_ptr, p.col, p.n)
    if not p.directed:
        _symmetric(p.row_ptr, p.col, p.n)
    assert p.s.dtype == np.float32 and len(p.s) == p.n
    if cid == 3:
        assert (p.s == 0).sum() == p.n // 2 and p.s.min() < 0
    if cid == 4:
        assert p.w is not None and len(p.w) == p.m
