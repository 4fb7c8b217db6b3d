"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins (P:n = PAPER.md line).  None of these
re-types the oracle's own formula: the expected values come from closed forms,
golden fixtures (tests/golden/, cited), dense Gaussian elimination, or
invariants that any correct implementation must satisfy.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import closed_forms as cf
from tests import graphs as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _csr(ex):
    if ex.get("directed"):
        return G.in_csr_from_arcs(ex["n"], ex.get("arcs", []))
    return G.in_csr_from_edges(ex["n"], ex.get("edges", []))


# ---------------------------------------------------------------- golden
@pytest.mark.parametrize("ex", GOLD["examples"], ids=lambda e: e["name"])
def test_golden_dense(ex):
    """Lemma 1: dense GE reproduces the cited worked examples."""
    rp, col, w = _csr(ex)
    z = oracle.dense_solve(rp, col, w, np.array(ex["s"], np.float32))
    np.testing.assert_allclose(z, ex["z"], rtol=0, atol=1e-7)  # s is fp32-rounded


@pytest.mark.parametrize("ex", GOLD["examples"], ids=lambda e: e["name"])
@pytest.mark.parametrize("omega", [1.0, 1.5])
def test_golden_push(ex, omega):
    """Alg. 2+1 / Alg. 2+3 land in the ε band around the worked example
    (Lemma 5, Lemma 6, reading R5)."""
    rp, col, w = _csr(ex)
    eps = 1e-3
    res = oracle.solve(rp, col, w, np.array(ex["s"], np.float32), eps, omega)
    z = np.array(ex["z"])
    assert res.status == 0
    assert np.all(np.abs(res.z - z) <= eps * np.maximum(np.abs(z), oracle.SIGMA) + 1e-7)


@pytest.mark.parametrize("m", GOLD["measures"], ids=lambda e: e["name"])
def test_golden_measures(m):
    """Table tab:measures on the cited P2 example."""
    rp, col, w = _csr(m)
    out = oracle.measures(rp, col, w, np.array(m["z"]), np.array(m["s"], np.float32),
                          directed=m["directed"])
    for k in "IDPC":
        assert out[k] == pytest.approx(m[k], rel=1e-12)


@pytest.mark.parametrize("o", GOLD["omega_opt"], ids=lambda e: e["name"])
def test_golden_omega_opt(o):
    """Eq. optimal-omega."""
    assert oracle.omega_opt(o["mu"]) == pytest.approx(o["omega"], abs=o["tol"])


def test_jacobi_mu_dense():
    """μ = ρ((I+D)^{-1}A): P2 → 1/2, K3 → 2/3 (eigenvalues by hand)."""
    rp, col, w = G.in_csr_from_edges(2, [(0, 1)])
    assert oracle.jacobi_mu_dense(rp, col, w) == pytest.approx(0.5)
    rp, col, w = G.in_csr_from_edges(3, [(0, 1), (1, 2), (0, 2)])
    assert oracle.jacobi_mu_dense(rp, col, w) == pytest.approx(2 / 3)


# ---------------------------------------------------- closed forms vs dense
def test_dense_complete_graph():
    k = 7
    edges = [(i, j) for i in range(k) for j in range(i + 1, k)]
    rp, col, w = G.in_csr_from_edges(k, edges)
    s = np.linspace(0, 1, k).astype(np.float32)
    np.testing.assert_allclose(oracle.dense_solve(rp, col, w, s), cf.complete_graph(s), atol=1e-14)


@pytest.mark.parametrize("wt", [0.25, 1.0, 3.5])
def test_dense_weighted_pair(wt):
    """Weighted edge (reading R3): d_i = Σ_j a_ij, off-diagonal −a_ij."""
    rp, col, w = G.in_csr_from_edges(2, [(0, 1)], [wt])
    z = oracle.dense_solve(rp, col, w, np.array([1.0, 0.0], np.float32))
    np.testing.assert_allclose(z, cf.weighted_pair(np.float32(wt)), atol=1e-14)


@pytest.mark.parametrize("wt", [1.0, 0.3])
def test_dense_directed_orientation(wt):
    """Reading R1 (listens-to): arc 0→1 ⇒ z1 = s1, z0 = (s0 + w s1)/(1+w).
    A transposed operand would give z0 = s0 instead."""
    rp, col, w = G.in_csr_from_arcs(2, [(0, 1)], [wt])
    z = oracle.dense_solve(rp, col, w, np.array([0.2, 0.9], np.float32))
    np.testing.assert_allclose(z, cf.directed_arc(np.float32(0.2), np.float32(0.9), np.float32(wt)),
                               atol=1e-7)


@pytest.mark.parametrize("k,l", [(1, 0), (2, 3), (5, 5)])
def test_dense_grid_mode(k, l):
    """Grid eigenmode closed form (path-Laplacian Kronecker sum)."""
    N = 9
    rp, col, w = G.in_csr_from_edges(N * N, G.grid_edges(N))
    s, z = cf.grid_mode(N, k, l)
    np.testing.assert_allclose(oracle.dense_solve(rp, col, w, s), z, atol=1e-13)


def test_dense_grid_rows_constant():
    N = 10
    rp, col, w = G.in_csr_from_edges(N * N, G.grid_edges(N))
    f = (np.arange(N) < N // 2).astype(float)
    s = np.tile(f, N)
    np.testing.assert_allclose(oracle.dense_solve(rp, col, w, s), cf.grid_rows_constant(N, f),
                               atol=1e-13)


def test_fj_iterate_converges_to_dense():
    """Eq. (1) converges to (I+L)^{-1}s (Lemma 1)."""
    rp, col, w = G.random_directed(60, 0.08, 3, weighted=True)
    s = np.random.default_rng(0).random(60).astype(np.float32)
    np.testing.assert_allclose(oracle.fj_iterate(rp, col, w, s, 3000),
                               oracle.dense_solve(rp, col, w, s), atol=1e-10)


# -------------------------------------------------------------- Alg. 1/2/3
CASES = [("und", lambda: G.random_undirected(120, 0.06, 1)),
         ("und-w", lambda: G.random_undirected(100, 0.08, 2, weighted=True)),
         ("dir", lambda: G.random_directed(110, 0.05, 4)),
         ("dir-w", lambda: G.random_directed(90, 0.07, 5, weighted=True))]


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("eps", [1e-2, 1e-5])
def test_lemma4_one_sided(name, mk, eps):
    """Lemma 4 / Lemma 5: (1−ε)z ≤ ẑ ≤ z at ω = 1."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = (0.01 + 0.99 * np.random.default_rng(7).random(n)).astype(np.float32)
    z = oracle.dense_solve(rp, col, w, s)
    res = oracle.solve(rp, col, w, s, eps, 1.0)
    assert res.status == 0 and res.cert_ratio <= 1.0
    assert np.all(res.z <= z + 1e-12)
    assert np.all(res.z >= (1 - eps) * z - 1e-12)


@pytest.mark.parametrize("name,mk", CASES[:2], ids=[c[0] for c in CASES[:2]])
@pytest.mark.parametrize("omega", [1.2, 1.5, 1.8])
def test_lemma6_two_sided(name, mk, omega):
    """Lemma 6: (1−ε)z ≤ ẑ ≤ (1+ε)z for SOR on undirected graphs."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = (0.01 + 0.99 * np.random.default_rng(8).random(n)).astype(np.float32)
    z = oracle.dense_solve(rp, col, w, s)
    eps = 1e-4
    res = oracle.solve(rp, col, w, s, eps, omega)
    assert res.status == 0
    assert np.all(np.abs(res.z - z) <= eps * z + 1e-12)


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("omega", [1.0, 1.4])
def test_lemma3_invariant_midrun(name, mk, omega):
    """Lemma 3: z' − ẑ' = (I+L)^{-1} r at any point of the run
    (checked after a bounded number of pushes, for any ω — equ:sor1–3)."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = np.random.default_rng(9).random(n).astype(np.float32)
    M = oracle.dense_system(rp, col, w)
    for k in [1, 7, n // 2, 3 * n]:
        res = oracle.solve(rp, col, w, s, 1e-6, omega, max_pushes=k)
        zprime = np.linalg.solve(M, s.astype(np.float64) + res.c)
        gap = (zprime - res.zprime) - np.linalg.solve(M, res.r)
        assert np.max(np.abs(gap)) <= 1e-10


@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_omega1_reduces_to_alg1(name, mk):
    """Alg. 3 'reduces to standard BoundLocalIter when ω = 1':
    identical pop sequence (same pushes / touched arcs) and identical ẑ."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = np.random.default_rng(10).random(n).astype(np.float32)
    a = oracle.solve(rp, col, w, s, 1e-5, 1.0, alg=1)
    b = oracle.solve(rp, col, w, s, 1e-5, 1.0, alg=3)
    assert (a.pushes, a.touched) == (b.pushes, b.touched)
    assert np.array_equal(a.z, b.z)


def test_zero_opinions_terminate():
    """Alg. 2 robustness: s = 0 terminates with ẑ ∈ [−ε'c, 0]
    (shifted consensus z' = c·1 and Lemma 4's one-sided band)."""
    rp, col, w = G.random_undirected(80, 0.1, 11)
    s = np.zeros(80, np.float32)
    eps = 1e-2
    res = oracle.solve(rp, col, w, s, eps, 1.0)
    assert res.status == 0
    # s_min = 0 ⇒ c = σ (Alg. 2 with reading R5) and ε' = σε/(c+σ) = ε/2
    # (P:337), computed here and not taken from the oracle's own result
    sig = oracle.SIGMA
    c = sig
    eps_p = sig * eps / (c + sig)
    assert res.c == c and res.eps_prime == pytest.approx(eps_p, rel=1e-15)
    assert np.all(res.z <= 1e-18) and np.all(res.z >= -eps_p * c - 1e-18)


def _sources_near_sigma(n=300, seed=21):
    """Opinions spread log-uniformly over [σ, 100σ] plus a third exact zeros:
    most z_v lie in (σ, 100σ), where ε' = σε/(c+σ) and ε' = ε give different
    bands (Lemma 5)."""
    rp, col, w = G.random_undirected(n, 0.02, seed)
    rng = np.random.default_rng(seed)
    s = (oracle.SIGMA * 10 ** rng.uniform(0, 2, n)).astype(np.float32)
    s[rng.choice(n, n // 3, replace=False)] = 0.0
    return rp, col, w, s


@pytest.mark.parametrize("eps", [1e-2, 1e-4])
def test_lemma5_relative_bound_near_sigma(eps):
    """Lemma 5: ImprovedBLI with c = σ and ε' = σε/(c+σ)
    gives (1−ε)z ≤ ẑ ≤ z for every z_v ≥ σ, against dense GE.  The shifted
    system's residual at termination is ≤ h = ε'·s' (Alg. 1 stops when no
    r_u > h_u; h per Alg. 2, P:340 with reading R4), checked with
    the dense matrix and ε' computed here — a slip to ε' = ε leaves residuals
    up to 2h (the realized max is ≈ 0.99h) and fails this test."""
    rp, col, w, s = _sources_near_sigma()
    sig = oracle.SIGMA
    z = oracle.dense_solve(rp, col, w, s)
    res = oracle.solve(rp, col, w, s, eps, 1.0)
    assert res.status == 0
    big = z >= sig
    assert big.sum() > 150
    assert np.all(res.z[big] <= z[big] + 1e-18)
    assert np.all(z[big] - res.z[big] <= eps * z[big])
    c = sig                                       # s ≥ 0: c = σ
    sp = s.astype(np.float64) + c                 # s' = s + c
    h = sig * eps / (c + sig) * sp                # ε' s'
    R = sp - oracle.dense_system(rp, col, w) @ res.zprime
    assert R.max() <= h.max() and np.all(R <= h * (1 + 1e-9) + 1e-18)
    assert np.all(R >= -1e-16)    # Lemma 4: r stays ≥ 0 at ω = 1 (dense matvec rounding ≈ 1e-18)


@pytest.mark.parametrize("omega", [1.0, 1.5])
def test_signed_opinions_floor(omega):
    """Reading R5: signed s (configs 3/5) with the floored thresholds gives
    |ẑ − z| ≤ ε·max(|z|, σ)."""
    rp, col, w = G.random_undirected(150, 0.05, 12)
    rng = np.random.default_rng(12)
    s = rng.uniform(-1, 1, 150).astype(np.float32)
    s[rng.choice(150, 75, replace=False)] = 0.0
    z = oracle.dense_solve(rp, col, w, s)
    eps = 1e-4
    res = oracle.solve(rp, col, w, s, eps, omega)
    assert res.status == 0 and res.c > 0.9
    assert np.all(np.abs(res.z - z) <= eps * np.maximum(np.abs(z), oracle.SIGMA))


def test_certificate_detects_error():
    """The certificate (Lemma 3 residual) passes the terminated state,
    is ~0 on the dense solution, and fails a perturbed estimate."""
    rp, col, w = G.random_directed(100, 0.06, 13, weighted=True)
    s = np.random.default_rng(13).random(100).astype(np.float32)
    eps = 1e-4
    res = oracle.solve(rp, col, w, s, eps, 1.0)
    ratio, _ = oracle.certificate(rp, col, w, s, res.zprime, eps)
    assert ratio <= 1.0
    zd = oracle.dense_solve(rp, col, w, s) + res.c
    assert oracle.certificate(rp, col, w, s, zd, eps)[0] < 1e-6
    bad = res.zprime.copy()
    bad[17] += 10 * eps
    assert oracle.certificate(rp, col, w, s, bad, eps)[0] > 1.0


# --------------------------------------------------------------- invariants
@pytest.mark.parametrize("name,mk", CASES, ids=[c[0] for c in CASES])
def test_bounds_and_conservation(name, mk):
    """(I+L)^{-1} nonnegative row-stochastic: min s ≤ z ≤ max s; for
    undirected graphs 1ᵀ(I+L) = 1ᵀ so 1ᵀz = 1ᵀs; nodes that listen to no one
    (d = 0) keep z = s."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = np.random.default_rng(14).random(n).astype(np.float32)
    res = oracle.solve(rp, col, w, s, 1e-8, 1.0)
    assert np.all(res.z >= s.min() - 1e-12) and np.all(res.z <= s.max() + 1e-12)
    d = oracle.degrees(rp, col, w)
    iso = d == 0
    np.testing.assert_allclose(res.z[iso], s[iso], atol=1e-12)
    if not name.startswith("dir"):
        assert res.z.sum() == pytest.approx(float(s.astype(np.float64).sum()), rel=1e-6)


def test_sor_fewer_updates():
    """BLISOR needs fewer updates than BLI at ω ≈ 1.5 on undirected graphs
    (P:488 'acceleration of more than approximately three times'; SPEC #6
    desk bar ≥ 1.5×)."""
    rp, col, w = G.random_undirected(400, 0.025, 15)
    s = np.random.default_rng(15).random(400).astype(np.float32)
    a = oracle.solve(rp, col, w, s, 1e-6, 1.0)
    b = oracle.solve(rp, col, w, s, 1e-6, 1.5)
    assert a.pushes > 1.5 * b.pushes


# ----------------------------------------------------------------- measures
def test_measures_identities():
    """D = zᵀLz on undirected graphs (north_star); P translation invariant and
    P ≤ C; consensus gives I = D = P = 0, C = n c²."""
    rp, col, w = G.random_undirected(70, 0.1, 16, weighted=True)
    rng = np.random.default_rng(16)
    z = rng.random(70)
    M = oracle.dense_system(rp, col, w)
    L = M - np.eye(70)
    m = oracle.measures(rp, col, w, z, None, directed=False)
    assert m["D"] == pytest.approx(z @ L @ z, rel=1e-12)
    m2 = oracle.measures(rp, col, w, z + 3.0, None, directed=False)
    assert m2["P"] == pytest.approx(m["P"], rel=1e-10)
    assert m["P"] <= m["C"]
    c = oracle.measures(rp, col, w, np.full(70, 0.3), np.full(70, 0.3, np.float32))
    assert c["D"] == 0 and c["P"] == pytest.approx(0, abs=1e-28) and c["I"] == pytest.approx(0, abs=1e-14)
    assert c["C"] == pytest.approx(70 * 0.09, rel=1e-12)


def test_measures_directed_arc_once():
    """Reading R14: a directed arc counts once; an undirected edge once."""
    rp, col, w = G.in_csr_from_arcs(3, [(0, 1), (2, 1)], [2.0, 1.0])
    z = np.array([1.0, 0.0, 3.0])
    assert oracle.measures(rp, col, w, z, directed=True)["D"] == pytest.approx(2 * 1 + 1 * 9)
    rp, col, w = G.in_csr_from_edges(2, [(0, 1)])
    assert oracle.measures(rp, col, w, np.array([1.0, 0.0]), directed=False)["D"] == 1.0


# ------------------------------------------------------ ω heuristic
def _mu_numpy(rp, col, w):
    """μ = ρ((I+D)^{-1}A) with numpy's eigenvalue routine on A built
    here from the arcs (independent of oracle.dense_system)."""
    n = len(rp) - 1
    A = np.zeros((n, n))
    for v in range(n):
        for e in range(rp[v], rp[v + 1]):
            A[col[e], v] = 1.0 if w is None else float(w[e])
    J = A / (1.0 + A.sum(axis=1))[:, None]
    return float(np.max(np.abs(np.linalg.eigvals(J))))


OMEGA_CASES = [  # (name, graph, speed-up over ω = 1 the SOR theory leaves room for)
    ("grid24", lambda: G.in_csr_from_edges(576, G.grid_edges(24)), 1.5),
    ("path200", lambda: G.in_csr_from_edges(200, [(i, i + 1) for i in range(199)]), 1.3),
    ("er400", lambda: G.random_undirected(400, 0.025, 15), 3.0),
]


@pytest.mark.parametrize("name,mk,gain", OMEGA_CASES, ids=[c[0] for c in OMEGA_CASES])
def test_omega_sweep_near_omega_opt(name, mk, gain):
    """The fewest-updates heuristic lands next to the SOR optimum
    ω_opt = 1 + (μ/(1+√(1−μ²)))² (Eq. optimal-omega; Young's theorem
    for consistently ordered SPD systems) with μ from numpy's eigenvalues —
    grid 1.25, path 1.15, ER 1.41 — and beats ω = 1 (by ≥ 3× on the random
    graph, P:488's "more than approximately three times"; the path's small μ
    leaves SOR less room)."""
    rp, col, w = mk()
    n = len(rp) - 1
    s = np.random.default_rng(1).random(n).astype(np.float32)
    best, table = oracle.omega_sweep(rp, col, w, s, 1e-6, prune=False)
    mu = _mu_numpy(rp, col, w)
    w_opt = 1.0 + (mu / (1.0 + np.sqrt(1.0 - mu * mu))) ** 2
    assert abs(best - w_opt) <= 0.1, (best, w_opt)
    cost = {om: c for om, c, _ in table}
    assert [om for om, _, _ in table] == oracle.omega_grid()          # 1.95 → 1.00
    assert cost[1.0] >= gain * cost[best]
    assert cost[best] == min(cost.values())
    # pruning only drops runs that cannot win: same pick, same winning count
    best2, table2 = oracle.omega_sweep(rp, col, w, s, 1e-6, prune=True)
    assert best2 == best and dict((o, c) for o, c, _ in table2)[best] == cost[best]


def test_omega_sweep_skips_divergence():
    """Directed graphs: SOR over-relaxation may diverge (P:484 covers only
    the symmetric case; reading R11); the heuristic gives such ω cost +∞
    and picks a converging ω, which still meets the ε band against dense GE."""
    rp, col, w = G.random_directed(200, 0.03, 4)
    s = np.random.default_rng(1).random(200).astype(np.float32)
    best, table = oracle.omega_sweep(rp, col, w, s, 1e-6, prune=False)
    diverged = [om for om, c, st in table if st == "diverged"]
    assert 1.95 in diverged and best not in diverged
    res = oracle.solve(rp, col, w, s, 1e-6, best)
    z = oracle.dense_solve(rp, col, w, s)
    assert res.status == 0
    assert np.all(np.abs(res.z - z) <= 1e-6 * np.maximum(np.abs(z), oracle.SIGMA))
    mu = _mu_numpy(rp, col, w)
    assert abs(best - (1.0 + (mu / (1.0 + np.sqrt(1.0 - mu * mu))) ** 2)) <= 0.1


def test_omega_sweep_ties_to_smaller():
    """Ties go to the smaller ω (reading R10): with an empty graph every
    node is its own component, z = s, and one push at ω = 1 is exact while any
    other ω needs more — so the pick is 1.0 on a grid whose every other point
    costs more, and a single-point grid returns that point."""
    rp = np.zeros(6, np.int64)
    col = np.zeros(0, np.int32)
    s = np.array([0.1, 0.2, 0.3, 0.4, 0.5], np.float32)
    best, table = oracle.omega_sweep(rp, col, None, s, 1e-6, prune=False)
    cost = {om: c for om, c, _ in table}
    assert best == 1.0 and cost[1.0] == 5
    assert all(c > 5 for om, c in cost.items() if om != 1.0)
    # a symmetric pair: |1 − ω| equal for ω = 0.9 and 1.1 ⇒ equal pop counts
    best, table = oracle.omega_sweep(rp, col, None, s, 1e-6, lo=0.9, hi=1.1, step=0.2,
                                     prune=False)
    assert [om for om, _, _ in table] == [1.1, 0.9]
    assert table[0][1] == table[1][1] and best == 0.9
