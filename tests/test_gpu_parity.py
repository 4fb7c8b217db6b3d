"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star):
  * z: max_v |ẑ_v − z_or,v| / max(|z_or,v|, σ) ≤ 1e-4 against the oracle's
    converged z at the same ε;
  * ε guarantee, independently: the oracle's compensated fp64 certificate of
    the GPU's ẑ' gives max |R_v|/h_v ≤ 1 ⇒ |ẑ − z| ≤ ε·max(|z|, σ);
  * P and D: relative error ≤ 1e-5.
"""
import numpy as np
import pytest

import fjgen
import oracle
from oracle import closed_forms as cf
from tests import graphs as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
fj = pytest.importorskip("paper_2507_14864_b200")

SIG = oracle.SIGMA


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _t(a, dev):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def gpu_solve(dev, rp, col, w, s, eps, omega=1.0, directed=True, method="auto", host=False,
              raise_on_numeric=True, **opts):
    n = len(rp) - 1
    if host:
        g = fj.Graph(n, rp, col, w, directed=directed)
        z = np.empty(n, np.float32)
        zp = np.empty(n, np.float64)
        st = fj.solve(g, np.ascontiguousarray(s, np.float32), z, eps, omega, method=method,
                      zprime_out=zp, raise_on_numeric=raise_on_numeric, **opts)
        return g, z.astype(np.float64), zp, st
    g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    zp = torch.empty(n, dtype=torch.float64, device=dev)
    st = fj.solve(g, _t(np.asarray(s, np.float32), dev), z, eps, omega, method=method,
                  zprime_out=zp, raise_on_numeric=raise_on_numeric, **opts)
    torch.cuda.synchronize()
    return g, z.cpu().numpy().astype(np.float64), zp.cpu().numpy(), st


def rel_err(z, ref):
    return np.max(np.abs(z - ref) / np.maximum(np.abs(ref), SIG)) if len(z) else 0.0


def check_parity(dev, rp, col, w, s, eps, omega, directed, method="auto", ref_omega=None, **opts):
    g, z, zp, st = gpu_solve(dev, rp, col, w, s, eps, omega, directed, method, **opts)
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    # independent certificate by the oracle's own routine
    ratio, _ = oracle.certificate(rp, col, w, s, zp, eps)
    assert ratio <= 1.0, ratio
    # oracle z at the same ε (reading R11: ω = 1 reference for directed SOR)
    ro = omega if ref_omega is None else ref_omega
    ref = oracle.solve(rp, col, w, s, eps, ro)
    assert ref.status == 0
    assert rel_err(z, ref.z) <= 1e-4
    # measures: GPU reduction on GPU z vs oracle measures of oracle z
    m = fj.measures(g, torch.from_numpy(z.astype(np.float32)).to(dev))
    om = oracle.measures(rp, col, w, ref.z, directed=directed)
    for k in ("P", "D"):
        assert abs(m[k] - om[k]) <= 1e-5 * abs(om[k]) + 1e-300, (k, m[k], om[k])
    # reduction alone: same fp32 input on both sides
    om2 = oracle.measures(rp, col, w, z.astype(np.float32).astype(np.float64), directed=directed)
    for k in ("P", "D"):
        assert abs(m[k] - om2[k]) <= 1e-9 * abs(om2[k]) + 1e-300
    g.close()
    return st, z, ref


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("host", [False, True])
def test_golden_examples(dev, host):
    import json, os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
    for ex in gold["examples"]:
        if ex.get("directed"):
            rp, col, w = G.in_csr_from_arcs(ex["n"], ex["arcs"])
        else:
            rp, col, w = G.in_csr_from_edges(ex["n"], ex["edges"])
        s = np.array(ex["s"], np.float32)
        for omega in (1.0, 1.5):
            g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, omega, ex.get("directed", False),
                                     host=host)
            zt = np.array(ex["z"])
            assert np.all(np.abs(z - zt) <= 1e-6 * np.maximum(np.abs(zt), SIG) + 1e-7), ex["name"]
            g.close()
    m = gold["measures"][0]
    rp, col, w = G.in_csr_from_edges(2, [(0, 1)])
    g = fj.Graph(2, rp, col, None, directed=False)
    out = fj.measures(g, np.array(m["z"], np.float32), np.array(m["s"], np.float32))
    for k in "IDPC":
        assert out[k] == pytest.approx(m[k], rel=1e-6)
    P, D = fj.measures_pd(g, np.array(m["z"], np.float32))
    assert P == pytest.approx(m["P"], rel=1e-6) and D == pytest.approx(m["D"], rel=1e-6)
    g.close()


# -------------------------------------------------------------- tiny suite
TINY = {
    "er2000": lambda: (*fjgen.er_graph(2000, 10.0, 11), None, fjgen.uniform(2000, 11), False),
    "rmat12": lambda: (*fjgen.rmat_graph(12, 16, 12), None, fjgen.uniform(4096, 12), True),
    "rmat12w": lambda: (lambda rp, col: (rp, col, fjgen.arc_weights(rp, col, 13),
                                         fjgen.beta25(4096, 13), True))(*fjgen.rmat_graph(12, 16, 13)),
    "chunglu4k": lambda: (lambda rp, col: (rp, col, None,
                                           fjgen.zero_mask(fjgen.uniform(4096, 14, -1, 1), 2048, 14),
                                           False))(*fjgen.chunglu_graph(4096, 2.1, 20, 14)),
    "lattice64": lambda: (*fjgen.lattice_graph(64, 0.01, 15), None, fjgen.step_noise(64, 15), False),
    "dirw-dense": lambda: (*G.random_directed(300, 0.05, 16, weighted=True),
                           fjgen.uniform(300, 16), True),
}


@pytest.mark.parametrize("name", sorted(TINY))
def test_tiny_async(dev, name):
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed)


@pytest.mark.parametrize("name", ["er2000", "chunglu4k", "lattice64"])
@pytest.mark.parametrize("omega", [1.25, 1.5, 1.8])
def test_tiny_colored_sor_undirected(dev, name, omega):
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, omega, directed)


@pytest.mark.parametrize("name", ["rmat12", "rmat12w", "dirw-dense"])
@pytest.mark.parametrize("omega", [1.2, 1.4])
def test_tiny_colored_sor_directed(dev, name, omega):
    """Reading R11: directed SOR is compared with the oracle at ω = 1."""
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, omega, directed, ref_omega=1.0)


@pytest.mark.parametrize("omega", [1.0, 1.3])
def test_async_vs_colored_methods(dev, omega):
    rp, col, w, s, directed = TINY["er2000"]()
    if omega == 1.0:
        check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="colored")
    else:
        # ASYNC with ω > 1 is not guaranteed; if it converges it is certified
        g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, omega, directed, method="async",
                                 raise_on_numeric=False)
        if st.status == 0:
            assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
        g.close()


# ------------------------------------------------------------- edge cases
def test_single_isolated_node(dev):
    rp = np.array([0, 0], np.int64)
    col = np.zeros(0, np.int32)
    g, z, zp, st = gpu_solve(dev, rp, col, None, np.array([0.4], np.float32), 1e-6)
    assert z[0] == pytest.approx(0.4, abs=1e-7) and st.sweeps == 1
    g.close()


def test_no_arcs_ragged(dev):
    n = 1237
    rp = np.zeros(n + 1, np.int64)
    s = fjgen.uniform(n, 3)
    g, z, _, st = gpu_solve(dev, rp, np.zeros(0, np.int32), None, s, 1e-6, 1.5)
    np.testing.assert_allclose(z, s, atol=1e-7)
    g.close()


def test_constant_and_zero_opinions(dev):
    rp, col, w, _, _ = TINY["lattice64"]()
    n = len(rp) - 1
    g, z, _, st = gpu_solve(dev, rp, col, w, np.full(n, 0.4, np.float32), 1e-6, 1.0, False)
    assert np.all(np.abs(z - 0.4) <= 1e-6 * 0.4 + 1e-7)
    g.close()
    g, z, _, st = gpu_solve(dev, rp, col, w, np.zeros(n, np.float32), 1e-6, 1.0, False)
    assert np.all(np.abs(z) <= 1e-6 * SIG + 1e-12)
    g.close()


@pytest.mark.parametrize("hub_deg", [300, 2048, 2049, 20000])
def test_long_rows_star(dev, hub_deg):
    """Hub rows above 256 arcs are split in 2048-arc pieces reduced across
    CTAs (deterministic partials); the star has a closed form for the hub."""
    n = hub_deg + 1
    edges = [(0, i) for i in range(1, n)]
    rp, col, w = G.in_csr_from_edges(n, edges)
    s = fjgen.uniform(n, 5)
    check_parity(dev, rp, col, w, s, 1e-6, 1.0, False)
    check_parity(dev, rp, col, w, s, 1e-6, 1.5, False)


def test_determinism_colored(dev):
    """COLORED sweeps read only other colors' values: bit-reproducible (with the
    tail merge of reading R23 off: the merged tail phase is asynchronous)."""
    rp, col, w, s, directed = TINY["rmat12w"]()
    a = gpu_solve(dev, rp, col, w, s, 1e-6, 1.2, directed, method="colored", tail_frac=0.0)
    b = gpu_solve(dev, rp, col, w, s, 1e-6, 1.2, directed, method="colored", tail_frac=0.0)
    assert np.array_equal(a[2], b[2])
    a[0].close(); b[0].close()


# ------------------------------------------- tail-color merge (reading R23)
@pytest.mark.parametrize("name", ["chunglu4k", "er2000", "rmat12w"])
@pytest.mark.parametrize("omega", [1.3, 1.7])
def test_tail_merge_parity(dev, name, omega):
    """Merged tail phase: certified, same z as the oracle, fewer phases."""
    rp, col, w, s, directed = TINY[name]()
    if directed and omega > 1.5:
        pytest.skip("SOR with ω > 1 on a non-symmetric M-matrix may diverge (as in exact SOR)")
    ref_omega = 1.0 if directed else None
    st0, z0, ref = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, method="colored",
                                ref_omega=ref_omega, tail_frac=0.0)
    st1, z1, _ = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, method="colored",
                              ref_omega=ref_omega, tail_frac=0.2)
    assert st1.colors <= st0.colors
    if st0.colors > 3:
        assert st1.colors < st0.colors


@pytest.mark.parametrize("omega", [1.5, 1.9])
def test_tail_merge_complete_graph(dev, omega):
    """K_200: every color holds one row, so merging 90% of the rows makes a
    tail whose rows are all adjacent (β_i ≈ 0.9).  The per-row bound
    ω_i = min(ω, 1.98/(1+β_i)) keeps the asynchronous tail a contraction; the
    result is the closed form of oracle.closed_forms.complete_graph."""
    k = 200
    edges = [(i, j) for i in range(k) for j in range(i + 1, k)]
    rp, col, w = G.in_csr_from_edges(k, edges)
    s = fjgen.uniform(k, 77)
    g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, omega, False, method="colored",
                             tail_frac=0.9)
    assert st.status == 0 and st.colors < k
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    assert rel_err(z, cf.complete_graph(s.astype(np.float64))) <= 1e-4
    g.close()


@pytest.mark.parametrize("coloring", ["spec", "jp"])
@pytest.mark.parametrize("name", ["chunglu4k", "rmat12w"])
def test_colorings(dev, coloring, name):
    """Both colorings (default speculative largest-first, fj_opts.coloring = 1
    Jones–Plassmann) give valid colored solves; the colors are a proper coloring
    (checked through the sequential-SOR parity of the COLORED schedule without
    the tail merge).  Switching the option on one graph rebuilds the coloring."""
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, 1.3, directed, method="colored",
                 ref_omega=1.0 if directed else None, coloring=coloring, tail_frac=0.0)


@pytest.mark.parametrize("compact", ["0", "1"])
@pytest.mark.parametrize("omega", [1.0, 1.197, 1.6])
def test_push_certifies_rows_without_arcs(dev, compact, omega):
    """Rows with d_v = 0 are exact after the pull solvers' init (R20) but PUSH
    relaxes them like any other row, so the certificate (and the residual it
    hands back on a resume) must cover them: the GPU ratio is at least the
    oracle's ratio over those rows, and the result meets the ε bound.  (A
    directed R-MAT graph with isolated nodes and sinks.)"""
    rp, col = fjgen.rmat_graph(11, 8, 161)
    n = len(rp) - 1
    s = fjgen.uniform(n, 161)
    eps = 6e-7
    d = oracle.degrees(rp, col, None)
    E = np.nonzero(d == 0)[0]
    assert len(E) > 0
    ref = oracle.solve(rp, col, None, s, eps, 1.0)
    g = fj.Graph(n, rp, col, None, directed=True)
    for rep in range(3):
        z = np.empty(n, np.float32)
        zp = np.empty(n, np.float64)
        st = fj.solve(g, s, z, eps, omega, method="push", zprime_out=zp,
                      push_compact=compact == "1", push_sparse_div=15)
        ratio, R = oracle.certificate(rp, col, None, s, zp, eps)
        _, h, _, _ = oracle.thresholds(s, eps)
        assert ratio <= 1.0 and st.cert_ratio <= 1.0
        assert st.cert_ratio >= (np.abs(R[E]) / h[E]).max() * (1 - 1e-6)
        assert rel_err(z.astype(np.float64), ref.z) <= 2 * eps + 1e-6
    g.close()


def mixed_hub_graph(weighted, seed=17):
    """Directed graph whose in-rows mix hubs around the 2048-arc chunk size
    (2047, 2048, 2049, 4096, 5000, 7000 arcs), empty rows and short rows, so
    32-row chunks of the build's chunked walks hold several pieces, rows that
    cross piece boundaries and empty rows between them."""
    rng = np.random.default_rng(seed)
    n = 9000
    lens = rng.integers(0, 6, n)
    lens[rng.random(n) < 0.2] = 0
    hubs = {3: 2047, 4: 2048, 5: 2049, 6: 0, 7: 5000, 9: 7000, 10: 1, 11: 0, 40: 4096,
            41: 300, 8000: 6000}
    for v, L in hubs.items():
        lens[v] = L
    rows = []
    for v in range(n):
        c = rng.choice(n - 1, lens[v], replace=False)
        c[c >= v] += 1                       # no self-loops
        # popular columns: long rows on the transposed (pull) side as well
        for hub, p in ((100, 0.5), (101, 0.25), (102, 0.23)):
            if v != hub and rng.random() < p:
                c = np.append(c, hub)
        rows.append(np.unique(c))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    col = np.concatenate(rows).astype(np.int32)
    w = fjgen.arc_weights(rp, col, seed) if weighted else None
    return rp, col, w


@pytest.mark.parametrize("weighted", [False, True])
def test_chunked_build_mixed_hubs(dev, weighted):
    """Graph build from device tensors (packed transpose) and from host arrays
    (index transpose, weights staged on the side stream) give the same layout:
    COLORED results agree bit for bit; both pass the oracle's parity bar."""
    rp, col, w = mixed_hub_graph(weighted)
    s = fjgen.uniform(len(rp) - 1, 23)
    check_parity(dev, rp, col, w, s, 1e-6, 1.0, True, method="async")
    outs = []
    for host in (False, True):
        g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, 1.0, True, method="colored", host=host)
        assert st.status == 0
        outs.append(zp)
        g.close()
    assert np.array_equal(outs[0], outs[1])
    assert oracle.certificate(rp, col, w, s, outs[0], 1e-6)[0] <= 1.0


@pytest.mark.parametrize("weighted", [False, True])
def test_many_hub_pieces(dev, weighted):
    """A hub row of 150,000 arcs (74 warp pieces of 2048 arcs, combined by the
    last-arriving warp in piece order) next to a random directed graph: the
    piece-combine path of the sweep and of the certificate, against the oracle."""
    n = 150_001
    rng = np.random.default_rng(31)
    arcs = [(0, v) for v in range(1, n)]                       # node 0 listens to everyone
    extra = rng.integers(1, n, size=(60_000, 2))
    arcs += [(int(u), int(v)) for u, v in extra if u != v]
    arcs = sorted(set(arcs))
    wts = list(rng.uniform(0.1, 1.0, len(arcs))) if weighted else None
    rp, col, w = G.in_csr_from_arcs(n, arcs, wts)
    check_parity(dev, rp, col, w, fjgen.uniform(n, 31), 1e-6, 1.0, True, method="async")


@pytest.mark.parametrize("name", ["er2000", "rmat12w", "lattice64"])
@pytest.mark.parametrize("eps", [1e-2, 1e-4])
def test_accuracy_protocol(dev, name, eps):
    """The paper's accuracy protocol (tab:measure_li): against the exact
    z of a dense solve, the maximum relative opinion error stays within ε
    (with σ, reading R5) and every measure's relative error within 2ε."""
    rp, col, w, s, directed = TINY[name]()
    zref = oracle.dense_solve(rp, col, w, s)
    mref = oracle.measures(rp, col, w, zref, directed=directed, s=np.asarray(s, np.float64))
    for omega in (1.0, 1.3 if not directed else 1.2):
        g, z, zp, st = gpu_solve(dev, rp, col, w, s, eps, omega, directed)
        m = fj.measures(g, torch.from_numpy(z.astype(np.float32)).to(dev),
                        torch.from_numpy(np.asarray(s, np.float32)).to(dev))
        g.close()
        assert np.max(np.abs(z - zref) / np.maximum(np.abs(zref), SIG)) <= eps
        for k in "CDIP":
            assert abs(m[k] - mref[k]) <= 2 * eps * abs(mref[k]) + 1e-12, (k, m[k], mref[k])


def test_gather_probe(dev):
    """fj_gather_probe runs on the layout and reports a positive time."""
    rp, col, w, s, directed = TINY["rmat12w"]()
    g = fj.Graph(len(rp) - 1, rp, col, w, directed=directed)
    ms = fj.gather_probe(g, 3)
    assert 0.0 < ms < 100.0
    with pytest.raises(fj.FJError):
        fj.gather_probe(g, 0)
    g.close()


def test_invalid_inputs(dev):
    def create(n, arcs, w=None, directed=True, rp=None, col=None):
        if rp is None:
            rp, col, _ = G.in_csr_from_arcs(n, arcs)
        return fj.Graph(n, rp, col, w, directed=directed)
    with pytest.raises(fj.FJError, match="self-loop"):
        create(3, [(0, 0), (1, 2)])
    rp = np.array([0, 2, 2], np.int64)
    with pytest.raises(fj.FJError, match="duplicate"):
        create(2, None, rp=rp, col=np.array([1, 1], np.int32))
    with pytest.raises(fj.FJError, match="range"):
        create(2, None, rp=rp, col=np.array([1, 5], np.int32))
    with pytest.raises(fj.FJError, match="row_ptr"):
        create(2, None, rp=np.array([0, 3, 2], np.int64), col=np.array([1, 0], np.int32))
    with pytest.raises(fj.FJError, match="symmetric"):
        create(3, [(0, 1), (1, 2), (2, 1)], directed=False)
    rp, col, _ = G.in_csr_from_arcs(2, [(0, 1)])
    with pytest.raises(fj.FJError, match="weight"):
        fj.Graph(2, rp, col, np.array([-1.0], np.float32))
    g = fj.Graph(2, rp, col, None)
    z = np.empty(2, np.float32)
    for eps, om in [(0.0, 1.0), (1.0, 1.0), (1e-3, 0.0), (1e-3, 2.0)]:
        with pytest.raises(fj.FJError) as e:
            fj.solve(g, np.ones(2, np.float32), z, eps, om)
        assert e.value.status == fj.FJ_ERR_INVALID
    with pytest.raises(fj.FJError) as e:
        fj.solve(g, np.array([np.nan, 1], np.float32), z, 1e-3, 1.0)
    assert e.value.status == fj.FJ_ERR_INVALID
    g.close()


def test_divergence_reported(dev):
    """A directed graph where ω = 1.9 over-relaxation diverges must come back
    as FJ_ERR_NUMERIC (sentinel), not as a wrong answer."""
    rp, col, w, s, _ = TINY["rmat12w"]()
    g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, 1.95, True, raise_on_numeric=False)
    if st.status == 0:
        assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    else:
        assert st.status == fj.FJ_ERR_NUMERIC and st.reason in (1, 2)
    g.close()


def test_simple_abi_calls(dev):
    rp, col, w, s, directed = TINY["er2000"]()
    g = fj.Graph(2000, _t(rp, dev), _t(col, dev), None, directed=False)
    z = torch.empty(2000, dtype=torch.float32, device=dev)
    fj.solve_simple(g, _t(s, dev), z, 1e-6, 1.0)
    ref = oracle.solve(rp, col, w, s, 1e-6, 1.0)
    assert rel_err(z.cpu().numpy().astype(np.float64), ref.z) <= 1e-4
    P, D = fj.measures_pd(g, z)
    om = oracle.measures(rp, col, w, ref.z, directed=False)
    assert P == pytest.approx(om["P"], rel=1e-5) and D == pytest.approx(om["D"], rel=1e-5)
    g.close()


# ------------------------------------------------- full-size closed forms
def test_full_lattice_eigenmode(dev):
    """Config 5's 4096² grid (no shortcuts) with a cosine eigenmode opinion
    vector: the exact z is known at full size (oracle/closed_forms.py)."""
    N = 4096
    rp, col = fjgen.lattice_graph(N, 0.0, 0)
    s, zt = cf.grid_mode(N, 3, 5)
    s32 = s.astype(np.float32)
    # closed form of the fp32-rounded input: z(s32) = z(s) + (I+L)^{-1}(s32 − s),
    # and |(I+L)^{-1}(s32 − s)| ≤ max|s32 − s| (row-stochastic)
    slack = np.max(np.abs(s32 - s))
    eps = 1e-6
    g, z, zp, st = gpu_solve(dev, rp, col, None, s32, eps, 1.0, False)
    assert np.all(np.abs(z - zt) <= eps * np.abs(zt) + slack + 6e-8 * np.abs(zt))
    g.close()


def test_full_lattice_step_1d(dev):
    """Noise-free step on the 4096² grid reduces to the 1-D tridiagonal
    system (I + L_path) g = f (oracle/closed_forms.py)."""
    N = 4096
    rp, col = fjgen.lattice_graph(N, 0.0, 0)
    f = (np.arange(N) < N // 2).astype(np.float64)
    zt = cf.grid_rows_constant(N, f)
    eps = 1e-6
    for omega in (1.0, 1.25):
        g, z, zp, st = gpu_solve(dev, rp, col, None, np.tile(f, N).astype(np.float32), eps,
                                 omega, False)
        assert np.all(np.abs(z - zt) <= eps * np.maximum(np.abs(zt), SIG) + 6e-8 * np.abs(zt))
        g.close()


# --------------------------------------------------- frontier push (row a3)
@pytest.mark.parametrize("name", sorted(TINY))
def test_tiny_push(dev, name):
    """FJ_METHOD_PUSH (Alg. 1 data-parallel: pop phase + atomic scatter)."""
    rp, col, w, s, directed = TINY[name]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="push")
    assert st.relaxations > 0 and st.edge_updates > 0


@pytest.mark.parametrize("name", ["rmat12w", "chunglu4k", "lattice64"])
@pytest.mark.parametrize("div", ["1", "64"])
def test_tiny_push_compacted_frontier(dev, name, div):
    """PUSH with frontier compaction (ballot + per-warp atomic slots) and the
    sparse warp-per-row scatter of the compacted list."""
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="push", push_compact=True,
                 push_sparse_div=int(div))


@pytest.mark.parametrize("name", ["er2000", "lattice64", "chunglu4k"])
def test_tiny_push_sor_colored(dev, name):
    """FJ_METHOD_PUSH with ω ≠ 1: Alg. 3 per color (pushes of one color commute)."""
    rp, col, w, s, directed = TINY[name]()
    check_parity(dev, rp, col, w, s, 1e-6, 1.5, directed, method="push")


@pytest.mark.parametrize("hub_deg", [3000, 20000])
def test_push_long_scatter_lists(dev, hub_deg):
    n = hub_deg + 1
    rp, col, w = G.in_csr_from_edges(n, [(0, i) for i in range(1, n)])
    check_parity(dev, rp, col, w, fjgen.uniform(n, 9), 1e-6, 1.0, False, method="push")


# ------------------------------------------------------- ω selection (f1)
def test_omega_opt_small_closed_forms(dev):
    """Eq. optimal-omega with μ by power iteration: P2 → μ = 1/2,
    ω = 1.0718; K3 → μ = 2/3, ω = 1.1459."""
    for edges, n, mu_t, om_t in [([(0, 1)], 2, 0.5, 1.0718), ([(0, 1), (1, 2), (0, 2)], 3, 2 / 3, 1.1459)]:
        rp, col, w = G.in_csr_from_edges(n, edges)
        g = fj.Graph(n, rp, col, None, directed=False)
        mu, om = fj.omega_opt(g)
        assert mu == pytest.approx(mu_t, abs=1e-6) and om == pytest.approx(om_t, abs=1e-4)
        g.close()


SMALL = {
    "er2000": lambda: TINY["er2000"]()[:3] + (False,),
    "lattice32": lambda: (*fjgen.lattice_graph(32, 0.01, 15), None, False),
    "rmat10w": lambda: (lambda rp, col: (rp, col, fjgen.arc_weights(rp, col, 13), True))(
        *fjgen.rmat_graph(10, 16, 13)),
    "dirw-dense": lambda: TINY["dirw-dense"]()[:3] + (True,),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_omega_opt_vs_dense(dev, name):
    rp, col, w, directed = SMALL[name]()
    g = fj.Graph(len(rp) - 1, rp, col, w, directed=directed)
    mu, om = fj.omega_opt(g, max_iters=20000, tol=1e-12)
    mu_d = oracle.jacobi_mu_dense(rp, col, w)
    assert mu == pytest.approx(mu_d, rel=1e-4)
    assert om == pytest.approx(oracle.omega_opt(mu_d), rel=1e-4)
    g.close()


@pytest.mark.parametrize("name", ["er2000", "lattice64", "rmat12"])
def test_omega_sweep_vs_oracle_heuristic(dev, name):
    """f1: the GPU's fewest-updates pick (fj_omega_sweep: relaxations
    of its own schedule) against the ORACLE's pick (FIFO pops of Alg. 3, the
    paper's "number of updates") over the same grid 1.95:−0.05:1.00 (R10).
    Undirected graphs run COLORED sweeps — a true SOR ordering, like FIFO
    ImprovedBLISOR's — and the GPU pick must lie in the oracle's near-optimal
    band (FIFO pops within 1.25× of the oracle's minimum).  On the directed
    graph the GPU runs chaotic (ASYNC) over-relaxation, a different iteration:
    the two heuristics may pick different ω (measured: GPU 1.6, oracle 1.5 on
    rmat12); there each pick must converge under the other implementation.
    Both tables are in the assertion message."""
    rp, col, w, s, directed = TINY[name]()
    n = len(rp) - 1
    best_o, table = oracle.omega_sweep(rp, col, w, s, 1e-6, prune=False)
    cost = {round(om, 2): c for om, c, _ in table}
    cmin = min(cost.values())
    band = sorted(om for om, c in cost.items() if c <= 1.25 * cmin)
    g = fj.Graph(n, rp, col, w, directed=directed)
    best_g, rows = fj.omega_sweep(g, s, 1e-6, lo=1.0, hi=1.95, step=0.05)
    g.close()
    msg = f"gpu {best_g} {[(round(r[0], 2), r[1], r[2]) for r in rows]} | oracle {best_o} {table}"
    assert best_o in band
    if not directed:
        assert round(best_g, 2) in band, msg
    else:
        assert cost[round(best_g, 2)] != float("inf"), msg       # the GPU pick converges on the oracle
        gstat = {round(r[0], 2): r[2] for r in rows}
        assert gstat[round(best_o, 2)] == 0, msg                  # and the oracle pick on the GPU


def test_omega_sweep_heuristic(dev):
    """P:488 heuristic: the returned ω has the fewest relaxations among the
    converged grid points (ties to the smaller ω); undirected ER favours ω > 1."""
    rp, col, w, s, directed = TINY["er2000"]()
    g = fj.Graph(2000, rp, col, None, directed=False)
    best, rows = fj.omega_sweep(g, s, 1e-6, lo=1.0, hi=1.9, step=0.1)
    assert len(rows) == 10
    ok = [r for r in rows if r[2] == 0]
    mincost = min(r[1] for r in ok)
    assert best == pytest.approx(min(r[0] for r in ok if r[1] == mincost))
    assert best > 1.0
    g.close()


# ----------------------------------------------------- batched RHS (f2)
def _batch_columns(n, s0, k):
    """The paper's opinion distributions (Unif / Exp / Pareto) plus
    signed and shifted ones, k columns."""
    cols = [s0, fjgen.exponential(n, 21), fjgen.pareto(n, 22), fjgen.uniform(n, 23, -1.0, 1.0),
            fjgen.uniform(n, 24), fjgen.uniform(n, 25, -0.5, 0.5), fjgen.exponential(n, 26),
            fjgen.pareto(n, 27)][:k]
    return np.ascontiguousarray(np.stack(cols, axis=1).astype(np.float32))


@pytest.mark.parametrize("name", ["er2000", "rmat12w", "chunglu4k", "lattice64"])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("omega", [1.0, 1.5])
def test_batch_solve(dev, name, k, omega):
    """fj_solve_batch (row f2): k opinion vectors solved together, padded to
    K = 2 / 4 / 8; ω = 1.5 runs multicolor SOR (with the merged tail, R23) on
    the undirected graphs and asynchronous over-relaxation on the directed one
    (which may be reported as FJ_ERR_NUMERIC, reading R11).  Every column
    matches the oracle at the same ε (the oracle at ω for undirected graphs, at
    ω = 1 for the directed one, R11)."""
    rp, col, w, s0, directed = TINY[name]()
    n = len(rp) - 1
    S = _batch_columns(n, s0, k)
    g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
    Z = torch.empty(n * k, dtype=torch.float32, device=dev)
    st = fj.solve_batch(g, _t(S.ravel(), dev), Z, k, 1e-6, omega, raise_on_numeric=False)
    torch.cuda.synchronize()
    g.close()
    if st.status == fj.FJ_ERR_NUMERIC:
        assert directed and omega > 1.0 and st.reason in (1, 2), st
        return
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    if omega != 1.0 and not directed:
        assert st.colors > 1  # AUTO picked the multicolor schedule
    Zh = Z.cpu().numpy().reshape(n, k).astype(np.float64)
    for r in range(k):
        ref = oracle.solve(rp, col, w, S[:, r], 1e-6, 1.0 if directed else omega)
        assert rel_err(Zh[:, r], ref.z) <= 1e-4, r


# ------------------------------------------------ Lemma 4 on the GPU path
@pytest.mark.parametrize("name", ["er2000", "rmat10w", "dirw-dense"])
def test_gpu_lemma4_one_sided(dev, name):
    """Lemma 4 / Lemma 5: at ω = 1 with s ≥ 0 every relaxation
    adds a nonnegative amount, so (1−ε)z ≤ ẑ ≤ z elementwise (up to the fp32
    output rounding) — for any order of relaxations, hence for the GPU's."""
    rp, col, w, directed = SMALL[name]()
    n = len(rp) - 1
    s = (0.05 + 0.95 * fjgen.uniform(n, 31).astype(np.float64)).astype(np.float32)
    z = oracle.dense_solve(rp, col, w, s)
    for eps in (1e-2, 1e-4):
        g, zg, zp, st = gpu_solve(dev, rp, col, w, s, eps, 1.0, directed)
        tol = 2.0 ** -23 * np.abs(z)
        assert np.all(zg <= z + tol)
        assert np.all(zg >= (1 - eps) * z - tol)
        g.close()


# ------------------------------------------------ the C-ABI from plain C
@pytest.mark.parametrize("prog", ["fj_example", "fj_shard_example"])
def test_c_program_against_abi(dev, tmp_path, prog):
    """examples/*.c link libfj.so directly (no Python marshalling): the P2
    worked example (tab:measures) and a two-shard path against the
    tridiagonal closed form."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2507_14864_b200")
    exe = str(tmp_path / prog)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(root, "include"),
                           os.path.join(root, "examples", prog + ".c"), "-L", libdir, "-l:libfj.so",
                           f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout


# --------------------------------------- full BASELINE sizes (configs 2–5)
@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_full_size_config_properties(dev, cid):
    """At the full BASELINE.json size, in the launch configuration bench.py
    times (AUTO schedule, ω = 1, ε = 1e-6), with properties that hold at any
    size: (i) the oracle's compensated certificate of the GPU's ẑ' is ≤ 1, so
    |ẑ − z| ≤ ε·max(|z|, σ) (Lemma 6 + R5); (ii) the GPU measures equal the
    oracle's measures of the same z; (iii) min s ≤ z ≤ max s and nodes that
    listen to no one keep z = s (fundamental matrix row-stochastic).
    The oracle's own full-size FIFO solves are in profiles/r01_full_parity.md."""
    p = fjgen.config(cid)
    g = fj.Graph(p.n, _t(p.row_ptr, dev), _t(p.col, dev), _t(p.w, dev), directed=p.directed)
    z = torch.empty(p.n, dtype=torch.float32, device=dev)
    zp = torch.empty(p.n, dtype=torch.float64, device=dev)
    st = fj.solve(g, _t(p.s, dev), z, 1e-6, 1.0, zprime_out=zp)
    m = fj.measures(g, z)
    zh = z.cpu().numpy().astype(np.float64)
    ratio, _ = oracle.certificate(p.row_ptr, p.col, p.w, p.s, zp.cpu().numpy(), 1e-6)
    assert st.status == 0 and st.cert_ratio <= 1.0 and ratio <= 1.0
    om = oracle.measures(p.row_ptr, p.col, p.w, zh, directed=p.directed)
    assert abs(m["P"] - om["P"]) <= 1e-9 * om["P"] and abs(m["D"] - om["D"]) <= 1e-9 * om["D"]
    s64 = p.s.astype(np.float64)
    assert zh.min() >= s64.min() - 1e-6 and zh.max() <= s64.max() + 1e-6
    outdeg = np.bincount(p.col, minlength=p.n)
    iso = outdeg == 0
    if iso.any():
        np.testing.assert_allclose(zh[iso], s64[iso], rtol=0,
                                   atol=2e-7 * np.abs(s64[iso]).max() + 1e-12)
    g.close()


# --------------------------------------------- warm start (resume, §5)
@pytest.mark.parametrize("name", ["er2000", "rmat12w", "lattice64"])
def test_warm_start_resume(dev, name):
    """Resume from an earlier estimate (Lemma 3: any ẑ is a valid state): a
    solve warm-started from a converged z needs ≤ 2 sweeps and still passes
    the oracle's certificate; one warm-started from a loose (ε = 1e-2) z
    needs less work (edge updates) than a cold start."""
    rp, col, w, s, directed = TINY[name]()
    n = len(rp) - 1
    g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    zp = torch.empty(n, dtype=torch.float64, device=dev)
    cold = fj.solve(g, _t(s, dev), z, 1e-6, 1.0)
    fj.solve(g, _t(s, dev), z, 1e-2, 1.0)
    warm = fj.solve(g, _t(s, dev), z, 1e-6, 1.0, z_init=z.double(), zprime_out=zp)
    # less work, not necessarily fewer sweeps: the sweep count is set by the
    # slowest component, which a loose start barely advances (rmat12w: 227 vs
    # 226 sweeps once in ~40 runs, with 5.7 M vs 9.0 M edge updates)
    assert warm.edge_updates < 0.8 * cold.edge_updates
    assert oracle.certificate(rp, col, w, s, zp.cpu().numpy(), 1e-6)[0] <= 1.0
    again = fj.solve(g, _t(s, dev), z, 1e-6, 1.0, z_init=(zp - warm.c).contiguous())
    assert again.sweeps <= 2
    with pytest.raises(fj.FJError):
        fj.solve(g, _t(s, dev), z, 1e-6, 1.0, method="push", z_init=(zp - warm.c).contiguous())
    g.close()


def test_unsorted_rows_canonicalised(dev):
    """fj_graph_create accepts rows in any order (the library sorts them,
    carrying the weights along): same z as the sorted input, bit for bit in
    COLORED mode (deterministic)."""
    rp, col, w, s, directed = TINY["rmat12w"]()
    rng = np.random.default_rng(5)
    col2 = col.copy()
    w2 = w.copy()
    for v in range(len(rp) - 1):
        a, b = rp[v], rp[v + 1]
        perm = rng.permutation(b - a)
        col2[a:b] = col[a:b][perm]
        w2[a:b] = w[a:b][perm]
    outs = []
    for c_, w_ in ((col, w), (col2, w2)):
        g, z, zp, st = gpu_solve(dev, rp, c_, w_, s, 1e-6, 1.2, directed, method="colored")
        outs.append(zp)
        g.close()
    assert np.array_equal(outs[0], outs[1])


# ------------------------- full BASELINE sizes against the oracle (round 2)
_CFG = {}


def _config(cid):
    """Full-size config `cid` (fjgen), generated once per test process."""
    if cid not in _CFG:
        _CFG.clear() if len(_CFG) >= 2 else None   # keep host memory bounded
        _CFG[cid] = fjgen.config(cid)
    return _CFG[cid]


def _full_solve(dev, p, omega, raise_on_numeric=True):
    g = fj.Graph(p.n, _t(p.row_ptr, dev), _t(p.col, dev), _t(p.w, dev), directed=p.directed)
    z = torch.empty(p.n, dtype=torch.float32, device=dev)
    zp = torch.empty(p.n, dtype=torch.float64, device=dev)
    st = fj.solve(g, _t(p.s, dev), z, p_eps(p), omega, zprime_out=zp,
                  raise_on_numeric=raise_on_numeric)
    m = fj.measures(g, z)
    torch.cuda.synchronize()
    out = z.cpu().numpy().astype(np.float64), zp.cpu().numpy(), st, m
    g.close()
    return out


def p_eps(p):
    return 1e-6   # every config (BASELINE.json configs; fjgen.CONFIG_SOLVE)


# (config, ω): the oracle's FIFO solve at the same ω and ε finishes in seconds
# to ~30 s on one host core (profiles/r01f_full_parity.md)
FULL_VS_ORACLE = [(1, 1.0), (1, 1.5), (2, 1.0), (5, 1.0), (5, 1.25), (5, 1.3)]


@pytest.mark.parametrize("cid,omega", FULL_VS_ORACLE, ids=[f"C{c}-w{o}" for c, o in FULL_VS_ORACLE])
def test_full_size_vs_oracle_z(dev, cid, omega):
    """The north_star parity bar at the full BASELINE size, in the launch
    configuration bench.py times (AUTO schedule; ε = 1e-6): the GPU z against
    the oracle's converged z (ImprovedBLI / ImprovedBLISOR, FIFO, fp64; Alg. 2
    + Alg. 1/3) element by element, max rel ≤ 1e-4;
    the oracle's own certificate of the GPU ẑ' ≤ 1 (Lemma 6); P and D
    (tab:measures P:105–106) within 1e-5 of the oracle's measures of its z."""
    p = _config(cid)
    z, zp, st, m = _full_solve(dev, p, omega)
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    ratio, _ = oracle.certificate(p.row_ptr, p.col, p.w, p.s, zp, 1e-6)
    assert ratio <= 1.0, ratio
    ref = oracle.solve(p.row_ptr, p.col, p.w, p.s, 1e-6, omega)
    assert ref.status == 0
    assert rel_err(z, ref.z) <= 1e-4
    om = oracle.measures(p.row_ptr, p.col, p.w, ref.z, directed=p.directed)
    for k in ("P", "D"):
        assert abs(m[k] - om[k]) <= 1e-5 * abs(om[k]), (k, m[k], om[k])


# (config, ω) whose oracle FIFO solve takes minutes (C3 ω = 1.6: 64 s, C4: 221–1000 s;
# C3's 1.6 is also its tuned ω, fjgen.CONFIG_SOLVE):
# certified by the oracle's compensated certificate (any size), measures of the same z
FULL_CERTIFIED = [(3, 1.6), (4, 1.2), (4, 1.4), (4, 1.6)]


@pytest.mark.parametrize("cid,omega", FULL_CERTIFIED, ids=[f"C{c}-w{o}" for c, o in FULL_CERTIFIED])
def test_full_size_sor_certified(dev, cid, omega):
    """BLISOR at full size (Alg. 3): C3 at ω = 1.6 runs the
    COLORED schedule with the merged tail (reading R23), C4 the ASYNC directed
    schedule (R11).  The oracle's compensated certificate of the GPU ẑ' is ≤ 1
    (⇒ |ẑ − z| ≤ ε·max(|z|, σ), Lemma 6 P:474 + R5); the GPU measures equal the
    oracle's measures of the same z (≤ 1e-9); min s ≤ z ≤ max s."""
    p = _config(cid)
    z, zp, st, m = _full_solve(dev, p, omega)
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    if cid == 3:
        assert st.colors > 1   # AUTO picked the multicolor schedule
    ratio, _ = oracle.certificate(p.row_ptr, p.col, p.w, p.s, zp, 1e-6)
    assert ratio <= 1.0, ratio
    om = oracle.measures(p.row_ptr, p.col, p.w, z, directed=p.directed)
    for k in ("P", "D"):
        assert abs(m[k] - om[k]) <= 1e-9 * abs(om[k]), (k, m[k], om[k])
    s64 = p.s.astype(np.float64)
    assert z.min() >= s64.min() - 1e-6 and z.max() <= s64.max() + 1e-6


def test_full_size_c4_omega18_numeric(dev):
    """C4 at ω = 1.8 (BASELINE.json's ω list): asynchronous over-relaxation of
    the directed R-MAT-24 system diverges; the library reports FJ_ERR_NUMERIC
    (divergence sentinel S:339 / watchdog) instead of a wrong answer (R11)."""
    p = _config(4)
    z, zp, st, m = _full_solve(dev, p, 1.8, raise_on_numeric=False)
    assert st.status == fj.FJ_ERR_NUMERIC and st.reason in (1, 2), st


def test_full_size_c2_tuned_omega(dev):
    """C2 at its tuned ω = 1.55 (the oracle's fewest-updates pick, reading R10):
    the directed graph runs the ASYNC schedule, where over-relaxation carries
    no guarantee (P:484 covers the symmetric case; R11) — the solve is either
    certified by the oracle's own certificate or reported as FJ_ERR_NUMERIC."""
    p = _config(2)
    z, zp, st, m = _full_solve(dev, p, fjgen.CONFIG_SOLVE[2]["tuned"], raise_on_numeric=False)
    if st.status == 0:
        assert st.cert_ratio <= 1.0
        assert oracle.certificate(p.row_ptr, p.col, p.w, p.s, zp, 1e-6)[0] <= 1.0
    else:
        assert st.status == fj.FJ_ERR_NUMERIC and st.reason in (1, 2), st


# ------------------------------------------------ ω batch (rows f1 / f2)
@pytest.mark.parametrize("name", ["er2000", "lattice64", "chunglu4k", "rmat12w"])
def test_batch_omega_columns(dev, name):
    """fj_solve_batch_omega: one opinion vector at several ω in one solve.
    Every converged column matches the oracle at the same ε (at its ω on
    undirected graphs, at ω = 1 on the directed one, R11); on the directed
    graph a diverging column (ω = 1.95) is reported per column (FJ_ERR_NUMERIC)
    and frozen while the other columns converge; relaxation counts fall from
    ω = 1 to the paper's ω ≈ 1.5 on undirected graphs."""
    rp, col, w, s, directed = TINY[name]()
    n = len(rp) - 1
    omegas = [1.0, 1.2, 1.5, 1.95] if directed else [1.0, 1.25, 1.5, 1.7, 1.9]
    g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
    Z = torch.empty(n * len(omegas), dtype=torch.float32, device=dev)
    st, rel, stat = fj.solve_batch_omega(g, _t(np.asarray(s, np.float32), dev), Z, omegas, 1e-6)
    torch.cuda.synchronize()
    g.close()
    Zh = Z.cpu().numpy().reshape(n, len(omegas)).astype(np.float64)
    for r, om in enumerate(omegas):
        if stat[r] != 0:
            assert directed and om > 1.5, (om, stat)
            continue
        ref = oracle.solve(rp, col, w, s, 1e-6, 1.0 if directed else om)
        assert rel_err(Zh[:, r], ref.z) <= 1e-4, om
    assert stat[0] == 0 and stat[1] == 0
    if not directed:
        assert all(x == 0 for x in stat)
        assert rel[2] < rel[0]   # over-relaxation needs fewer updates


# ------------------------------------------------- shadow sweeps (fj_opts.shadow)
# The sweeps gather from the 32-bit fixed-point shadow of ẑ' until nothing relaxes (or only
# the shadow's rounding noise does), then fp64 sweeps finish: same bar as every solve — the
# oracle's z, the oracle's certificate of the GPU's ẑ', P and D.
@pytest.mark.parametrize("name", sorted(TINY))
def test_shadow_async(dev, name):
    rp, col, w, s, directed = TINY[name]()
    st, z, ref = check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async", shadow=1)
    assert 0 < st.shadow_sweeps <= st.sweeps  # (the frontier phase may finish without an fp64 sweep)
    # the shadow changes the path, not the answer: fp64-only solve of the same input
    _, z0, _, st0 = gpu_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async", shadow=0)
    assert st0.shadow_sweeps == 0
    assert rel_err(z, z0) <= 4e-6


@pytest.mark.parametrize("name", ["er2000", "chunglu4k", "lattice64"])
@pytest.mark.parametrize("omega", [1.25, 1.6])
def test_shadow_colored_sor(dev, name, omega):
    # floored thresholds (chunglu4k, lattice64: h ≈ 1e-11) lie far below the shadow's
    # resolution: the shadow loop must hand over to fp64 (at ω ≠ 1 its rounding noise need
    # not die out) instead of running into the watchdog
    rp, col, w, s, directed = TINY[name]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, shadow=1, max_sweeps=20000)
    assert 0 < st.shadow_sweeps <= st.sweeps


@pytest.mark.parametrize("name", ["rmat12", "rmat12w"])
def test_shadow_async_sor_directed(dev, name):
    rp, col, w, s, directed = TINY[name]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.3, directed, method="async", ref_omega=1.0,
                            shadow=1)
    assert st.shadow_sweeps > 0


@pytest.mark.parametrize("hub_deg", [300, 2049, 20000])
def test_shadow_long_rows_star(dev, hub_deg):
    # hub pieces (partials + arrival counters) under the shadow kernel, then under the fp64 tail
    n = hub_deg + 1
    edges = [(0, i) for i in range(1, n)]
    rp, col, w = G.in_csr_from_edges(n, edges)
    s = fjgen.uniform(n, 31)
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, False, method="async", shadow=1)
    assert st.shadow_sweeps > 0


def test_shadow_warm_start_and_range(dev):
    # a warm start far above max s' leaves the shadow's range [0, 2·2^e): the shadow loop
    # ends at once and the fp64 sweeps solve from that ẑ (any ẑ is a valid state, Lemma 3)
    rp, col, w, s, directed = TINY["er2000"]()
    ref = oracle.solve(rp, col, w, s, 1e-6, 1.0)
    for z0 in (np.full(len(s), 50.0), ref.z.copy()):
        g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async", shadow=1,
                                 z_init=_t(z0, dev))
        assert st.status == 0 and st.cert_ratio <= 1.0
        assert rel_err(z, ref.z) <= 1e-4
        ratio, _ = oracle.certificate(rp, col, w, s, zp, 1e-6)
        assert ratio <= 1.0
        g.close()


def test_shadow_divergence_reported(dev):
    # a diverging ω under the shadow kernel still ends in FJ_ERR_NUMERIC (range exit or
    # sentinel, then the fp64 sweeps' own sentinel)
    rp, col, w, s, directed = TINY["rmat12"]()
    g, z, zp, st = gpu_solve(dev, rp, col, w, s, 1e-6, 1.95, directed, method="async",
                             raise_on_numeric=False, shadow=1, max_sweeps=5000)
    if st.status == 0:
        assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    else:
        assert st.status == fj.FJ_ERR_NUMERIC and st.reason in (1, 2)
    g.close()


# ------------------------------------------------- row slices / warp tiles (fj_opts.slices)
# Short rows run as row slices (sliced ELL, one lane per row) or as warp tiles (CSR arcs,
# shared-memory staging); the default picks per layout.  Both walks are held to the bar of
# every solve on every tiny graph, with and without shadow gathers, and on a graph whose
# slices mix lengths, padding and hub pieces.
@pytest.mark.parametrize("slices", [0, 1])
@pytest.mark.parametrize("name", sorted(TINY))
def test_row_walks_async(dev, name, slices):
    rp, col, w, s, directed = TINY[name]()
    for shadow in (0, 1):
        st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async",
                                slices=slices, shadow=shadow)
        assert (st.shadow_sweeps > 0) == (shadow == 1)


@pytest.mark.parametrize("slices", [0, 1])
@pytest.mark.parametrize("name,omega", [("er2000", 1.5), ("chunglu4k", 1.6), ("lattice64", 1.25)])
def test_row_walks_colored_sor(dev, name, omega, slices):
    rp, col, w, s, directed = TINY[name]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, method="colored",
                            slices=slices)
    assert st.colors > 1


@pytest.mark.parametrize("weighted", [False, True])
def test_row_slices_mixed_lengths(dev, weighted):
    """Every row length from 1 to 300 a few times (slices that straddle a length or class
    boundary are padded), a ragged last slice per class, rows without arcs, and two hub
    rows cut into pieces: slices and tiles agree with the oracle and with each other."""
    rng = np.random.default_rng(77)
    n = 6000
    lens = np.concatenate([np.repeat(np.arange(1, 301), 3), [5000, 2500], np.zeros(40, np.int64)])
    lens = np.concatenate([lens, rng.integers(1, 9, n - len(lens))])
    rng.shuffle(lens)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.empty(rp[-1], np.int32)
    for i in range(n):
        c = rng.choice(n - 1, int(lens[i]), replace=False)
        c[c >= i] += 1  # no self-loops
        col[rp[i]:rp[i + 1]] = np.sort(c)
    w = rng.uniform(0.05, 1.0, rp[-1]).astype(np.float32) if weighted else None
    s = fjgen.uniform(n, 78)
    zs = []
    for slices in (0, 1):
        _, z, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, True, method="async", slices=slices)
        zs.append(z)
    assert rel_err(zs[0], zs[1]) <= 2e-6


# ------------------------------------------------- frontier phase (fj_opts.frontier)
# After a thin sweep the solve switches to the push form on the rows above threshold
# (k_front).  A huge threshold makes every sweep "thin", so the push rounds do nearly the
# whole solve: the strictest test of their residual bookkeeping against the oracle.
@pytest.mark.parametrize("frontier", [10**9, 64])
@pytest.mark.parametrize("name", sorted(TINY))
def test_frontier_phase_async(dev, name, frontier):
    rp, col, w, s, directed = TINY[name]()
    st, z, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async",
                            frontier=frontier)
    assert st.frontier_rounds > 0 and st.frontier_pushes > 0
    # same answer as the sweeps alone (both meet the ε rule: they differ by ≤ 2ε relative)
    g, z0, _, st0 = gpu_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async", frontier=0)
    g.close()
    assert st0.frontier_rounds == 0 and st0.frontier_ms == 0.0
    assert rel_err(z, z0) <= 2.5e-6
    if frontier == 10**9:
        assert st.sweeps < st0.sweeps


@pytest.mark.parametrize("name,omega", [("rmat12", 1.3), ("rmat12w", 1.2), ("dirw-dense", 1.4),
                                        ("rmat12w", 0.7)])
def test_frontier_phase_sor_directed(dev, name, omega):
    """ω ≠ 1: a popped row keeps (1−ω) r_v and is listed again while that is above h."""
    rp, col, w, s, directed = TINY[name]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, method="async",
                            ref_omega=1.0, frontier=10**9)
    assert st.frontier_rounds > 0


@pytest.mark.parametrize("shadow", [0, 1])
@pytest.mark.parametrize("hub_deg", [3000, 70000])
def test_frontier_phase_hub_rows(dev, hub_deg, shadow):
    """A hub that gathers and is gathered by tens of thousands of rows: its scatter is cut
    into chunks, its residual is the compensated one of the hub-piece path."""
    n = hub_deg + 50
    # undirected star (node 0 ↔ 1..hub_deg) plus a ring over the other nodes
    src = np.concatenate([np.zeros(hub_deg, np.int64), np.arange(1, hub_deg + 1),
                          np.arange(1, n), np.r_[np.arange(2, n), 1]])
    dst = np.concatenate([np.arange(1, hub_deg + 1), np.zeros(hub_deg, np.int64),
                          np.r_[np.arange(2, n), 1], np.arange(1, n)])
    key = np.unique(src * n + dst)
    src, dst = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, src + 1, 1)
    rp = np.cumsum(rp)
    col = dst.astype(np.int32)
    s = fjgen.uniform(n, 91)
    st, _, _ = check_parity(dev, rp, col, None, s, 1e-6, 1.0, False, method="async",
                            frontier=n // 16, shadow=shadow)
    assert st.frontier_rounds > 0
    # every sweep "thin": after sweep 1 nearly all rows are above threshold and the phase's
    # lists (a quarter of the rows) overflow on the larger star — it must hand back to the
    # sweeps (reason 3) with ẑ' intact, and the solve must still meet the bar
    st, _, _ = check_parity(dev, rp, col, None, s, 1e-6, 1.0, False, method="async",
                            frontier=10**9, shadow=shadow)
    assert st.status == 0


def test_frontier_phase_zero_heavy_floored(dev):
    """Signed, zero-heavy opinions (floored thresholds h ≈ 1e-11, the fp64 floor of hub
    rows): the phase must leave rows it cannot move to the certificate, not spin."""
    rp, col, w, s, directed = TINY["chunglu4k"]()
    st, _, _ = check_parity(dev, rp, col, w, s, 1e-6, 1.0, directed, method="async",
                            frontier=10**9, max_sweeps=20000)
    assert st.frontier_rounds > 0 and st.status == 0


@pytest.mark.parametrize("frontier", [10**9, 64])
@pytest.mark.parametrize("name,omega", [("er2000", 1.5), ("chunglu4k", 1.6), ("lattice64", 1.25),
                                        ("lattice64", 1.8)])
def test_frontier_phase_after_colored_sor(dev, name, omega, frontier):
    """COLORED BLISOR sweeps, then the frontier phase with plain (ω = 1) pops: the oracle at
    the same ω is the reference (both meet the ε rule), certificate and measures as always."""
    rp, col, w, s, directed = TINY[name]()
    st, z, _ = check_parity(dev, rp, col, w, s, 1e-6, omega, directed, method="colored",
                            frontier=frontier, max_sweeps=20000)
    assert st.colors > 1
    # (with a small threshold fast SOR may go from many relaxations to none in one sweep)
    assert st.frontier_rounds > 0 or frontier == 64
    g, z0, _, st0 = gpu_solve(dev, rp, col, w, s, 1e-6, omega, directed, method="colored",
                              frontier=0, max_sweeps=20000)
    g.close()
    assert st0.frontier_rounds == 0
    assert rel_err(z, z0) <= 2.5e-6


@pytest.mark.parametrize("name,omega", [("rmat12w", 1.0), ("er2000", 1.0), ("er2000", 1.5),
                                        ("chunglu4k", 1.0)])
@pytest.mark.parametrize("k", [3, 8])
def test_batch_solve_frontier_phase(dev, name, omega, k):
    """Batched solve with the frontier phase forced early (every sweep "thin"): each column
    finishes on its own in the push form and is written back; the padding columns follow the
    last real one; the second launch of the batched sweeps confirms.  Columns vs the oracle."""
    rp, col, w, s0, directed = TINY[name]()
    n = len(rp) - 1
    S = _batch_columns(n, s0, k)
    g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
    Z = torch.empty(n * k, dtype=torch.float32, device=dev)
    st = fj.solve_batch(g, _t(S.ravel(), dev), Z, k, 1e-6, omega, frontier=10**9)
    st0 = fj.solve_batch(g, _t(S.ravel(), dev), torch.empty_like(Z), k, 1e-6, omega, frontier=0)
    torch.cuda.synchronize()
    g.close()
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    assert st.frontier_rounds > 0 and st0.frontier_rounds == 0
    assert st.sweeps < st0.sweeps
    Zh = Z.cpu().numpy().reshape(n, k).astype(np.float64)
    for r in range(k):
        ref = oracle.solve(rp, col, w, S[:, r], 1e-6, omega)
        assert rel_err(Zh[:, r], ref.z) <= 1e-4, r
