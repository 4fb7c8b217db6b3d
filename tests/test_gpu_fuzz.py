"""Randomised parity sweep (GPU): many small seeded graphs, every schedule.

Each case draws a graph family (ER, R-MAT, Chung–Lu, lattice, random digraph),
weights on/off, an opinion distribution (uniform, signed with zeros, Pareto),
ε, ω and a schedule (ASYNC, COLORED, PUSH, batched, sharded), solves through
the C-ABI and checks the result the way tests/test_gpu_parity.py does: the
oracle's compensated certificate of the GPU ẑ′ (the ε guarantee, Lemma 3) and
z against the oracle's z.  Directed SOR may diverge; such cases must
then report FJ_ERR_NUMERIC, never a wrong answer."""
import numpy as np
import pytest

import fjgen
import oracle
from tests import graphs as G
from tests.test_gpu_parity import rel_err

torch = pytest.importorskip("torch")
fj = pytest.importorskip("paper_2507_14864_b200")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def draw(seed):
    rng = np.random.default_rng(seed)
    fam = ["er", "rmat", "chunglu", "lattice", "digraph"][seed % 5]
    if fam == "er":
        n = int(rng.integers(50, 3000))
        rp, col = fjgen.er_graph(n, float(rng.uniform(2, 12)), seed)
        directed = False
    elif fam == "rmat":
        rp, col = fjgen.rmat_graph(int(rng.integers(6, 12)), int(rng.integers(4, 16)), seed)
        directed = True
    elif fam == "chunglu":
        n = int(rng.integers(200, 4000))
        rp, col = fjgen.chunglu_graph(n, float(rng.uniform(2.05, 2.8)), float(rng.uniform(4, 20)),
                                      seed)
        directed = False
    elif fam == "lattice":
        rp, col = fjgen.lattice_graph(int(rng.integers(8, 48)), float(rng.uniform(0, 0.05)), seed)
        directed = False
    else:
        n = int(rng.integers(30, 400))
        rp, col, _ = G.random_directed(n, float(rng.uniform(0.01, 0.1)), seed)
        directed = True
    n = len(rp) - 1
    w = fjgen.arc_weights(rp, col, seed) if rng.random() < 0.5 else None
    if w is not None and not directed:
        # symmetric weights: the weight of an undirected edge hashes the pair
        u = np.repeat(np.arange(n), np.diff(rp))
        lo, hi = np.minimum(u, col), np.maximum(u, col)
        w = (((lo * 2654435761 + hi * 40503) % 1000) + 1).astype(np.float32) / 1000.0
    kind = rng.integers(0, 3)
    if kind == 0:
        s = fjgen.uniform(n, seed)
    elif kind == 1:
        s = fjgen.zero_mask(fjgen.uniform(n, seed, -1, 1), n // 3, seed)
    else:
        s = fjgen.pareto(n, seed)
    eps = float(10 ** rng.uniform(-7, -4))
    return fam, rp, col, w, s, directed, eps, rng


CASES = list(range(1, 301))


@pytest.mark.parametrize("seed", CASES)
def test_fuzz_case(dev, seed):
    fam, rp, col, w, s, directed, eps, rng = draw(seed)
    n = len(rp) - 1
    sched = ["async", "colored", "push", "batch", "sharded"][(seed // 5) % 5]
    # opt-in paths ride along: the loopback transport (the NCCL path's
    # bookkeeping) for half the sharded cases, the compacted frontier for half
    # the PUSH cases
    loopback = sched == "sharded" and seed % 2 == 1
    push_opts = {}
    if sched == "push" and seed % 2:
        push_opts = dict(push_compact=True, push_sparse_div=int(rng.integers(1, 64)))
    omega = 1.0 if sched in ("batch", "sharded") or rng.random() < 0.4 else \
        float(rng.uniform(1.05, 1.9))
    ref = oracle.solve(rp, col, w, s, eps, 1.0)
    assert ref.status == 0
    s32 = np.asarray(s, np.float32)
    if sched == "batch":
        k = int(rng.integers(1, 5))
        S = np.stack([s32] + [fjgen.uniform(n, seed + 100 + r) for r in range(k - 1)], 1)
        S = np.ascontiguousarray(S.astype(np.float32))
        g = fj.Graph(n, rp, col, w, directed=directed)
        Z = np.empty(n * k, np.float32)
        st = fj.solve_batch(g, S.ravel(), Z, k, eps, omega)
        g.close()
        assert st.status == 0 and st.cert_ratio <= 1.0
        assert rel_err(Z.reshape(n, k)[:, 0].astype(np.float64), ref.z) <= 2 * eps + 1e-6
        return
    if sched == "sharded":
        W = int(rng.integers(1, 5))
        W = min(W, n)
        orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
        begin = np.array(fj.shard_plan(orp, W))
        comm = fj.Comm.in_process(W, loopback=loopback)
        shards = []
        for r in range(W):
            srp, scol, sw = fjgen.shard_rows(orp, ocol, ow, begin, r)
            shards.append(fj.Shard(comm, r, n, begin, srp, scol, sw, directed=directed))
        fj.shard_connect(shards)
        zl = [np.empty(begin[r + 1] - begin[r], np.float32) for r in range(W)]
        zpl = [np.empty(begin[r + 1] - begin[r], np.float64) for r in range(W)]
        sl = [s32[begin[r]:begin[r + 1]].copy() for r in range(W)]
        st = fj.shard_solve(shards, sl, zl, eps, omega, zprime_list=zpl)
        for sh in shards:
            sh.close()
        comm.close()
        zp = np.concatenate(zpl)
        assert st.status == 0
        assert oracle.certificate(rp, col, w, s, zp, eps)[0] <= 1.0
        assert rel_err(np.concatenate(zl).astype(np.float64), ref.z) <= 2 * eps + 1e-6
        return
    g = fj.Graph(n, rp, col, w, directed=directed)
    z = np.empty(n, np.float32)
    zp = np.empty(n, np.float64)
    st = fj.solve(g, s32, z, eps, omega, method=sched, zprime_out=zp, raise_on_numeric=False,
                  **push_opts)
    g.close()
    if st.status == fj.FJ_ERR_NUMERIC:
        # only over-relaxation may fail to converge, and it must say so
        assert omega > 1.0 and st.reason in (1, 2), st
        return
    assert st.status == 0, st
    assert oracle.certificate(rp, col, w, s, zp, eps)[0] <= 1.0
    # both are within ε·max(|z|, σ) of z (plus fp32 rounding of the output)
    assert rel_err(z.astype(np.float64), ref.z) <= 2 * eps + 1e-6
