"""GPU tests of the sharded solve through the C-ABI.

One GPU is available, so the multi-rank path runs with the in-process
transport (all W shards of one process on cuda:0, exchanges as device
copies; nothing waits on another rank), and the NCCL transport is exercised
with a one-rank communicator.  Everything is compared with the oracle
(`oracle/`) exactly as the single-GPU parity tests do."""
import numpy as np
import pytest

import fjgen
import oracle
from tests import graphs as G
from tests.test_gpu_parity import TINY, rel_err, SIG

torch = pytest.importorskip("torch")
fj = pytest.importorskip("paper_2507_14864_b200")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def make_shards(comm, rp, col, w, directed, begin, on_device, dev):
    orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
    n = len(rp) - 1
    shards = []
    for r in range(len(begin) - 1):
        srp, scol, sw = fjgen.shard_rows(orp, ocol, ow, begin, r)
        if on_device:
            srp, scol = torch.from_numpy(srp).to(dev), torch.from_numpy(scol).to(dev)
            sw = None if sw is None else torch.from_numpy(sw).to(dev)
        shards.append(fj.Shard(comm, r, n, begin, srp, scol, sw, directed=directed))
    return shards


def sharded_solve(dev, rp, col, w, s, eps, omega, directed, W, on_device=True, begin=None,
                  loopback=False):
    n = len(rp) - 1
    if begin is None:
        orp, _, _ = fjgen.to_out_csr(rp, col, w)
        begin = np.array(fj.shard_plan(orp, W))
    comm = fj.Comm.in_process(len(begin) - 1, loopback=loopback)
    shards = make_shards(comm, rp, col, w, directed, begin, on_device, dev)
    fj.shard_connect(shards)
    s32 = np.asarray(s, np.float32)
    sl, zl, zpl = [], [], []
    for r in range(len(begin) - 1):
        a, b = int(begin[r]), int(begin[r + 1])
        if on_device:
            sl.append(torch.from_numpy(s32[a:b].copy()).to(dev))
            zl.append(torch.empty(b - a, dtype=torch.float32, device=dev))
            zpl.append(torch.empty(b - a, dtype=torch.float64, device=dev))
        else:
            sl.append(s32[a:b].copy())
            zl.append(np.empty(b - a, np.float32))
            zpl.append(np.empty(b - a, np.float64))
    st = fj.shard_solve(shards, sl, zl, eps, omega, zprime_list=zpl)
    tohost = (lambda t: t.cpu().numpy()) if on_device else (lambda t: t)
    z = np.concatenate([tohost(t) for t in zl]).astype(np.float64)
    zp = np.concatenate([tohost(t) for t in zpl])
    m = fj.shard_measures(shards, zl, sl)
    for sh in shards:
        sh.close()
    comm.close()
    return st, z, zp, m


@pytest.mark.parametrize("name", sorted(TINY))
@pytest.mark.parametrize("W", [1, 2, 3, 5])
def test_shard_parity(dev, name, W):
    rp, col, w, s, directed = TINY[name]()
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, W)
    assert st.status == 0 and st.cert_ratio <= 1.0, st
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    ref = oracle.solve(rp, col, w, s, 1e-6, 1.0)
    assert rel_err(z, ref.z) <= 1e-4
    om = oracle.measures(rp, col, w, z.astype(np.float32).astype(np.float64), directed=directed,
                         s=np.asarray(s, np.float64))
    for k in ("P", "D", "I", "C"):
        assert abs(m[k] - om[k]) <= 1e-9 * abs(om[k]) + 1e-300, (k, m[k], om[k])


@pytest.mark.parametrize("name", ["lattice64", "rmat12w", "er2000"])
def test_shard_halo_exact(dev, name):
    """Each shard receives exactly the distinct remote nodes its rows read."""
    rp, col, w, s, directed = TINY[name]()
    n = len(rp) - 1
    orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
    begin = np.array(fj.shard_plan(orp, 4))
    comm = fj.Comm.in_process(4)
    shards = make_shards(comm, rp, col, w, directed, begin, True, dev)
    assert all(sh.info()[1] == 0 for sh in shards)
    fj.shard_connect(shards)
    for r, sh in enumerate(shards):
        c = ocol[orp[begin[r]]:orp[begin[r + 1]]]
        remote = np.unique(c[(c < begin[r]) | (c >= begin[r + 1])])
        assert sh.info() == (int(begin[r + 1] - begin[r]), len(remote))
    if name == "lattice64":  # a grid split into row bands: the halo is the band edges
        assert sum(sh.info()[1] for sh in shards) < 0.15 * n
    for sh in shards:
        sh.close()
    comm.close()


@pytest.mark.parametrize("name", ["rmat12w", "chunglu4k", "lattice64", "dirw-dense"])
@pytest.mark.parametrize("W", [2, 3, 5])
def test_shard_loopback_nccl_bookkeeping(dev, name, W):
    """fj_comm_create_loopback: the in-process transport runs the NCCL path's
    send lists, pack kernel and per-peer segments, with device copies in place
    of ncclSend/ncclRecv — the multi-rank logic one GPU can check."""
    rp, col, w, s, directed = TINY[name]()
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, W, loopback=True)
    assert st.status == 0 and st.cert_ratio <= 1.0
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    assert rel_err(z, oracle.solve(rp, col, w, s, 1e-6, 1.0).z) <= 1e-4
    om = oracle.measures(rp, col, w, z.astype(np.float32).astype(np.float64), directed=directed)
    assert abs(m["D"] - om["D"]) <= 1e-9 * abs(om["D"])


def test_shard_host_pointers(dev):
    rp, col, w, s, directed = TINY["rmat12w"]()
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, 3, on_device=False)
    assert st.status == 0
    assert rel_err(z, oracle.solve(rp, col, w, s, 1e-6, 1.0).z) <= 1e-4


def test_shard_ragged_partition(dev):
    """Parts of very different sizes, including one node."""
    rp, col, w, s, directed = TINY["er2000"]()
    begin = np.array([0, 1, 2, 1000, 1999, 2000], np.int64)
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, 5, begin=begin)
    assert st.status == 0
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0


def test_shard_isolated_and_long_rows(dev):
    """A star hub with 3000 arcs (several warp pieces) split from its leaves,
    plus isolated nodes (rows with d = 0 solved at init, reading R20)."""
    k = 3000
    edges = [(0, j) for j in range(1, k + 1)]
    n = k + 11
    rp, col, w = G.in_csr_from_edges(n, edges)
    s = fjgen.uniform(n, 5)
    begin = np.array([0, 1, 1500, n], np.int64)
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, False, 3, begin=begin)
    assert st.status == 0
    assert rel_err(z, oracle.dense_solve(rp, col, w, s)) <= 1e-4


def test_shard_matches_single_gpu(dev):
    rp, col, w, s, directed = TINY["chunglu4k"]()
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.0, directed, 4)
    g = fj.Graph(len(rp) - 1, rp, col, w, directed=directed)
    z1 = np.empty(len(rp) - 1, np.float32)
    fj.solve(g, np.asarray(s, np.float32), z1, 1e-6, 1.0)
    g.close()
    # both within ε·max(|z|, σ) of z (Lemma 5 with reading R5)
    assert np.max(np.abs(z - z1) / np.maximum(np.abs(z1), SIG)) <= 4e-6


def test_shard_sor_undirected(dev):
    """ω > 1 across shards (block-Jacobi outside, in-place SOR inside): when it
    converges it is certified and matches the oracle."""
    rp, col, w, s, directed = TINY["er2000"]()
    st, z, zp, m = sharded_solve(dev, rp, col, w, s, 1e-6, 1.2, directed, 2)
    assert st.status == 0
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0


def test_shard_nccl_one_rank(dev):
    """The NCCL transport end to end with a one-rank communicator."""
    rp, col, w, s, directed = TINY["rmat12w"]()
    n = len(rp) - 1
    comm = fj.Comm.nccl(fj.comm_unique_id(), 0, 1)
    orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
    begin = np.array([0, n], np.int64)
    sh = fj.Shard(comm, 0, n, begin, orp, ocol, ow, directed=directed)
    fj.shard_connect([sh])
    z = np.empty(n, np.float32)
    zp = np.empty(n, np.float64)
    st = fj.shard_solve([sh], [np.asarray(s, np.float32)], [z], 1e-6, 1.0, zprime_list=[zp])
    assert st.status == 0
    assert oracle.certificate(rp, col, w, s, zp, 1e-6)[0] <= 1.0
    assert rel_err(z.astype(np.float64), oracle.solve(rp, col, w, s, 1e-6, 1.0).z) <= 1e-4
    m = fj.shard_measures([sh], [z])
    om = oracle.measures(rp, col, w, z.astype(np.float64), directed=directed)
    assert abs(m["P"] - om["P"]) <= 1e-9 * om["P"] and abs(m["D"] - om["D"]) <= 1e-9 * om["D"]
    sh.close()
    comm.close()


def test_shard_invalid(dev):
    rp, col, w, s, directed = TINY["er2000"]()
    n = len(rp) - 1
    orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
    comm = fj.Comm.in_process(2)
    begin = np.array([0, 1000, n], np.int64)
    srp, scol, _ = fjgen.shard_rows(orp, ocol, None, begin, 0)
    bad_cases = [
        dict(begin=np.array([0, 1000, n - 1], np.int64)),            # begin[W] != n
        dict(begin=np.array([0, 0, n], np.int64)),                   # empty part
        dict(rank=2),                                                # rank out of range
        dict(col=np.where(scol == scol[0], n + 5, scol).astype(np.int32)),  # id out of range
        dict(col=np.where(np.arange(len(scol)) == 0, 0, scol).astype(np.int32)),  # self-loop / order
        dict(col=scol[::-1].copy()),                                 # unsorted rows
        dict(rp=np.concatenate([srp[:-1], [srp[-1] + 1]]).astype(np.int64)),  # bad row_ptr end
    ]
    for case in bad_cases:
        args = dict(rank=0, begin=begin, rp=srp, col=scol)
        args.update(case)
        with pytest.raises(fj.FJError) as e:
            fj.Shard(comm, args["rank"], n, args["begin"], args["rp"], args["col"])
        assert "status 2" in str(e.value)
    sh0 = fj.Shard(comm, 0, n, begin, srp, scol)
    with pytest.raises(fj.FJError):
        fj.shard_connect([sh0])                     # a local comm needs all shards
    srp1, scol1, _ = fjgen.shard_rows(orp, ocol, None, begin, 1)
    sh1 = fj.Shard(comm, 1, n, begin, srp1, scol1)
    with pytest.raises(fj.FJError):
        fj.shard_connect([sh1, sh0])                # rank order
    z = [np.empty(1000, np.float32), np.empty(n - 1000, np.float32)]
    sl = [np.asarray(s[:1000], np.float32), np.asarray(s[1000:], np.float32)]
    with pytest.raises(fj.FJError):
        fj.shard_solve([sh0, sh1], sl, z, 1e-6)     # not connected
    fj.shard_connect([sh0, sh1])
    with pytest.raises(fj.FJError):
        fj.shard_solve([sh0, sh1], sl, z, 1e-6, omega=2.5)
    st = fj.shard_solve([sh0, sh1], sl, z, 1e-6)
    assert st.status == 0
    sh0.close()
    sh1.close()
    comm.close()
