"""Host-side logic of the sharded path (row f4) on CPU: the partition plan,
the per-rank out-row slices, and the two-process (gloo, world_size 2)
exchange of the NCCL id and of the slices a multi-GPU run performs before
any device work."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import fjgen

fj = pytest.importorskip("paper_2507_14864_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _work(rp, a, b):
    return int(rp[b] - rp[a]) + (b - a)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_properties(seed, world):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(world, 400))
    deg = rng.zipf(2.0, n).clip(0, 5000) * rng.integers(0, 2, n)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    begin = np.array(fj.shard_plan(rp, world))
    assert begin[0] == 0 and begin[-1] == n
    assert np.all(np.diff(begin) >= 1)
    total = int(rp[-1]) + n
    maxrow = int(np.max(np.diff(rp))) + 1
    for r in range(world):
        assert _work(rp, begin[r], begin[r + 1]) <= total / world + maxrow + 1


def test_shard_plan_extremes():
    rp = np.arange(0, 11, dtype=np.int64)  # 10 rows, one arc each
    assert list(fj.shard_plan(rp, 10)) == list(range(11))
    assert list(fj.shard_plan(rp, 1)) == [0, 10]
    assert list(fj.shard_plan(rp, 2)) == [0, 5, 10]
    for bad in [(rp, 0), (rp, 11), (np.array([1, 2], np.int64), 1),
                (np.array([0, 3, 2], np.int64), 1)]:
        with pytest.raises(fj.FJError):
            fj.shard_plan(*bad)


@pytest.mark.parametrize("directed", [False, True])
def test_shard_rows_reassemble(directed):
    if directed:
        rp, col = fjgen.rmat_graph(9, 8, 4)
        w = fjgen.arc_weights(rp, col, 4)
    else:
        rp, col = fjgen.er_graph(700, 6.0, 4)
        w = None
    orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
    begin = np.array(fj.shard_plan(orp, 3))
    parts = [fjgen.shard_rows(orp, ocol, ow, begin, r) for r in range(3)]
    lens = np.concatenate([np.diff(p[0]) for p in parts])
    assert np.array_equal(lens, np.diff(orp))
    assert np.array_equal(np.concatenate([p[1] for p in parts]), ocol)
    if w is not None:
        assert np.array_equal(np.concatenate([p[2] for p in parts]), ow)
    # every arc u→v of the in-CSR appears in row u of the out-CSR
    n = len(rp) - 1
    v_of = np.repeat(np.arange(n), np.diff(rp))
    arcs_in = set(zip(col.tolist(), v_of.tolist()))
    u_of = np.repeat(np.arange(n), np.diff(orp))
    assert arcs_in == set(zip(u_of.tolist(), ocol.tolist()))


_WORKER = r'''
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch.distributed as dist
import fjgen, paper_2507_14864_b200 as fj
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
# the NCCL id travels as bytes from rank 0 (as bench.py --mode sharded does)
box = [fj.comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(box, src=0)
uid = box[0]
assert isinstance(uid, bytes) and len(uid) == 128
ids = [None] * world
dist.all_gather_object(ids, uid)
assert all(i == uid for i in ids)
# every rank derives the same plan and its own slice; rank 0 reassembles
rp, col = fjgen.rmat_graph(10, 8, 9)
w = fjgen.arc_weights(rp, col, 9)
orp, ocol, ow = fjgen.to_out_csr(rp, col, w)
begin = np.array(fj.shard_plan(orp, world))
plans = [None] * world
dist.all_gather_object(plans, begin.tolist())
assert all(p == begin.tolist() for p in plans)
mine = fjgen.shard_rows(orp, ocol, ow, begin, rank)
parts = [None] * world
dist.all_gather_object(parts, (rank, mine[0].tolist(), mine[1].tolist(), mine[2].tolist()))
parts.sort()
lens = np.concatenate([np.diff(p[1]) for p in parts])
assert np.array_equal(lens, np.diff(orp))
assert np.array_equal(np.concatenate([p[2] for p in parts]), ocol)
assert np.array_equal(np.concatenate([p[3] for p in parts]).astype(np.float32), ow)
dist.barrier()
dist.destroy_process_group()
open(os.path.join(sys.argv[2], f"ok{rank}"), "w").write("ok")
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_world2_gloo(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(script), ROOT, str(tmp_path)]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()
