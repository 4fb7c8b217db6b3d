"""Sharded solve (row f4) at full size on ONE GPU with the in-process transport:
what the block-Jacobi split costs in sweeps and what the per-sweep exchange
and reductions cost in time, against the single-GPU solve (diagnostics).

usage: python tools/shard_exp.py CID [CID ...]   (env SHARDS=1,2,4,8)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

dev = torch.device("cuda:0")
for cid in [int(a) for a in sys.argv[1:]]:
    p = fjgen.config(cid)
    eps = 1e-6
    g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
                 None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
    s = torch.from_numpy(p.s).to(dev)
    z = torch.empty(p.n, dtype=torch.float32, device=dev)
    best = None
    for _ in range(3):
        st = fj.solve(g, s, z, eps, 1.0, method="async")
        best = st if best is None or st.solve_ms < best.solve_ms else best
    print(f"C{cid} single GPU: sweeps {best.sweeps} solve {best.solve_ms:.1f} ms "
          f"({best.solve_ms / best.sweeps:.3f} ms/sweep)", flush=True)
    z1 = z.cpu().numpy()
    g.close()
    orp, ocol, ow = fjgen.to_out_csr(p.row_ptr, p.col, p.w)
    for W in [int(x) for x in os.environ.get("SHARDS", "1,2,4,8").split(",")]:
        begin = fj.shard_plan(orp, W)
        comm = fj.Comm.in_process(W)
        t0 = time.time()
        shards = []
        for r in range(W):
            srp, scol, sw = fjgen.shard_rows(orp, ocol, ow, begin, r)
            shards.append(fj.Shard(comm, r, p.n, begin, torch.from_numpy(srp).to(dev),
                                   torch.from_numpy(scol).to(dev),
                                   None if sw is None else torch.from_numpy(sw).to(dev),
                                   directed=p.directed))
        fj.shard_connect(shards)
        torch.cuda.synchronize()
        tb = time.time() - t0
        halo = sum(sh.info()[1] for sh in shards) / W
        sl = [s[begin[r]:begin[r + 1]].contiguous() for r in range(W)]
        zl = [torch.empty(begin[r + 1] - begin[r], dtype=torch.float32, device=dev)
              for r in range(W)]
        bs = None
        for _ in range(2):
            st = fj.shard_solve(shards, sl, zl, eps, 1.0)
            bs = st if bs is None or st.solve_ms < bs.solve_ms else bs
        zs = torch.cat(zl).cpu().numpy()
        dz = float(np.max(np.abs(zs - z1) / np.maximum(np.abs(z1), 1e-5)))
        print(f"  W={W}: build {tb * 1e3:.0f} ms, halo/rank {halo / p.n:.3f}·n, sweeps {bs.sweeps}, "
              f"solve {bs.solve_ms:.1f} ms, "
              f"sweep kernels {bs.sweep_ms:.1f} ms ({bs.sweep_ms / bs.sweeps:.3f} ms/sweep), "
              f"cert {bs.cert_ratio:.3f}, max rel dz vs single {dz:.1e}", flush=True)
        for sh in shards:
            sh.close()
        comm.close()
