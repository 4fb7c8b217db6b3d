"""Thin-sweep threshold of the batched solve's frontier phase on config 4 (diagnostics).
usage: python tools/batch_frontier_ab.py K T[,T...]   (T rows per right-hand side; 0 = off, -1 = default)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

k = int(sys.argv[1])
Ts = [int(t) for t in sys.argv[2].split(",")]
dev = torch.device("cuda:0")
p = fjgen.config(4)
g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
             torch.from_numpy(p.w).to(dev), directed=p.directed)
cols = [p.s, fjgen.exponential(p.n, 21), fjgen.pareto(p.n, 22), fjgen.uniform(p.n, 23),
        fjgen.uniform(p.n, 24), fjgen.exponential(p.n, 26), fjgen.pareto(p.n, 27), fjgen.beta25(p.n, 28)]
S = torch.from_numpy(np.ascontiguousarray(np.stack(cols[:k], 1).astype(np.float32)).ravel()).to(dev)
Z = torch.empty(p.n * k, dtype=torch.float32, device=dev)
for T in Ts:
    res = [fj.solve_batch(g, S, Z, k, 1e-6, 1.0, frontier=T) for _ in range(3)]
    res.sort(key=lambda t: t.solve_ms)
    t = res[1]
    print(f"k={k} T={T:8d} {t.solve_ms:8.1f} ms sweeps {t.sweeps} rounds {t.frontier_rounds} "
          f"pushes {t.frontier_pushes} eu/s {t.edge_updates / t.solve_ms * 1e3:.4g} cert {t.cert_ratio:.4f} "
          f"all " + " ".join(f"{x.solve_ms:.0f}/{x.sweeps}" for x in res), flush=True)
g.close()
