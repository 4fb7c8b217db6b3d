"""Sweeps of a warm start from a certified state, repeated (diagnostics for test_warm_start_resume)."""
import sys, os, collections
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2507_14864_b200 as fj
from tests.test_gpu_parity import TINY, _t
dev = torch.device("cuda:0")
for name in ["er2000", "rmat12w", "lattice64"]:
    rp, col, w, s, directed = TINY[name]()
    n = len(rp) - 1
    cnt = collections.Counter(); rel = 0
    for r in range(60):
        g = fj.Graph(n, _t(rp, dev), _t(col, dev), _t(w, dev), directed=directed)
        z = torch.empty(n, dtype=torch.float32, device=dev)
        zp = torch.empty(n, dtype=torch.float64, device=dev)
        fj.solve(g, _t(s, dev), z, 1e-2, 1.0)
        warm = fj.solve(g, _t(s, dev), z, 1e-6, 1.0, z_init=z.double(), zprime_out=zp)
        again = fj.solve(g, _t(s, dev), z, 1e-6, 1.0, z_init=(zp - warm.c).contiguous())
        cnt[again.sweeps] += 1; rel = max(rel, again.relaxations)
        g.close()
    print(name, n, dict(cnt), "max relaxations", rel, flush=True)
