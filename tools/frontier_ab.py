"""A/B of the frontier phase (fj_opts.frontier) on full configs (diagnostics).
usage: python tools/frontier_ab.py CIDS OMEGA [FRONTIERS]   FRONTIERS: comma list (0 = off, -1 = default, T)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

cids = [int(c) for c in sys.argv[1].split(",")]
om = float(sys.argv[2])
fronts = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "0,-1").split(",")]
reps = int(os.environ.get("AB_REPS", "5"))
dev = torch.device("cuda:0")
T = lambda a: None if a is None else torch.from_numpy(a).to(dev)  # noqa: E731
for cid in cids:
    p = fjgen.config(cid)
    n = len(p.row_ptr) - 1
    g = fj.Graph(n, T(p.row_ptr), T(p.col), T(p.w), directed=p.directed)
    s = T(p.s)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    zref = None
    for fr in fronts:
        res = []
        for r in range(reps):
            st = fj.solve(g, s, z, 1e-6, om, raise_on_numeric=False, max_sweeps=4000, frontier=fr)
            res.append(st)
        res.sort(key=lambda t: t.solve_ms)
        t = res[len(res) // 2]
        if zref is None:
            zref = z.clone()
            dz = 0.0
        else:
            dz = float(((z - zref).abs() / zref.abs().clamp_min(1e-5)).max())
        print(f"C{cid} w={om} frontier={fr:6d} {t.solve_ms:8.1f} ms  sweeps {t.sweeps} (shadow {t.shadow_sweeps}) "
              f"rounds {t.frontier_rounds} pushes {t.frontier_pushes} front_ms {t.frontier_ms:.2f} "
              f"cert {t.cert_ratio:.4f} cr {t.cert_rounds} status {t.status} relax {t.relaxations} eu {t.edge_updates:.4g} "
              f"dz {dz:.1e}  all " + " ".join(f"{x.solve_ms:.1f}/{x.sweeps}/{x.frontier_rounds}" for x in res), flush=True)
    g.close()
