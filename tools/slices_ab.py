"""A/B of row slices vs warp tiles (fj_opts.slices) on full configs (diagnostics).

usage: python tools/slices_ab.py CIDS OMEGA [METHOD] [SHADOWS]
One process per config; every variant solves the same resident graph AB_REPS times."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

cids = [int(c) for c in sys.argv[1].split(",")]
om = float(sys.argv[2])
method = sys.argv[3] if len(sys.argv) > 3 else "auto"
shadows = [int(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "-1").split(",")]
reps = int(os.environ.get("AB_REPS", "3"))
dev = torch.device("cuda:0")
T = lambda a: None if a is None else torch.from_numpy(a).to(dev)  # noqa: E731
for cid in cids:
    p = fjgen.config(cid)
    n = len(p.row_ptr) - 1
    g = fj.Graph(n, T(p.row_ptr), T(p.col), T(p.w), directed=p.directed)
    s = T(p.s)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    zref = None
    for sh in shadows:
        for sl in (0, 1, 0, 1):
            res = []
            for r in range(reps):
                st = fj.solve(g, s, z, 1e-6, om, method=method, raise_on_numeric=False,
                              max_sweeps=4000, shadow=sh, slices=sl)
                res.append(st)
            res.sort(key=lambda t: t.solve_ms)
            t = res[len(res) // 2]
            fs = t.sweeps - t.shadow_sweeps
            shms = t.shadow_ms / max(1, t.shadow_sweeps)
            fms = (t.sweep_ms - t.shadow_ms) / max(1, fs)
            if zref is None:
                zref = z.clone()
                dz = 0.0
            else:
                dz = float(((z - zref).abs() / zref.abs().clamp_min(1e-5)).max())
            print(f"C{cid} w={om} {method} shadow={sh:2d} slices={sl} "
                  f"{t.solve_ms:8.1f} ms  sweeps {t.sweeps} (shadow {t.shadow_sweeps} @ {shms:.4f} ms, "
                  f"fp64 {fs} @ {fms:.4f} ms)  cert {t.cert_ratio:.4f} rounds {t.cert_rounds} "
                  f"status {t.status} colors {t.colors} eu {t.edge_updates:.4g} dz_vs_first {dz:.2e}  all "
                  + " ".join(f"{x.solve_ms:.1f}/{x.sweeps}" for x in res), flush=True)
    g.close()
