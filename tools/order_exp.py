"""Does the Gauss–Seidel order change the sweep count?  (diagnostics)

The ASYNC sweep visits rows roughly in layout order: length class, then id.
Relabelling node ids changes the order inside each class.  Orders tried:
  id       the generator's ids (R-MAT: low ids are hubs)
  level    increasing shortest distance to a node with no out-arcs, along
           reversed arcs (information flows from sinks to their listeners)
  level_r  decreasing level
  random   a seeded random permutation
usage: python tools/order_exp.py CID [CID ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402


def sink_levels(rp, col, n):
    """BFS from the nodes with zero out-degree over the in-CSR (row v lists
    the u with u→v, i.e. v's listeners)."""
    outdeg = np.bincount(col, minlength=n)
    lev = np.full(n, np.iinfo(np.int32).max, np.int64)
    front = np.flatnonzero(outdeg == 0)
    lev[front] = 0
    k = 0
    while len(front):
        k += 1
        starts, ends = rp[front], rp[front + 1]
        lens = ends - starts
        idx = np.repeat(starts - np.cumsum(np.r_[0, lens[:-1]]), lens) + np.arange(lens.sum())
        nb = np.unique(col[idx])
        nb = nb[lev[nb] > k]
        lev[nb] = k
        front = nb
    return lev


def relabel(rp, col, w, s, new_of_old):
    n = len(rp) - 1
    old_of_new = np.argsort(new_of_old)
    lens = np.diff(rp)[old_of_new]
    nrp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=nrp[1:])
    starts = rp[old_of_new]
    idx = np.repeat(starts - nrp[:-1], lens) + np.arange(nrp[-1])
    ncol = new_of_old[col[idx]].astype(np.int32)
    nw = None if w is None else w[idx]
    # rows must be sorted for a canonical input; the library sorts if not
    return nrp, ncol, nw, s[old_of_new], old_of_new


dev = torch.device("cuda:0")
for cid in [int(a) for a in sys.argv[1:]]:
    p = fjgen.config(cid)
    n = p.n
    lev = sink_levels(p.row_ptr, p.col, n)
    fin = lev[lev < np.iinfo(np.int32).max]
    print(f"C{cid}: levels 0..{fin.max()}, {np.bincount(fin).tolist()[:12]} ..., "
          f"unreached {int((lev == np.iinfo(np.int32).max).sum())}", flush=True)
    rng = np.random.default_rng(7)
    orders = {
        "id": np.arange(n),
        "level": np.argsort(np.argsort(lev, kind="stable"), kind="stable"),
        "level_r": np.argsort(np.argsort(-lev, kind="stable"), kind="stable"),
        "random": rng.permutation(n),
    }
    for name, new_of_old in orders.items():
        rp, col, w, s, _ = relabel(p.row_ptr, p.col, p.w, p.s, new_of_old.astype(np.int64))
        g = fj.Graph(n, torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev),
                     None if w is None else torch.from_numpy(w).to(dev), directed=p.directed)
        st_ = torch.from_numpy(s).to(dev)
        z = torch.empty(n, dtype=torch.float32, device=dev)
        best = None
        for _ in range(2):
            st = fj.solve(g, st_, z, 1e-6, 1.0, method="async")
            best = st if best is None or st.solve_ms < best.solve_ms else best
        print(f"  {name:8s} sweeps {best.sweeps:4d}  solve {best.solve_ms:7.1f} ms  "
              f"{best.sweep_ms / best.sweeps:.3f} ms/sweep  EU {best.edge_updates / p.m:.0f}·m",
              flush=True)
        g.close()
