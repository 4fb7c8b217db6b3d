"""Relative-error harness of the paper's accuracy tables (tab:measure_li,
PAPER.md P:639).

For each config and each ε, BLI (ω = 1) and BLISOR (the config's tuned ω) are
solved through the C-ABI; every quantity ρ — the maximum over v of the
relative error of z_v, and the measures C, D, I, P (tab:measures) — is
compared with an exact reference as σ = |ρ − ρ̃| / |ρ|.  The
reference is independent of the GPU path: a sparse direct solve of
(I+L)z = s (scipy SuperLU) for the ER config, and a tightly converged Krylov
solve (CG for undirected, BiCGSTAB for directed, relative residual 1e-13)
for the larger ones, with the measures of that z computed by the oracle.

usage: python tests/harness/accuracy_table.py [CID ...]   (default 1 2 5)
"""
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import fjgen  # noqa: E402
import oracle  # noqa: E402
import paper_2507_14864_b200 as fj  # noqa: E402

TUNED = {1: 1.5, 2: 1.4, 3: 1.6, 4: 1.6, 5: 1.25}


def system(p):
    """(I + L) as a scipy CSR matrix: row u has 1 + d_u on the diagonal and −a_uv
    for its out-arcs u→v; the in-CSR row v lists the u with u→v."""
    n = p.n
    v = np.repeat(np.arange(n), np.diff(p.row_ptr))
    u = p.col.astype(np.int64)
    a = np.ones(len(u)) if p.w is None else p.w.astype(np.float64)
    A = sp.csr_matrix((a, (u, v)), shape=(n, n))
    d = np.asarray(A.sum(axis=1)).ravel()
    return (sp.identity(n, format="csr") + sp.diags(d) - A).tocsr()


def reference(p, cid):
    M = system(p)
    s = p.s.astype(np.float64)
    t0 = time.time()
    if cid == 1:
        z = spla.spsolve(M.tocsc(), s)
        how = "sparse LU"
    elif not p.directed:
        z, info = spla.cg(M, s, rtol=1e-13, maxiter=200000)
        how = f"CG (info {info})"
    else:
        z, info = spla.bicgstab(M, s, rtol=1e-13, maxiter=200000)
        how = f"BiCGSTAB (info {info})"
    res = np.linalg.norm(M @ z - s) / np.linalg.norm(s)
    return z, f"{how}, rel. residual {res:.1e}, {time.time() - t0:.1f} s"


def rel(a, b):
    return abs(a - b) / abs(b)


def main():
    cids = [int(a) for a in sys.argv[1:]] or [1, 2, 5]
    dev = torch.device("cuda:0")
    for cid in cids:
        p = fjgen.config(cid)
        zref, how = reference(p, cid)
        mref = oracle.measures(p.row_ptr, p.col, p.w, zref, directed=p.directed,
                               s=p.s.astype(np.float64))
        print(f"# {p.name}: reference {how}", flush=True)
        g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev),
                     None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
        s = torch.from_numpy(p.s).to(dev)
        z = torch.empty(p.n, dtype=torch.float32, device=dev)
        for eps in [1e-2, 1e-3, 1e-4, 1e-5, 1e-6]:
            for name, om in [("BLI", 1.0), ("BLISOR", TUNED[cid])]:
                st = fj.solve(g, s, z, eps, om, raise_on_numeric=False)
                if st.status != 0:
                    print(json.dumps({"config": cid, "eps": eps, "alg": name, "omega": om,
                                      "status": st.status}), flush=True)
                    continue
                zg = z.cpu().numpy().astype(np.float64)
                m = fj.measures(g, z, s)
                zerr = float(np.max(np.abs(zg - zref) / np.maximum(np.abs(zref), 1e-5)))  # σ (R5)
                row = {"config": cid, "eps": eps, "alg": name, "omega": om,
                       "time_ms": round(st.solve_ms, 3), "sweeps": st.sweeps,
                       "z_max_rel": zerr, "C": rel(m["C"], mref["C"]), "D": rel(m["D"], mref["D"]),
                       "I": rel(m["I"], mref["I"]), "P": rel(m["P"], mref["P"])}
                print(json.dumps(row), flush=True)
        g.close()


if __name__ == "__main__":
    main()
