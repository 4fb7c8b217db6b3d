"""PUSH (frontier push with compacted frontiers) vs ASYNC on full configs (diagnostics).
usage: PUSH_SPARSE_DIV=d python tools/push_exp.py CID [CID ...]"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
for cid in [int(x) for x in sys.argv[1:]]:
    p = fjgen.config(cid)
    g = fj.Graph(p.n, torch.from_numpy(p.row_ptr).to(dev), torch.from_numpy(p.col).to(dev), None if p.w is None else torch.from_numpy(p.w).to(dev), directed=p.directed)
    s = torch.from_numpy(p.s).to(dev); z = torch.empty(p.n, dtype=torch.float32, device=dev)
    for meth in ["push", "async"]:
        best=None
        for _ in range(2):
            st = fj.solve(g, s, z, 1e-6, 1.0, method=meth, push_compact=True,
                          push_sparse_div=int(os.environ.get("PUSH_SPARSE_DIV", "8")))
            best = st if best is None or st.solve_ms < best.solve_ms else best
        print(f"C{cid} {meth:6s} div={os.environ.get('PUSH_SPARSE_DIV','8')}: sweeps {best.sweeps} solve {best.solve_ms:.1f} ms EU {best.edge_updates/p.m:.0f}m cert {best.cert_ratio:.3f}", flush=True)
    g.close()
