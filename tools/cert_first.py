import sys, torch
sys.path.insert(0, '/root/repo')
import fjgen, paper_2507_14864_b200 as fj
dev = torch.device("cuda:0")
T = lambda a: None if a is None else torch.from_numpy(a).to(dev)
for cid in (3, 5, 1):
    p = fjgen.config(cid)
    n = len(p.row_ptr) - 1
    g = fj.Graph(n, T(p.row_ptr), T(p.col), T(p.w), directed=p.directed)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    for cr in (0, 3):
        st = fj.solve(g, T(p.s), z, 1e-6, 1.0, raise_on_numeric=False, cert_rounds=cr)
        print(cid, 'cert_rounds', cr, 'ratio', st.cert_ratio, 'sweeps', st.sweeps, 'rounds', st.cert_rounds, 'ms', st.solve_ms, flush=True)
    g.close()
